/*
 * pase.h -- C ABI of the B200-native PaSE strategy-search hot path
 * ("PaSE: Parallelization Strategies for Efficient DNN Training", arXiv 2407.04001).
 *
 * Citation convention: P:<n> = /root/reference/PAPER.md line n (section / equation /
 * figure named alongside).  DESIGN.md §2 lists every reading of an ambiguous passage.
 *
 * What the library computes (one call to pase_solve = the whole hot path):
 *   a1 graph ingest/validation       G = (V, E), weakly connected (§2)
 *   a2 configurations C(v)           d-tuples, c_k | size_k, prod c_k = p
 *   a3 SortNodes + D(i)              Fig. 4
 *   a4 elimination tree              children(i) = {j : min-rank D(j) = i}; equals Fig. 5's
 *                                    connected subsets S(i)
 *   a5 cost tables (GPU)             L_v[C] = t_l(v,C,r); W_e = r*t_x (Eq. 1)
 *   a6 DP fill (GPU)                 Eq. 4 / Fig. 5 lines 8-20:
 *                                    T(i)[phi] = min_C L[C] + sum_{e in E>(sigma_i)} W_e + sum_j T(j)[phi'|D(j)]
 *   a7 back-substitution (GPU)       from sigma_|V|.cfg
 *   a8 total cost                    f(|V|, ∅) = T(|V|)[0]
 *
 * Conventions for every entry point:
 *   - all functions are extern "C", never throw, and return pase_status;
 *   - pointers are HOST pointers unless the name ends in _dev;
 *   - caller-allocated outputs; the library never retains caller pointers after return;
 *   - a pase_ctx is not thread-safe; distinct contexts are independent.
 *   - errors: PASE_ERR_INVALID (bad input; message names the node / edge), PASE_ERR_RESOURCE
 *     (size guard or allocation failure; message carries M and K, cf. Table 1 "OOM"),
 *     PASE_ERR_CUDA / PASE_ERR_NCCL (runtime failures), PASE_ERR_STATE (call out of order).
 *     pase_last_error(ctx) returns the message (valid until the next call on ctx);
 *     pase_last_error(NULL) returns the message of the last failed pase_create.
 */
#ifndef PASE_H
#define PASE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PASE_MAX_DIMS 8      /* iteration-space dimensions per vertex */
#define PASE_MAX_HALO 4      /* conv halo (spatial, filter) pairs per vertex */
#define PASE_MAX_DEP 12      /* max |D(i)| (M); larger -> PASE_ERR_RESOURCE */
#define PASE_HANDLE_BYTES 256 /* pase_export_handle blob */
#define PASE_MAX_WORLD 8     /* search GPUs in one group */

typedef enum {
    PASE_OK = 0,
    PASE_ERR_INVALID = 1,
    PASE_ERR_RESOURCE = 2,
    PASE_ERR_CUDA = 3,
    PASE_ERR_NCCL = 4,
    PASE_ERR_STATE = 5
} pase_status;

/* C(v) policy (DESIGN reading B).  Both require c_k | size_k ("equal parts").
 * EXACT_P: prod c_k = p (north star); if no tuple reaches p, the tuples of the largest
 * achievable product <= p.  LE_P: prod c_k <= p (the set-builder of P:204-205). */
typedef enum { PASE_CFG_EXACT_P = 0, PASE_CFG_LE_P = 1 } pase_cfg_policy;

/* Vertex ordering: SortNodes (Fig. 4; the paper's DP-Alg) or breadth-first
 * (Table 1's "BF" baseline) -- same Eq. 4 DP over either; the BF
 * ordering's dependent sets grow large on Inception/Transformer and trip the size guard
 * (PASE_ERR_RESOURCE, the paper's "OOM"). */
typedef enum { PASE_ORDER_SORTNODES = 0, PASE_ORDER_BFS = 1 } pase_ordering;

/* One vertex = one layer with its iteration space. */
typedef struct {
    int32_t n_dims;                        /* 1..PASE_MAX_DIMS */
    int64_t size[PASE_MAX_DIMS];           /* extents, 1 <= size < 2^31 */
    uint32_t splittable_mask;              /* bit k: dim k may be split */
    int32_t n_out_axes;                    /* output tensor rank, 1..n_dims */
    int32_t out_axes[PASE_MAX_DIMS];       /* iteration dim of each output-tensor axis (distinct) */
    int32_t n_w_axes;                      /* 0 = no weight */
    int32_t w_axes[PASE_MAX_DIMS];         /* iteration dims indexing the weight (distinct) */
    uint32_t flop_dims_mask;               /* dims in the FLOP product; 0 = all dims */
    int64_t flops_per_point;               /* fwd+bwd FLOPs per iteration point (e.g. 6 for GEMM) */
    int32_t n_halo;                        /* 0..PASE_MAX_HALO */
    int32_t halo_spatial[PASE_MAX_HALO];   /* spatial iteration dim h ... */
    int32_t halo_filter[PASE_MAX_HALO];    /* ... paired with filter dim r */
    int32_t elem_bytes;                    /* bytes per tensor element, >= 1 */
    int32_t n_in_axes;                     /* input tensor rank, 0..n_dims (0 = not given) */
    int32_t in_axes[PASE_MAX_DIMS];        /* iteration dim of each input-tensor axis (distinct; conv:
                                              b, c, h, w).  The halo of pair q exchanges
                                              (size[r] - 1) input rows whose face is the product of the
                                              shard extents of the input axes other than h (DESIGN
                                              reading L); every halo_spatial[q] must be one of
                                              them, else PASE_ERR_INVALID */
} pase_node;

/* Tensor flowing src -> dst.  axis_map[a] = dst iteration dim aligned with
 * src output axis a (a < src.n_out_axes), or -1 (consumer does not split it). */
typedef struct {
    int32_t src, dst;
    int32_t axis_map[PASE_MAX_DIMS];
} pase_edge;

typedef struct {
    int32_t n_nodes;
    const pase_node* nodes;    /* node id = index */
    int32_t n_edges;
    const pase_edge* edges;    /* edge id = index; parallel / antiparallel edges allowed */
} pase_graph;

/* Machine model: r = F / B computed once in fp64. */
typedef struct {
    double flops_per_device;           /* F, FLOP/s */
    double link_bandwidth;             /* B, bytes/s (may be +inf: r = 0) */
    int32_t cfg_policy;                /* pase_cfg_policy */
    int32_t ordering;                  /* pase_ordering (0 = SortNodes) */
    uint64_t table_budget_bytes;       /* size guard over all DP tables; 0 = 64 GiB */
    uint64_t redundant_below_bytes;    /* multi-GPU: tables smaller than this are computed on every
                                          rank; bigger ones are partitioned */
    int32_t cuda_device;               /* device ordinal for this process; < 0 = host-only planning
                                          context (a1-a4 + stats + introspection; pase_solve and the
                                          table hooks return PASE_ERR_STATE; no device is touched) */
    int32_t rank, world;               /* search GPUs G in [1, PASE_MAX_WORLD]; world = 1: single GPU */
    int32_t virtual_ranks;             /* 1: all ranks of the group share one device (testing):
                                          each rank's persistent grid uses 1/world of the SMs */
    const void* reserved;              /* must be NULL */
    void* cuda_stream;                 /* cudaStream_t to run on; NULL = library-owned stream */
} pase_machine;

typedef struct {
    int32_t n_vertices, n_edges;
    int32_t max_dep;                   /* M = max |D(i)| */
    int32_t max_configs;               /* K = max |C(v)| */
    int32_t tree_levels;               /* elimination-tree depth */
    int32_t n_launches;                /* kernels launched per pase_solve */
    uint64_t candidates;               /* sum_i K(sigma_i) * |T(i)|  ("combinations") */
    uint64_t table_entries;            /* sum_i |T(i)| */
    uint64_t cost_entries;             /* sum_v K_v + sum_e K_u K_v */
    uint64_t alg_bytes_dp;             /* algorithmic HBM bytes of the DP fill */
    uint64_t alg_bytes_tables;         /* bytes written by the cost-table kernel */
    uint64_t comm_bytes;               /* multi-GPU all-gather bytes per solve (this rank) */
    double ms_create;                  /* host: ingest..plan..alloc (excl. NCCL init) */
    double ms_nccl_init;
    double ms_solve;                   /* device time of the last pase_solve (CUDA events) */
    double ms_tables, ms_dp;           /* phase split of the last pase_solve (CUDA events in the graph) */
    uint64_t dp_fp64_ops;              /* sum_i N_i * (terms_i - 1 adds + 1 compare) of the DP fill */
    uint64_t h2d_bytes;                /* bytes copied host->device by pase_create */
    uint64_t d2h_bytes;                /* bytes copied device->host per pase_solve */
} pase_stats;

typedef struct pase_ctx pase_ctx;

/* a1-a4 + allocation: validates and deep-copies g (caller may free it on return), enumerates
 * C(v), runs SortNodes, builds the elimination tree, plans table layouts, applies the size
 * guard, allocates device memory on m->cuda_device and records the solve schedule as a
 * CUDA graph.  p >= 1 is the simulated device count.  *out is NULL on failure. */
pase_status pase_create(const pase_graph* g, int32_t p, const pase_machine* m, pase_ctx** out);

/* a5-a8: runs the whole search on the GPU (cost tables, DP fill over the elimination tree,
 * back-substitution).  Scheduler and group-barrier waits are bounded by PASE_SPIN_TIMEOUT_MS
 * (environment at pase_create, default 4000, 0 = unbounded): a wait past it fails the solve
 * with PASE_ERR_STATE instead of hanging; a DP entry with no finite candidate (fp64 overflow
 * of a sum) fails it with PASE_ERR_RESOURCE.  configs_out: caller-allocated int32[n_nodes * PASE_MAX_DIMS], row v =
 * the split tuple of node v (unused dims = 1); may be NULL.  config_index_out: int32[n_nodes]
 * index of phi*(v) in C(v) (lexicographic order); may be NULL.  total_cost_out: f(|V|, ∅).
 * May be called repeatedly; every call recomputes everything. */
pase_status pase_solve(pase_ctx* ctx, int32_t* configs_out, int32_t* config_index_out,
                       double* total_cost_out);

pase_status pase_get_stats(const pase_ctx* ctx, pase_stats* out);
const char* pase_last_error(const pase_ctx* ctx);
void pase_destroy(pase_ctx* ctx);   /* NULL-safe; frees device memory, graph, comm */

/* ---- introspection / test hooks (host pointers, caller-allocated) -------------------- */

/* counts[n_nodes] = |C(v)|; tuples (may be NULL) = per node in id order, counts[v] rows of
 * PASE_MAX_DIMS int32 (unused dims = 1), lexicographic (dim 0 most significant). */
pase_status pase_get_configs(const pase_ctx* ctx, int32_t* counts, int32_t* tuples);

/* sigma[n] (rank -> node), dep_off[n+1] / dep_ids[<= n*PASE_MAX_DEP] = D(i) ascending rank,
 * parent[n] = rank of min-rank D(i) (-1 for the root).  Any pointer may be NULL. */
pase_status pase_get_order(const pase_ctx* ctx, int32_t* sigma, int32_t* dep_off,
                           int32_t* dep_ids, int32_t* parent);

/* Cost tables of the last pase_solve, in the ORACLE layout: is_edge = 0: L_v[K_v];
 * is_edge = 1: W_e[c_src * K_dst + c_dst] (already multiplied by r). */
pase_status pase_get_cost_tables(const pase_ctx* ctx, int32_t index, int32_t is_edge, double* out);

/* T(i) and A(i) of rank i after pase_solve (|T(i)| entries; coordinates D(i) ascending rank,
 * lowest rank fastest).  On a connected multi-GPU context the other ranks' slices of a
 * partitioned T(i) are gathered from their pools through the peer mappings (A(i) is complete
 * on every rank).  PASE_ERR_STATE between pase_launch and pase_finish. */
pase_status pase_get_dp_table(const pase_ctx* ctx, int32_t rank, double* T_out, uint16_t* A_out);
int64_t pase_table_entries(const pase_ctx* ctx, int32_t rank);

/* Replace the cost model by explicit tables (synthetic-cost tests): L concatenated
 * over nodes in id order (K_v each), W over edges in id order (K_src*K_dst each, src-major).
 * Subsequent pase_solve calls use these tables instead of running the cost-table kernel.
 * Every value must be finite (PASE_ERR_INVALID names the first that is not); PASE_ERR_STATE
 * between pase_launch and pase_finish.  The copy is ordered on the context's stream and
 * complete when the call returns. */
pase_status pase_set_cost_tables(pase_ctx* ctx, const double* L, const double* W);

/* Persistent-schedule timeline (tracing; enabled by env PASE_TRACE=1 at pase_create): per DP
 * task of the last pase_solve, 22 int64 = {(smid << 32) | rank, t_claim_ns, t_start_ns (descriptors
 * staged; dependencies met unless the early gate is on), t_computed_ns (warp 0 done), t_synced_ns
 * (CTA done), t_end_ns (parent counter released)}, then per warp w = 0..7 {t_gate_seen_ns (the
 * children's counter seen at zero), t_gate_fenced_ns (acquire fence done)} (0: the warp had no
 * gate in this task) (%globaltimer).  Copies min(cap, n_tasks) records into out (may be NULL); returns n_tasks
 * (0 when tracing is off, -1 on a CUDA error). */
int64_t pase_get_trace(const pase_ctx* ctx, int64_t* out, int64_t cap);

/* Time the solve phases separately on the next pase_solve (adds syncs; default off). */
pase_status pase_set_profiling(pase_ctx* ctx, int32_t enable);

/* ---- Eq. 1 on the GPU (eval.cu) -------------------------------------------
 * Both use the context's cost tables: the cost-table kernel's L_v / W_e (recomputed by the
 * call on the context's stream), or the tables given to pase_set_cost_tables.  The sum is Eq. 1
 * written out in one fixed order: 0 + L_v[phi(v)] over node ids, then + W_e over
 * edge ids, each an IEEE round-to-nearest add.  Synchronous (return after the device work).
 * Multi-GPU contexts evaluate on their own device only (no group call). */

/* cost(G, phi) for n_strategies strategies: config_index = int32[n_strategies * n_nodes]
 * (row s = strategy s, entry v = index of phi(v) in C(v)); cost_out = double[n_strategies].
 * PASE_ERR_INVALID names the first index outside [0, K_v). */
pase_status pase_evaluate(pase_ctx* ctx, const int32_t* config_index, int64_t n_strategies, double* cost_out);

/* Exhaustive search: the minimum of Eq. 1 over all prod_v K_v strategies, which
 * Theorem 1 says equals pase_solve's total.  Strategy index = mixed radix over
 * node ids, node 0 fastest; among equal costs the lowest index wins.  max_strategies = 0
 * means 2^40; a larger space returns PASE_ERR_RESOURCE.  Outputs (each may be NULL):
 * config_index_out = int32[n_nodes], total_cost_out, n_strategies_out = prod_v K_v. */
pase_status pase_brute_force(pase_ctx* ctx, uint64_t max_strategies, int32_t* config_index_out,
                             double* total_cost_out, uint64_t* n_strategies_out);

/* ---- device assignment (assign.cpp) --------------------------------------
 * A strategy fixes how each vertex is split, not which device runs which part; PaSE places the
 * parts with "a simple greedy assignment that maximizes data locality".  Reading U
 * (DESIGN §2): shard s of v = the digits of s in the radix of v's split tuple (dim 0 most
 * significant); vertices in node-id order, shards in index order, each on the free device with
 * the largest summed overlap (elements) between what consumer shards need of a producer's
 * output and what the producer shard on that device holds, over edges to placed neighbours;
 * ties -> lowest device id.  Host-side integer work; also valid on host-only contexts.
 *   config_index: int32[n_nodes], index of phi(v) in C(v) (e.g. pase_solve's output).
 *   device_out:   int32[n_nodes * p] (may be NULL): row v = device of each shard, -1 past the
 *                 shard count prod c(v).
 *   tx_out:       double[n_edges] (may be NULL): realized t_x bytes of each edge under the
 *                 assignment, 2 elem max_d (|needed on d| - |needed on d ∩ held on d|)
 *                 (P:271-276); never below the cost model's aligned t_x (reading K).
 * PASE_ERR_INVALID names the first config index outside [0, K_v). */
pase_status pase_assign_devices(const pase_ctx* ctx, const int32_t* config_index, int32_t* device_out,
                                double* tx_out);

/* ---- split solve (a multi-GPU group launches every rank before waiting on any) ---------- */
pase_status pase_launch(pase_ctx* ctx);       /* enqueue one solve on the context's stream */
pase_status pase_finish(pase_ctx* ctx, int32_t* configs_out, int32_t* config_index_out,
                        double* total_cost_out);   /* wait for it; outputs as pase_solve */

/* ---- multi-GPU group (world > 1) -------------------------------------
 * Every rank creates its context with the same graph, p and machine (except rank /
 * cuda_device), exports a handle, the caller exchanges the world handles (e.g. an all-gather
 * over torch.distributed) and passes them, ordered by rank, to pase_connect.  Big DP tables
 * are partitioned by their highest-rank coordinate; the DP kernel writes the partitions other
 * ranks need directly into their tables over NVLink (CUDA IPC peer memory) and signals them
 * with system-scope atomics: no separate collective.  Contexts of one process on one device
 * (virtual_ranks = 1) exercise the same path on a single GPU.  pase_solve on a group context
 * must be called by every rank (the solve contains two group barriers). */
pase_status pase_export_handle(const pase_ctx* ctx, void* blob /* PASE_HANDLE_BYTES */);
pase_status pase_connect(pase_ctx* ctx, const void* blobs /* world * PASE_HANDLE_BYTES */);

/* Schedule introspection (also on host-only contexts): per DP rank i, vinfo[8i..8i+7] =
 * {partitioned, broadcast flags, this rank's task count, initial pending counter, kernel
 * shape (-1 generic, 0..63 1-D tile, >= 64 2-D tile), log2 lanes per item group, log2 warps
 * per item (latency mode), second tiled coordinate (-1 none)}; tasks =
 * this rank's {rank i, first item, end item, kind} quadruples (kind 0: the items [first, end)
 * with the vertex's lane groups; > 0: with lane groups widened to 2^kind lanes (wave tail));
 * order = claim order.  Returns the task count (arrays may be NULL). */
int64_t pase_get_schedule(const pase_ctx* ctx, int32_t* vinfo, int64_t* tasks, int32_t* order);

#ifdef __cplusplus
}
#endif
#endif /* PASE_H */
