// pase_internal.h -- internal types shared by the host core (host.cpp), the C ABI
// (capi.cu) and the sm_100a kernels (kernels.cu).  Not installed; include/pase.h is
// the public boundary.  Citations: P:<n> = PAPER.md line n.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "pase.h"

namespace pase {

constexpr int kMaxDims = PASE_MAX_DIMS;
constexpr int kMaxDep = PASE_MAX_DEP;

// ---------------------------------------------------------------------------------
// Host plan (a1-a4): everything pase_create derives from the graph, before the GPU.
// ---------------------------------------------------------------------------------
struct Plan {
    int n = 0, m = 0, p = 1, policy = 0;
    double r = 0.0;                              // F / B
    std::vector<pase_node> nodes;
    std::vector<pase_edge> edges;

    // a2: C(v) -- per node K_v and its tuples (row-major, kMaxDims int32 per config)
    std::vector<int32_t> K;
    std::vector<int64_t> cfg_off;                // n+1, in configs: start of C(v) in cfg (nodes of one
                                                 // iteration space share a block); [n] = rows in cfg
    std::vector<int32_t> cfg;                    // cfg_off[n] * kMaxDims (distinct spaces only)

    // a3: SortNodes (Fig. 4): sigma (rank -> node), rank (node -> rank), D(i) by rank
    std::vector<int32_t> sigma, rank;
    std::vector<std::vector<int32_t>> dep;       // D(i) node ids, ascending rank

    // a4: elimination tree over ranks, E>(sigma_i), levels
    std::vector<int32_t> parent;                 // rank of min-rank D(i), -1 for root
    std::vector<std::vector<int32_t>> children;  // ranks, ascending
    std::vector<std::vector<int32_t>> egt;       // edge ids, by (rank(other end), edge id)
    std::vector<int32_t> level;                  // 0 = leaves
    int levels = 0;

    // layout: per rank |T(i)|, offsets into the T / A pools (entries)
    std::vector<int64_t> tsize, toff;
    std::vector<int64_t> loff;                   // n+1: L_v offset (doubles)
    std::vector<int64_t> woff;                   // m+1: W_e offset (doubles)
    int max_dep = 0, max_k = 0;
    uint64_t candidates = 0, entries = 0;
};

// x / d for 0 <= x < 2^31 as (x * mul) >> sh, 1 <= d < 2^31 (round-up method: with
// 2^(s-1) < d <= 2^s, mul = ceil(2^(31+s) / d) < 2^32 and the error term stays below 2^(31+s))
inline void fastdiv_magic(uint32_t d, uint32_t& mul, int32_t& sh) {
    int s = 0;
    while ((1ull << s) < d) ++s;
    const unsigned __int128 num = (unsigned __int128)1 << (31 + s);
    mul = (uint32_t)((num + d - 1) / d);
    sh = 31 + s;
}

// Builds a Plan.  Returns PASE_OK or an error with a message.
pase_status build_plan(const pase_graph* g, int32_t p, const pase_machine* m, Plan& plan,
                       std::string& err);

// ---------------------------------------------------------------------------------
// Device descriptors (kernels.cu)
// ---------------------------------------------------------------------------------
struct EdgeDesc {            // cost-table kernel: one per edge
    int32_t src, dst;
    int32_t later_is_src;    // W row = config of the later-ranked endpoint
    int32_t pad;
    int32_t axis_map[kMaxDims];
    int64_t woff;            // doubles
};

struct CostChunk {           // cost-table work unit (one CTA)
    int32_t item;            // < n: vertex (all of L_v); >= n: edge item - n
    int32_t row0, nrows;     // edge: rows [row0, row0 + nrows) of W_e (later-endpoint configs)
    int32_t node;            // the vertex, or the edge's src (staged with the edge descriptor)
    int32_t consumer;        // rank of the DP vertex that reads it (persistent schedule)
};

struct TermDesc {            // one summand of Eq. 4 for a vertex (L, one W_e, or one child T_j)
    const double* base;      // element(phi, C) = base[sum_q c_q * stride[q] + C]
    int64_t stride[kMaxDep];
};

constexpr int kMaxWorld = 8;     // search GPUs per context group (1, 2, 4, 8)

struct VertexDesc {          // one DP vertex (rank i)
    int32_t K;               // |C(sigma_i)|, the reduction extent
    int32_t m;               // |D(i)|
    int32_t nterms;          // 1 + |E>(sigma_i)| + |children(i)|, canonical order
    int32_t term0;           // first TermDesc
    int64_t nout;            // |T(i)|
    int32_t radix[kMaxDep];  // K of each D(i) coordinate, ascending rank (lowest fastest)
    double* T;               // output table
    uint16_t* A;             // argmin table
    // tiled schedule: outputs are tiled along coordinate qstar; terms
    // [0, tstar) do not depend on qstar and are summed once per C per tile (hoisted prefix).
    int32_t qstar;           // tiled coordinate (-1: root, D(i) = ∅)
    int32_t tstar;           // first term depending on qstar
    int32_t rq;              // radix of qstar (1 for the root)
    int32_t ntile;           // tiles along qstar = ceil(rq / kTile)
    int64_t ostride_q;       // output stride of qstar
    int64_t ncombo;          // nout / rq
    int64_t nitems;          // ncombo * ntile
    // 2-D register tile (shape >= kShape2D): a kTile1 x kTile2 block of outputs
    // along (qstar, q2).  Terms [0, t2star) depend on neither (scalar prefix), [t2star, tstar)
    // on q2 at most, [tstar, nterms) on qstar and maybe q2.  ntile = ntile1 * ntile2 and
    // ncombo = nout / (rq * rq2) then; item = combo + ncombo * (t2 + ntile2 * t1).
    int32_t q2;              // second tiled coordinate (-1: 1-D tiling)
    int32_t rq2;             // its radix
    int32_t ntile2;          // tiles along q2
    int32_t t2star;          // first term depending on q2
    int64_t ostride_q2;      // output stride of q2
    int32_t glog;            // log2 lane-group size
    int32_t wlog;            // log2 warps per item (latency mode, glog == 5 only)
    int32_t shape;           // tiled variant (NP-1)*16 + NS*4 + (glog-2), or -1 = generic kernel
    int32_t ntasks;          // persistent schedule: this rank's tasks of the vertex ...
    int32_t task0;           // ... with local ids [task0, task0 + ntasks)
    int32_t parent;          // rank of the elimination-tree parent (-1: root)
    // division by invariant integers (decode of work items): x / d == (x * mul) >> sh for
    // x < 2^31 (magic numbers from fastdiv_magic on the host), per coordinate radix and for
    // ncombo, ntile, ntile2, psub
    uint32_t rmul[kMaxDep];
    int32_t rsh[kMaxDep];
    uint32_t mul_combo, mul_tile, mul_tile2, mul_psub;
    int32_t sh_combo, sh_tile, sh_tile2, sh_psub;
    int32_t part;            // multi-GPU: table partitioned by its top coordinate
    int32_t psub;            // partitioned: combinations below the top coordinate (ncombo / K_top)
    int32_t bcast;           // bit 0: write T to every rank, bit 1: write A to every rank
    int32_t pf_ahead;        // stream L2-prefetch form: items of lookahead (0 = the current item)
    int32_t cb1, cb2;        // CTA-tiled shape: block of (qstar, q2) values per CTA item (multiples of 4)
    int32_t npeer;           // peers written when bcast != 0 (world - 1)
    double* Tpeer[kMaxWorld - 1];     // this vertex's T / A in the peers' pools
    uint16_t* Apeer[kMaxWorld - 1];
};
constexpr int kSchedLine = 32;   // int32 words per 128-B line (scheduler control block)
constexpr int kMaxTermsSh = 8;   // terms staged in shared memory (tiled shapes use <= 7)

struct TaskDesc {            // persistent schedule: item range [i0, i1) of vertex vtx
    int32_t vtx;
    int32_t glog;            // 0: the vertex's lane groups; > 0: log2 lanes per item (wave tail)
    int64_t i0, i1;
};

struct Peers {               // kernel parameter: the group's scheduler words (device pointers)
    int32_t* pending[kMaxWorld];   // each rank's pending[n] (index = this context's rank order)
    int32_t* bar[kMaxWorld];       // each rank's barrier counter
    int32_t world, rank;
};

constexpr int kTraceTaskWords = 6;            // PASE_TRACE record per task (pase_get_trace) ...
constexpr int kTraceWords = kTraceTaskWords + 2 * 8;   // ... + per warp {gate seen, gate fenced}
constexpr int kTasksPerBlock = 4;   // big vertices: ~4 tasks per CTA of the grid

struct SchedPlan {           // build_schedule output for one rank
    std::vector<TaskDesc> tasks;   // this rank's tasks, vertex-major (VertexDesc.task0)
    std::vector<int32_t> order;    // claim order (indices into tasks)
    std::vector<int32_t> pending;  // initial pending counter per vertex
    std::vector<int32_t> ready0;   // ready-queue mode: tasks ready at the start (no children), in order
    int64_t total_tasks = 0;       // over all ranks
};

// schedule.cpp: tasks, broadcast flags, pending counters and claim order (needs VertexDesc
// shape / tiling / part fields filled in).
// chunk_consumer (optional): per cost-table chunk the rank of the DP vertex reading it; the
// chunks then become tasks of the persistent schedule (vtx = -1 - chunk) that the consumer's
// tasks wait for.
pase_status build_schedule(const Plan& P, std::vector<VertexDesc>& vd, int world, int rank, int nblocks,
                           SchedPlan& out, std::string& err,
                           const std::vector<int32_t>* chunk_consumer = nullptr, bool simulate = true);
constexpr int kTile = 8;     // max outputs per lane group along qstar
constexpr int kTile1 = 4, kTile2 = 4;   // 2-D tile: outputs along qstar x q2
constexpr int kShape2D = 64;            // shapes >= kShape2D: 2-D tiled (NS-1)*4 + (glog-2)
constexpr int kShape2S = 96;            // shapes >= kShape2S: 2-D single-suffix ((NP0-1)*4 + form)*4 + (glog-2)
constexpr int kShapeG1 = 160;           // shapes >= kShapeG1: 1-D tile, one lane per item (K <= 3): (NP-1)*4 + NS
constexpr int kShapeStream = 192;       // [192, 224): 1-D tile, G = 32, last term TMA-staged in smem: (NP-1)*4 + NS
constexpr int kShapeStreamPF = 224;     // [224, 256): 1-D tile, G = 32, next item's last-term rows TMA-prefetched to L2
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool stream_smem_shape(int s) { return s >= kShapeStream && s < kShapeStreamPF; }
// [256, 268): CTA-tiled min-plus, the single-suffix structure of kShape2S:
// (NP0 - 1) * 4 + form; one CTA item = one combination x a cb1 x cb2 block of (qstar, q2)
constexpr int kShapeCta = 256;
constexpr int kCtaCC = 8;               // values of C per thread group per staged round
constexpr int kCtaG = 4;                // thread groups of 64 per CTA (each reduces its own C run)
constexpr size_t kCtaSmemMax = 69632;   // dynamic shared memory the persistent kernel gets
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr bool cta_shape(int s) { return s >= kShapeCta && s < kShapeCta + 12; }
// list-schedule task-duration families (schedule.cpp dur_model)
enum { kDurGeneric, kDurLatency, kDur1D, kDur2D, kDur2S, kDurG1, kDurStream, kDurCta, kDurFamilies };
struct DurModel { double a[kDurFamilies], rate[kDurFamilies]; };
int dur_family(const VertexDesc& d);
const DurModel& dur_model();
//   form 0: P1 = [A], S = [S1]; 1: P1 = [A, B], S = [S1]; 2: S = [S1, const]; 3: S = [S1, S2 on q1]
constexpr int kMaxP0 = 4, kMaxP1 = 2;   // 2-D tile: max scalar-prefix / q2-prefix terms
#ifndef PASE_COST_ROWS
#define PASE_COST_ROWS 64
#endif
constexpr int kCostRows = PASE_COST_ROWS;  // edge-table rows per cost-table CTA
constexpr int kCostCols = 512; // edge-table columns staged per pass

struct CostArgs {            // the cost-table computation (kernel parameter)
    const pase_node* nodes;
    const int32_t* K;
    const int64_t* cfg_off;
    const int32_t* cfg;
    const int64_t* loff;
    int32_t n, enabled;      // enabled = 0: tables were given by pase_set_cost_tables
    const EdgeDesc* edges;
    const CostChunk* chunks;
    double r;
    double* L;
    double* W;
    // stand-alone kernel only (nullptr otherwise): CTA 0 also zeroes *err and copies the
    // scheduler's initial state sched_init -> sched (sched_words int32) for the DP that follows
    int32_t* err;
    int32_t* sched;
    const int32_t* sched_init;
    int32_t sched_words;
};

struct CostSmem {            // its shared memory ([axis][config]: conflict-free over configs)
    uint32_t rowq[kMaxDims][kCostRows];
    uint32_t colq[kMaxDims][kCostCols];
    uint64_t rowprod[kCostRows];
    uint64_t colprod[kCostCols];
    pase_node su;            // the vertex / the edge's producer
    EdgeDesc se;
};

struct BtDesc {               // back-substitution record of one rank, in back-level order
    const uint16_t* A;       // argmin table A(i)
    int32_t node;            // sigma_i
    int32_t K;               // |C(sigma_i)|: a stored argmin >= K means no finite candidate
    int32_t dep[kMaxDep];    // D(i) node ids (padding: node 0) ...
    int64_t stride[kMaxDep]; // ... and their A(i) index strides (padding: 0)
};

struct EvalEdge {             // Eq. 1 kernels (eval.cu): W_e element = W[off + c_row * kcol + c_col]
    int32_t row, col;        // node ids: later- / earlier-ranked endpoint (the DP layout of W_e)
    int32_t kcol, pad;       // K of the column node
    int64_t off;             // W_e offset (doubles)
};
constexpr int kBruteThreads = 128;

// kernels.cu entry points (host-side launchers)
void launch_cost_tables(const CostArgs& A, int nchunks, void* stream);
void launch_dp_vertex(const VertexDesc* vd_dev, const TermDesc* td_dev, int vertex,
                      const VertexDesc& vd_host, void* stream);
void launch_dp_persistent(const VertexDesc* vd_dev, const TermDesc* td_dev, const TaskDesc* tasks_dev,
                          const int32_t* order_dev, int ntasks, int32_t* sched_dev, int32_t* err_dev,
                          const Peers& peers, const CostArgs& cost, int nblocks, int64_t* trace_dev,
                          uint64_t timeout_ns, bool stream_tiles, int32_t* ring, int32_t* ring_tail,
                          int early_gate, void* stream);
void launch_rank_barrier(const Peers& peers, int32_t* bar_dev, int32_t* err_dev, uint64_t timeout_ns, void* stream);
int persistent_blocks_per_sm();
void launch_backtrack(const BtDesc* bt_dev, const int32_t* bt_off_dev, int ngroups, int n,
                      const double* root_T, int32_t* choice_dev, double* total_dev, int32_t* err_dev,
                      void* host_out, void* stream);

// assign.cpp (row f3): greedy device assignment of a strategy (DESIGN reading U)
pase_status assign_devices(const Plan& P, const int32_t* config_index, int32_t* device_out, double* tx_out,
                           std::string& err);

// eval.cu (row f2): Eq. 1 for given strategies; exhaustive minimum over all strategies
void launch_eval(int n, int m, const int64_t* loff_dev, const double* L_dev, const EvalEdge* ed_dev,
                 const double* W_dev, const int32_t* strat_dev, int64_t ns, double* out_dev, void* stream);
size_t brute_smem_bytes(int n, int m);
int launch_brute(int n, int m, const int32_t* K_dev, const int64_t* loff_dev, const double* L_dev,
                 const EvalEdge* ed_dev, const double* W_dev, uint64_t total, int nblocks,
                 double* blk_b, uint64_t* blk_i, double* out_b, uint64_t* out_i, void* stream);

}  // namespace pase
