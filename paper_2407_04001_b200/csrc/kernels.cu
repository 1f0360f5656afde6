// kernels.cu -- sm_100a kernels of the PaSE hot path.
//   K1 cost_tables   (row a5): L_v[C] = t_l(v, C, r), W_e = r * t_x (Eq. 1)
//   K2 dp_persistent (row a6): Eq. 4 / Fig. 5 lines 8-20 over the whole
//                    elimination tree in one launch (tile families: DESIGN §5.2; schedule: §5.3);
//                    dp_fill_vertex runs one vertex per launch (PASE_SCHEDULE=launches)
//   K3 backtrack     (row a7): back-substitution from sigma_|V|.cfg
// Bit-exactness rules: every fp64 op is an explicit IEEE RN intrinsic
// (__dadd_rn / __dmul_rn / __ddiv_rn / __ull2double_rn), never contracted to FMA; the sum
// over the terms of Eq. 4 follows the canonical order L, W_e (E> order), T_j (rank order);
// ties in the min over C keep the lowest C (strict <, Fig. 5 line 17).
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "pase_internal.h"

#ifndef PASE_CUNROLL
#define PASE_CUNROLL 2   // C iterations in flight per lane in the 1-D tile loop
#endif
constexpr int kCUnroll = PASE_CUNROLL;
// persistent-scheduler synchronisation variants (A/B builds; defaults = measured best,
// profiles/r01_ab_scheduling.txt: the fence + spin pair is 2-9 % faster on every workload)
#ifndef PASE_SPIN_SLEEP
#define PASE_SPIN_SLEEP 0      // back off with __nanosleep while polling a pending counter
#endif
#ifndef PASE_ACQ_FENCE
#define PASE_ACQ_FENCE 1       // acquire via fence.acq_rel after the relaxed poll (else ld.acquire)
#endif
#ifndef PASE_GATE_LDACQ
#define PASE_GATE_LDACQ 0      // per-warp gate: acquire via ld.acquire of the counter instead of a fence
#endif
#ifndef PASE_LAYOUT_PAD
#define PASE_LAYOUT_PAD 0      // dead-code pad in dp_persistent (code placement A/B)
#endif
#ifndef PASE_REL_RED
#define PASE_REL_RED 0         // release via red.release (no return) instead of atom.acq_rel
#endif

namespace pase {

// =====================================================================================
// K1: cost tables
// =====================================================================================
__device__ __forceinline__ double d_allreduce(int64_t g, int64_t bytes) {
    // ring all-reduce over g participants: 2(g-1)B/g (DESIGN reading J)
    if (g <= 1) return 0.0;
    return __ddiv_rn(__ull2double_rn((unsigned long long)(2 * (g - 1) * bytes)), __ll2double_rn(g));
}

// t_l (DESIGN reading I): FLOPs of one (equal) shard + r * (reduction AR + gradient AR + halo).
// The node lives in shared memory; every per-dim array is indexed by compile-time k (fully
// unrolled over kMaxDims, so they stay in registers) and the axis lists become dim masks
// (axes are distinct, so the products are the same integers in any order).
__device__ double d_layer_cost(const pase_node& x, const int32_t* __restrict__ c, double r) {
    int32_t cc[kMaxDims];
    {
        const int4 lo = *reinterpret_cast<const int4*>(c), hi = *reinterpret_cast<const int4*>(c + 4);
        cc[0] = lo.x; cc[1] = lo.y; cc[2] = lo.z; cc[3] = lo.w; cc[4] = hi.x; cc[5] = hi.y; cc[6] = hi.z; cc[7] = hi.w;
    }
    const int nd = x.n_dims;
    uint32_t out_m = 0, w_m = 0;
    for (int a = 0; a < x.n_out_axes; ++a) out_m |= 1u << x.out_axes[a];
    for (int a = 0; a < x.n_w_axes; ++a) w_m |= 1u << x.w_axes[a];
    const uint32_t fl_m = x.flop_dims_mask == 0u ? 0xffu : x.flop_dims_mask;
    int64_t s[kMaxDims];                       // sizes < 2^31 (validated): 32-bit divisions
    int64_t compute = x.flops_per_point, out_elems = 1, w_elems = 1, g_red = 1, g_grad = 1;
#pragma unroll
    for (int k = 0; k < kMaxDims; ++k) {
        const bool in = k < nd;
        s[k] = in ? (int64_t)((uint32_t)x.size[k] / (uint32_t)cc[k]) : 1;
        if (in && (fl_m >> k & 1u)) compute *= s[k];
        if (out_m >> k & 1u) out_elems *= s[k];
        if (w_m >> k & 1u) w_elems *= s[k];
        if (in && !(out_m >> k & 1u)) g_red *= cc[k];
        if (in && !(w_m >> k & 1u)) g_grad *= cc[k];
    }
    const int64_t out_bytes = (int64_t)x.elem_bytes * out_elems;
    const int64_t w_bytes = x.n_w_axes > 0 ? (int64_t)x.elem_bytes * w_elems : 0;
    if (x.n_w_axes == 0) g_grad = 1;
    // conv halo (DESIGN reading L): (size_f - 1) input rows of the face of the INPUT-tensor
    // shard across h, i.e. the input axes other than h
    uint32_t in_m = 0;
    for (int a = 0; a < x.n_in_axes; ++a) in_m |= 1u << x.in_axes[a];
    int64_t halo = 0;
    for (int q = 0; q < x.n_halo; ++q) {
        const int h = x.halo_spatial[q], f = x.halo_filter[q];
        int32_t ch = 1;
        int64_t face = 1;
#pragma unroll
        for (int k = 0; k < kMaxDims; ++k) {
            if (k == h) ch = cc[k];
            if ((in_m >> k & 1u) && k != h) face *= s[k];
        }
        if (ch > 1 && x.size[f] > 1) halo += 2 * (int64_t)x.elem_bytes * (x.size[f] - 1) * face;
    }
    double comm = d_allreduce(g_red, out_bytes);
    comm = __dadd_rn(comm, d_allreduce(g_grad, w_bytes));
    comm = __dadd_rn(comm, __ull2double_rn((unsigned long long)halo));
    return __dadd_rn(__ull2double_rn((unsigned long long)compute), __dmul_rn(r, comm));
}

// cooperative copy of a small struct into shared memory (4-byte words)
template <typename T>
__device__ __forceinline__ void stage_struct(T* dst, const T* src) {
    static_assert(sizeof(T) % 4 == 0, "word copy");
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    for (int w = threadIdx.x; w < (int)(sizeof(T) / 4); w += blockDim.x) d[w] = s[w];
}

// One CTA per chunk: a vertex (all K_v entries of L_v) or up to kCostRows rows of one
// edge table W_e[row = later endpoint config][col = earlier endpoint config].  Per-config,
// per-axis shard extents (and prod need) are precomputed in shared memory, so the inner
// loop is a min / multiply per axis, and stores are coalesced along the column.  Runs as its
// own kernel (per-vertex launch schedule) or as tasks of the persistent DP kernel.
// (force-inlined into both callers: the compiler then knows `sm` is shared memory -- LDS, not
// generic loads -- and keeps the loop invariants of A in registers / the constant bank)
__device__ __forceinline__ void cost_chunk(const CostArgs& A, int chunk, CostSmem& sm) {
    const CostChunk ch = A.chunks[chunk];
    // chunk.node = the vertex, or the edge's src: both structs are staged in one round of loads
    stage_struct(&sm.su, A.nodes + ch.node);
    if (ch.item >= A.n) stage_struct(&sm.se, A.edges + (ch.item - A.n));
    __syncthreads();
    if (ch.item < A.n) {
        const int v = ch.item;
        const int Kv = A.K[v];
        const int32_t* cv = A.cfg + A.cfg_off[v] * kMaxDims;
        double* Lv = A.L + A.loff[v];
        for (int c = threadIdx.x; c < Kv; c += blockDim.x) Lv[c] = d_layer_cost(sm.su, cv + c * kMaxDims, A.r);
        __syncthreads();                                    // sm reused by the caller's next chunk
        return;
    }
    const EdgeDesc& e = sm.se;
    const pase_node& u = sm.su;
    const int nax = u.n_out_axes;
    const int early = e.later_is_src ? e.dst : e.src;
    const int Ke = A.K[early];
    const uint64_t elem2 = 2ull * (uint64_t)u.elem_bytes;
    // t_x (DESIGN reading K): per output axis a of src, held_a = ext / c_src, need_a =
    // ceil(ext / c_dst[map_a]) (ext if unmapped); t_x = 2 elem (prod need - prod min(need, held))
    // (sizes < 2^31, validated on the host: 32-bit divisions)
    const int32_t* cfg_s = A.cfg + A.cfg_off[e.src] * kMaxDims;
    const int32_t* cfg_d = A.cfg + A.cfg_off[e.dst] * kMaxDims;
    auto held = [&](int cs, int a) -> uint32_t {
        const int32_t* c = cfg_s + cs * kMaxDims;
        return (uint32_t)u.size[u.out_axes[a]] / (uint32_t)c[u.out_axes[a]];
    };
    auto need = [&](int cd, int a) -> uint32_t {
        const int32_t* c = cfg_d + cd * kMaxDims;
        const uint32_t ext = (uint32_t)u.size[u.out_axes[a]];
        return e.axis_map[a] < 0 ? ext : (ext + (uint32_t)c[e.axis_map[a]] - 1u) / (uint32_t)c[e.axis_map[a]];
    };
    // rows = later endpoint: src configs (held) if later_is_src, else dst configs (need)
    for (int rr = threadIdx.x; rr < ch.nrows; rr += blockDim.x) {
        uint64_t pr = 1;
        for (int a = 0; a < nax; ++a) {
            const uint32_t x = e.later_is_src ? held(ch.row0 + rr, a) : need(ch.row0 + rr, a);
            sm.rowq[a][rr] = x;
            pr *= x;
        }
        sm.rowprod[rr] = pr;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool lis = e.later_is_src != 0;
    const double r = A.r;
    double* const W = A.W + e.woff;
    for (int c0 = 0; c0 < Ke; c0 += kCostCols) {
        const int nc = min(kCostCols, Ke - c0);
        __syncthreads();
        for (int cc = threadIdx.x; cc < nc; cc += blockDim.x) {
            uint64_t pr = 1;
            for (int a = 0; a < nax; ++a) {
                const uint32_t x = lis ? need(c0 + cc, a) : held(c0 + cc, a);
                sm.colq[a][cc] = x;
                pr *= x;
            }
            sm.colprod[cc] = pr;
        }
        __syncthreads();
        // rows: one warp each, columns over its lanes (coalesced stores); the axis loop is
        // specialised on the axis count (registers, no per-axis branch)
        auto rows = [&](auto nax_c) {
            constexpr int NAX = decltype(nax_c)::value;
            for (int rr = warp; rr < ch.nrows; rr += nw) {
                uint32_t rq[NAX > 0 ? NAX : 1];         // this row's extents: registers
#pragma unroll
                for (int a = 0; a < NAX; ++a) rq[a] = sm.rowq[a][rr];
                const uint64_t rp = sm.rowprod[rr];
                double* out = W + (int64_t)(ch.row0 + rr) * Ke + c0;
                for (int cc = lane; cc < nc; cc += 32) {
                    uint64_t ov = 1;
#pragma unroll
                    for (int a = 0; a < NAX; ++a) ov *= (uint64_t)min(rq[a], sm.colq[a][cc]);
                    const uint64_t nd = lis ? sm.colprod[cc] : rp;
                    out[cc] = __dmul_rn(r, __ull2double_rn((unsigned long long)(elem2 * (nd - ov))));
                }
            }
        };
        switch (nax) {
            case 0: rows(std::integral_constant<int, 0>{}); break;
            case 1: rows(std::integral_constant<int, 1>{}); break;
            case 2: rows(std::integral_constant<int, 2>{}); break;
            case 3: rows(std::integral_constant<int, 3>{}); break;
            case 4: rows(std::integral_constant<int, 4>{}); break;
            case 5: rows(std::integral_constant<int, 5>{}); break;
            case 6: rows(std::integral_constant<int, 6>{}); break;
            case 7: rows(std::integral_constant<int, 7>{}); break;
            default: rows(std::integral_constant<int, kMaxDims>{}); break;
        }
    }
    __syncthreads();                                        // sm reused by the caller's next chunk
}

__global__ void __launch_bounds__(256, 4) cost_tables_kernel(CostArgs A) {
    __shared__ CostSmem sm;
    if (blockIdx.x == 0) {                                  // per-solve resets (see CostArgs)
        if (A.err && threadIdx.x == 0) *A.err = 0;
        if (A.sched)
            for (int k = threadIdx.x; k < A.sched_words; k += blockDim.x) A.sched[k] = A.sched_init[k];
    }
    cost_chunk(A, blockIdx.x, sm);
}

void launch_cost_tables(const CostArgs& A, int nchunks, void* stream) {
    cost_tables_kernel<<<(unsigned)nchunks, 256, 0, (cudaStream_t)stream>>>(A);
}

// =====================================================================================
// K2: DP fill, tiled.
//   Work item = one combination of the D(i) coordinates other than qstar, times a tile of
//   up to kTile consecutive values of qstar.  A lane group of G lanes splits the reduction
//   over C (lane l takes C = l, l+G, ...; loads of every table row are coalesced over C).
//   Per C the prefix of the canonical sum over terms [0, tstar) -- which do not depend on
//   qstar -- is computed once and reused by the kTile outputs of the tile (loop-invariant
//   hoisting of a prefix only: the association ((L + W..) + T..) is unchanged, so results
//   stay bit-identical to the oracle).  The (cost, C) pairs are then reduced across the
//   group with a butterfly reduce-scatter (each exchange halves the values a lane holds).
//   Table reads use ld.global.ca (not the non-coherent path): in the persistent schedule a
//   child table is written earlier in the same kernel.
// =====================================================================================
__device__ __forceinline__ void combine(double& b, int& c, double ob, int oc) {
    // lexicographic min of (cost, C): strict < over increasing C == Fig. 5 line 17
    if (ob < b || (ob == b && oc < c)) { b = ob; c = oc; }
}

// Item -> (combination of the untiled coordinates, tile index).  Single GPU: combinations
// fastest (the warps of a CTA share a tile: L1 reuse; tiles-fastest was measured slower,
// profiles/r02_ab_warm.txt).  Multi-GPU partitioned vertex (vd.part):
// [combinations below the partition coordinate] fastest, then the tile, then the partition
// coordinate -- so each rank's share of the vertex is ONE contiguous item range.
// x / d for x < 2^31 with the host's magic numbers (VertexDesc, fastdiv_magic)
__device__ __forceinline__ uint32_t fdiv(uint32_t x, uint32_t mul, int sh) {
    return (uint32_t)(((uint64_t)x * mul) >> sh);
}

__device__ __forceinline__ void split_item(const VertexDesc& vd, uint32_t it, uint32_t& combo, uint32_t& tile) {
    if (vd.part) {
        const uint32_t S = (uint32_t)vd.psub;
        const uint32_t t2 = fdiv(it, vd.mul_psub, vd.sh_psub), low = it - t2 * S;
        const uint32_t t3 = fdiv(t2, vd.mul_tile, vd.sh_tile);
        tile = t2 - t3 * (uint32_t)vd.ntile;
        combo = low + S * t3;
    } else {
        tile = fdiv(it, vd.mul_combo, vd.sh_combo);
        combo = it - tile * (uint32_t)vd.ncombo;
    }
}

template <int N>
struct Log2 { static constexpr int value = 1 + Log2<N / 2>::value; };
template <>
struct Log2<1> { static constexpr int value = 0; };

// Coherent L1-cached global load / store.  Explicit ld.global: the table pointers come from
// shared-memory descriptors, so a plain dereference compiles to a generic LD; an explicit
// .ca operator makes ptxas build a cache-policy descriptor per load on sm_100a; and
// ld.global.nc would be unsafe for tables written earlier in the same persistent launch.
__device__ __forceinline__ double ld(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
template <int OFF>                       // element offset folded into the instruction
__device__ __forceinline__ double ld_at(const double* p) {
    double v;
    asm volatile("ld.global.f64 %0, [%1+%2];" : "=d"(v) : "l"(p), "n"(OFF * 8));
    return v;
}
__device__ __forceinline__ void st_f64(double* p, double v) {
    asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_u16(uint16_t* p, int c) {
    asm volatile("st.global.u16 [%0], %1;" ::"l"(p), "h"((unsigned short)c) : "memory");
}
// Output of one DP entry; multi-GPU broadcast vertices also write it into every peer's copy
// of the table (peer stores over NVLink: the all-gather fused into the producer).
// A vertex with a single configuration (K = 1) has no argmin to record: its A(i) is never
// written (the back-substitution knows the choice is 0).
__device__ __forceinline__ void st_out(const VertexDesc& vd, int64_t phi, double v, int c) {
    st_f64(vd.T + phi, v);
    const bool arg = vd.K > 1;
    if (arg) st_u16(vd.A + phi, c);
    if (vd.bcast)
        for (int q = 0; q < vd.npeer; ++q) {
            if (vd.bcast & 1) st_f64(vd.Tpeer[q] + phi, v);
            if (arg) st_u16(vd.Apeer[q] + phi, c);
        }
}

// Dependency gate of a persistent task (round 2): the task's vertex may only READ its child tables
// once every child task has released them (pending counter = 0).  Each warp waits at its gate
// right before its first table load -- after its work-item decode and pointer setup, which need
// only the static descriptors -- so that setup overlaps the wait on the critical chain.  Lane 0
// polls (relaxed, .gpu or .sys scope), then fences (the acquire pattern), then __syncwarp orders
// the other lanes' loads after it.  A wait past the timeout flags the solve as failed (its
// results are discarded) and lets the warp run on.
struct Gate {
    const int32_t* p;            // the vertex's pending counter; nullptr: nothing to wait for
    int32_t* err;
    uint64_t timeout_ns;
    int multi;                   // group contexts: system scope (peers decrement it over NVLink)
    int* elect;                  // shared words {elected, open}: with non-null, the first warp to reach
                                 // its gate polls the global counter and opens a shared flag the
                                 // other warps spin on (one global poller per CTA instead of 8)
    int64_t* stamp;              // PASE_TRACE: per-warp {counter seen at 0, fence done} (ns)
    int ldacq;                   // acquire by ld.acquire of the counter instead of fence.acq_rel
    int warm;                    // CTA-uniform: the children were still running when the task was
                                 // claimed -- run the first work item once WITHOUT stores before the
                                 // gate (warms this SM's instruction caches with the tile's code
                                 // path and its static rows; results discarded, L1 invalidated by
                                 // the gate's fence)
};
__device__ __forceinline__ uint64_t gate_clock() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int gate_poll(const int32_t* p, int multi) {
    int v;
    if (multi) asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_shared_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_shared_relaxed(int* p, int v) {
    asm volatile("st.relaxed.cta.shared.s32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void gate_wait(Gate& g) {
    if (!g.p) return;
    if ((threadIdx.x & 31) == 0) {
        // elected mode: the first warp here polls global memory, the others spin on the shared
        // flag it opens after its acquire; each warp then fences itself (the poller's fence
        // synchronises with the releases, a waiter's fence with the poller's flag store)
        const bool poller = !g.elect || atomicCAS_block(g.elect, 0, 1) == 0;
        if (poller) {
            if (gate_poll(g.p, g.multi) != 0) {
                const uint64_t t0 = gate_clock();
                while (gate_poll(g.p, g.multi) != 0)
                    if (g.timeout_ns && gate_clock() - t0 > g.timeout_ns) { atomicExch(g.err, 1); break; }
            }
        } else {
            while (ld_shared_relaxed(g.elect + 1) == 0) __nanosleep(64);
        }
        if (g.stamp) g.stamp[2 * (threadIdx.x >> 5)] = (int64_t)gate_clock();
        if (g.multi) { int v; asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(g.p) : "memory"); (void)v; }
        else if (PASE_GATE_LDACQ) { int v; asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(g.p) : "memory"); (void)v; }
        else if (g.ldacq) { int v; asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(g.p) : "memory"); (void)v; }
        else asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (poller && g.elect) st_shared_relaxed(g.elect + 1, 1);
        if (g.stamp) g.stamp[2 * (threadIdx.x >> 5) + 1] = (int64_t)gate_clock();
    }
    __syncwarp();
    g.p = nullptr;
}

// Items of [i0, i1) for the calling warp.  Throughput mode (wlog == 0): the warp's lane
// groups take items first + k*stride + sub (warp-uniform loop).  Latency mode (G == 32,
// W = 2^wlog warps per item, for small vertices on the critical path): the W warps of an item
// split its C range (one round of loads per lane instead of K / (2G)), and their partial
// minima are combined through shared memory (CTA-uniform loop, CTA barriers).
template <int NP, int NS, int G>
__device__ __noinline__ void tile_items(const VertexDesc& vd, const TermDesc* td, int64_t first,
                                        int64_t stride, int64_t i1, double* red_b, int* red_c, Gate gate) {
    constexpr int V = kTile;
    constexpr int LG = Log2<G>::value, LV = Log2<V>::value;
    constexpr int S = LG < LV ? LG : LV;          // halving (reduce-scatter) steps
    constexpr int H = V >> S;                     // values a lane holds afterwards
    const int lane = threadIdx.x & (G - 1);
    const int wlog = G == 32 ? vd.wlog : 0;
    const int wsub = (threadIdx.x >> 5) & ((1 << wlog) - 1);      // warp's slice of C
    const int sub = wlog ? 0 : (threadIdx.x & 31) / G;
    const int q = vd.qstar;
    int sq[NS > 0 ? NS : 1];                            // host guarantees strides < 2^31
#pragma unroll
    for (int t = 0; t < NS; ++t) sq[t] = (int)td[NP + t].stride[q];
    // latency mode: rounds start at the CTA's first slot so every warp runs the same count
    const int64_t wib = (threadIdx.x >> 5) >> wlog;                // item slot within the CTA
    const int64_t b0 = wlog ? first - wib : first;
    const int64_t end = i1;
    // warm pass (Gate::warm): the first round once without stores, then the live rounds; one
    // loop body (live is loop-variant, so the body is not duplicated)
    bool live = !(gate.warm && gate.p);

    for (int64_t base = b0; base < end;) {
        const int64_t item = wlog ? base + wib : base + sub;
        const bool valid = item < end;
        const uint32_t it = valid ? (uint32_t)item : 0u;   // host guarantees nitems < 2^31
        const uint32_t nc = (uint32_t)vd.ncombo;
        uint32_t rem, tix;                                  // combos fastest: warps of a CTA
        split_item(vd, it, rem, tix);                       // share the qstar tile (L1 reuse)
        (void)nc;
        const int x0 = (int)tix * V;
        const int nb = valid ? min(V, vd.rq - x0) : 0;
        const double* pp[NP];
        const double* sp[NS > 0 ? NS : 1];
#pragma unroll
        for (int t = 0; t < NP; ++t) pp[t] = td[t].base;
#pragma unroll
        for (int t = 0; t < NS; ++t) sp[t] = td[NP + t].base + (int64_t)x0 * sq[t];
        int64_t obase = 0, ost = 1;
        for (int c = 0; c < vd.m; ++c) {                    // mixed-radix decode (lowest fastest)
            const uint32_t r = (uint32_t)vd.radix[c];
            if (c != q) {
                const uint32_t qv = fdiv(rem, vd.rmul[c], vd.rsh[c]);
                const uint32_t v = rem - qv * r;
                rem = qv;
                obase += (int64_t)v * ost;
#pragma unroll
                for (int t = 0; t < NP; ++t) pp[t] += (int64_t)v * td[t].stride[c];
#pragma unroll
                for (int t = 0; t < NS; ++t) sp[t] += (int64_t)v * td[NP + t].stride[c];
            }
            ost *= r;
        }
        double best[V];
        int bestC[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        const int Kv = nb > 0 ? (live ? vd.K : min(vd.K, kCUnroll * (G << wlog))) : 0;   // warm: one unrolled trip
        const int jmax = nb > 0 ? nb - 1 : 0;
        const int cstep = G << wlog;
        if (live) gate_wait(gate);                          // children complete (first item only)
#pragma unroll kCUnroll
        for (int C = lane + (wsub << LG); C < Kv; C += cstep) {   // unrolled: 2 C in flight
            double pre = ld(pp[0] + C);                     // L[C] (term 0 is never in the suffix)
#pragma unroll
            for (int t = 1; t < NP; ++t) pre = __dadd_rn(pre, ld(pp[t] + C));
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int jj = j < jmax ? j : jmax;         // clamp: branch-free partial tiles
                double cost = pre;
#pragma unroll
                for (int t = 0; t < NS; ++t) cost = __dadd_rn(cost, ld(sp[t] + (int64_t)jj * sq[t] + C));
                if (cost < best[j]) { best[j] = cost; bestC[j] = C; }   // strict <: lowest C
            }
        }
        // butterfly reduce-scatter across the G lanes of the group
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int o = G >> (s + 1);
            const int half = V >> (s + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double sb = up ? best[k] : best[k + half];
                const int sc = up ? bestC[k] : bestC[k + half];
                double kb = up ? best[k + half] : best[k];
                int kc = up ? bestC[k + half] : bestC[k];
                const double rb = __shfl_xor_sync(0xffffffffu, sb, o);
                const int rc = __shfl_xor_sync(0xffffffffu, sc, o);
                combine(kb, kc, rb, rc);
                best[k] = kb;
                bestC[k] = kc;
            }
        }
#pragma unroll
        for (int o = G >> (S + 1); o >= 1; o >>= 1)
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double rb = __shfl_xor_sync(0xffffffffu, best[k], o);
                const int rc = __shfl_xor_sync(0xffffffffu, bestC[k], o);
                combine(best[k], bestC[k], rb, rc);
            }
        int jbase = 0;
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane & (G >> (s + 1))) jbase += V >> (s + 1);
        if (G == 32 && wlog) {                              // combine the W warps' partials
            const int w = threadIdx.x >> 5;
            if ((lane & ((G >> S) - 1)) == 0)
#pragma unroll
                for (int k = 0; k < H; ++k) {
                    red_b[w * V + jbase + k] = best[k];
                    red_c[w * V + jbase + k] = bestC[k];
                }
            __syncthreads();
            if (wsub == 0 && lane < V) {
                double b = red_b[w * V + lane];
                int c = red_c[w * V + lane];
                for (int k = 1; k < (1 << wlog); ++k) combine(b, c, red_b[(w + k) * V + lane], red_c[(w + k) * V + lane]);
                if (live && lane < nb) st_out(vd, obase + (int64_t)(x0 + lane) * vd.ostride_q, b, c);
            }
            __syncthreads();
        } else if (live && (lane & ((G >> S) - 1)) == 0) {
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const int j = jbase + k;
                if (j < nb) st_out(vd, obase + (int64_t)(x0 + j) * vd.ostride_q, best[k], bestC[k]);
            }
        }
        if (live) base += stride;
        live = true;
    }
}

// 2-D register tile: a work item is one combination of the D(i) coordinates
// other than (qstar, q2) times a kTile1 x kTile2 block of (qstar, q2) values.  Per C, the
// canonical sum is built in its own order with loop-invariant prefixes hoisted:
//   pre      = terms [0, t2star)            (scalar: depend on neither tiled coordinate)
//   p1[j2]   = pre + terms [t2star, tstar)  (depend on q2 at most: kTile2 partials)
//   cost     = p1[j2] + S terms             (S = [tstar, nterms): kTile1 x kTile2 candidates)
// so per C a lane loads t2star + (kTile2 or 1 per P1 term) + (kTile1 or kTile1*kTile2 per S
// term) values for 16 candidates instead of NP + 8 NS for 8 (1-D tile).  Association order
// is unchanged, so the results are bit-identical to the oracle's.  NS = 1 (S term on qstar,
// optionally also q2) or NS = 2 (both S terms on qstar only).
template <int NS, int G>
__device__ __noinline__ void tile2_items(const VertexDesc& vd, const TermDesc* td, int64_t first,
                                         int64_t stride, int64_t end, Gate gate) {
    constexpr int V1 = kTile1, V2 = kTile2, V = V1 * V2;
    constexpr int LG = Log2<G>::value, LV = Log2<V>::value;
    constexpr int S = LG < LV ? LG : LV;
    constexpr int H = V >> S;
    const int lane = threadIdx.x & (G - 1);
    const int sub = (threadIdx.x & 31) / G;
    const int q1 = vd.qstar, q2 = vd.q2;
    const int nP0 = vd.t2star, nP1 = vd.tstar - vd.t2star, ts = vd.tstar;
    // per-term strides along the tiled coordinates (host: < 2^31)
    int p1s[kMaxP1];
#pragma unroll
    for (int t = 0; t < kMaxP1; ++t) p1s[t] = t < nP1 ? (int)td[nP0 + t].stride[q2] : 0;
    int s1[NS], s2[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) { s1[t] = (int)td[ts + t].stride[q1]; s2[t] = (int)td[ts + t].stride[q2]; }

    bool live = !(gate.warm && gate.p);                 // warm pass: see tile_items
    for (int64_t base = first; base < end;) {
        const int64_t item = base + sub;
        const bool valid = item < end;
        const uint32_t it = valid ? (uint32_t)item : 0u;
        const uint32_t nc = (uint32_t)vd.ncombo;
        uint32_t rem, tidx;
        split_item(vd, it, rem, tidx);
        (void)nc;
        const uint32_t t1 = fdiv(tidx, vd.mul_tile2, vd.sh_tile2);
        const int x2 = (int)(tidx - t1 * (uint32_t)vd.ntile2) * V2;
        const int x1 = (int)t1 * V1;
        const int nb1 = valid ? min(V1, vd.rq - x1) : 0;
        const int nb2 = valid ? min(V2, vd.rq2 - x2) : 0;
        const double* pp[kMaxP0];
        const double* pq[kMaxP1];
        const double* ps[NS];
#pragma unroll
        for (int t = 0; t < kMaxP0; ++t) pp[t] = td[t < nP0 ? t : 0].base;
#pragma unroll
        for (int t = 0; t < kMaxP1; ++t) pq[t] = t < nP1 ? td[nP0 + t].base + (int64_t)x2 * p1s[t] : pp[0];
#pragma unroll
        for (int t = 0; t < NS; ++t) ps[t] = td[ts + t].base + (int64_t)x1 * s1[t] + (int64_t)x2 * s2[t];
        int64_t obase = 0, ost = 1;
        for (int c = 0; c < vd.m; ++c) {                    // mixed-radix decode (lowest fastest)
            const uint32_t r = (uint32_t)vd.radix[c];
            if (c != q1 && c != q2) {
                const uint32_t qv = fdiv(rem, vd.rmul[c], vd.rsh[c]);
                const uint32_t v = rem - qv * r;
                rem = qv;
                obase += (int64_t)v * ost;
#pragma unroll
                for (int t = 0; t < kMaxP0; ++t) if (t < nP0) pp[t] += (int64_t)v * td[t].stride[c];
#pragma unroll
                for (int t = 0; t < kMaxP1; ++t) if (t < nP1) pq[t] += (int64_t)v * td[nP0 + t].stride[c];
#pragma unroll
                for (int t = 0; t < NS; ++t) ps[t] += (int64_t)v * td[ts + t].stride[c];
            }
            ost *= r;
        }
        double best[V];
        int bestC[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        const int Kv = (nb1 > 0 && nb2 > 0) ? (live ? vd.K : min(vd.K, G)) : 0;   // warm: one trip
        const int m1 = nb1 > 0 ? nb1 - 1 : 0, m2 = nb2 > 0 ? nb2 - 1 : 0;
        // every load of an iteration is unconditional (unused slots re-read a valid address), so
        // they issue together; only the adds are predicated on the vertex's segment sizes
        if (live) gate_wait(gate);
#pragma unroll 1
        for (int C = lane; C < Kv; C += G) {
            double a[kMaxP0];
#pragma unroll
            for (int t = 0; t < kMaxP0; ++t) a[t] = ld(pp[t] + C);
            double b[kMaxP1][V2];
#pragma unroll
            for (int t = 0; t < kMaxP1; ++t)
#pragma unroll
                for (int j2 = 0; j2 < V2; ++j2) b[t][j2] = ld(pq[t] + (int64_t)min(j2, m2) * p1s[t] + C);
            double pre = a[0];
#pragma unroll
            for (int t = 1; t < kMaxP0; ++t) if (t < nP0) pre = __dadd_rn(pre, a[t]);
            double p1[V2];
#pragma unroll
            for (int j2 = 0; j2 < V2; ++j2) {
                p1[j2] = pre;
#pragma unroll
                for (int t = 0; t < kMaxP1; ++t) if (t < nP1) p1[j2] = __dadd_rn(p1[j2], b[t][j2]);
            }
            if (NS == 1 && s2[0] != 0) {                    // S term on (qstar, q2)
                double x[V1][V2];
#pragma unroll
                for (int j1 = 0; j1 < V1; ++j1)
#pragma unroll
                    for (int j2 = 0; j2 < V2; ++j2)
                        x[j1][j2] = ld(ps[0] + (int64_t)min(j1, m1) * s1[0] + (int64_t)min(j2, m2) * s2[0] + C);
#pragma unroll
                for (int j1 = 0; j1 < V1; ++j1)
#pragma unroll
                    for (int j2 = 0; j2 < V2; ++j2) {
                        const double cost = __dadd_rn(p1[j2], x[j1][j2]);
                        const int j = j1 * V2 + j2;
                        if (cost < best[j]) { best[j] = cost; bestC[j] = C; }
                    }
            } else {                                        // S terms on qstar only
                double x[NS][V1];
#pragma unroll
                for (int t = 0; t < NS; ++t)
#pragma unroll
                    for (int j1 = 0; j1 < V1; ++j1) x[t][j1] = ld(ps[t] + (int64_t)min(j1, m1) * s1[t] + C);
#pragma unroll
                for (int j1 = 0; j1 < V1; ++j1)
#pragma unroll
                    for (int j2 = 0; j2 < V2; ++j2) {
                        double cost = __dadd_rn(p1[j2], x[0][j1]);
#pragma unroll
                        for (int t = 1; t < NS; ++t) cost = __dadd_rn(cost, x[t][j1]);
                        const int j = j1 * V2 + j2;
                        if (cost < best[j]) { best[j] = cost; bestC[j] = C; }
                    }
            }
        }
        // butterfly reduce-scatter across the G lanes of the group (as tile_items)
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int o = G >> (s + 1);
            const int half = V >> (s + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double sb = up ? best[k] : best[k + half];
                const int sc = up ? bestC[k] : bestC[k + half];
                double kb = up ? best[k + half] : best[k];
                int kc = up ? bestC[k + half] : bestC[k];
                const double rb = __shfl_xor_sync(0xffffffffu, sb, o);
                const int rc = __shfl_xor_sync(0xffffffffu, sc, o);
                combine(kb, kc, rb, rc);
                best[k] = kb;
                bestC[k] = kc;
            }
        }
#pragma unroll
        for (int o = G >> (S + 1); o >= 1; o >>= 1)
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double rb = __shfl_xor_sync(0xffffffffu, best[k], o);
                const int rc = __shfl_xor_sync(0xffffffffu, bestC[k], o);
                combine(best[k], bestC[k], rb, rc);
            }
        int jbase = 0;
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lane & (G >> (s + 1))) jbase += V >> (s + 1);
        if (live && (lane & ((G >> S) - 1)) == 0) {
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const int j = jbase + k, j1 = j / V2, j2 = j % V2;
                if (j1 < nb1 && j2 < nb2)
                    st_out(vd, obase + (int64_t)(x1 + j1) * vd.ostride_q + (int64_t)(x2 + j2) * vd.ostride_q2,
                           best[k], bestC[k]);
            }
        }
        if (live) base += stride;
        live = true;
    }
}

// 2-D register tile, single-suffix form (shape >= kShape2S): the structure of
// the big vertices of the zoo, in canonical term order --
//   P0: NP0 terms on neither tiled coordinate          (summed once per C: pre)
//   P1: one term on q2 (not q1), then NB terms on neither   (per q2 value: p1[j2])
//   S : one term on q1 (not q2), then, FORM-dependent, one more term on q1 (NS2 = 2) or on
//       neither (NS2 = 1)
//   cost(j1, j2) = ((((pre + A[j2]) + B..) + S1[j1]) + S2[j1])      (association unchanged)
// Per C a lane loads NP0 + 4 + NB + 4 (+ 4 or 1) values for 16 candidates (the 1-D tile: NP +
// 8 NS for 8), every address a per-item row pointer advanced by induction.
template <int NP0, int NB, int NS2, int G>
__device__ __noinline__ void tile2s_items(const VertexDesc& vd, const TermDesc* td, int64_t first,
                                          int64_t stride, int64_t end, Gate gate) {
    constexpr int V1 = kTile1, V2 = kTile2, V = V1 * V2;
    constexpr int LG = Log2<G>::value, LV = Log2<V>::value;
    constexpr int S = LG < LV ? LG : LV;
    constexpr int H = V >> S;
    constexpr int TA = NP0, TS = NP0 + 1 + NB;          // term index of A (P1 head), of S1
    constexpr int NR2 = NS2 == 2 ? V1 : 1;              // rows of the second suffix term
    const int lane = threadIdx.x & (G - 1);
    const int sub = (threadIdx.x & 31) / G;
    const int q1 = vd.qstar, q2 = vd.q2;
    const int64_t sb = td[TA].stride[q2], ss = td[TS].stride[q1];
    const int64_t ss2 = NS2 == 2 ? td[TS + 1].stride[q1] : 0;
    bool live = !(gate.warm && gate.p);                 // warm pass: see tile_items
    for (int64_t base = first; base < end;) {
        const int64_t item = base + sub;
        const bool valid = item < end;
        const uint32_t it = valid ? (uint32_t)item : 0u;
        const uint32_t nc = (uint32_t)vd.ncombo;
        uint32_t rem, tidx;
        split_item(vd, it, rem, tidx);
        (void)nc;
        const uint32_t t1 = fdiv(tidx, vd.mul_tile2, vd.sh_tile2);
        const int x2 = (int)(tidx - t1 * (uint32_t)vd.ntile2) * V2;
        const int x1 = (int)t1 * V1;
        const int nb1 = valid ? min(V1, vd.rq - x1) : 0;
        const int nb2 = valid ? min(V2, vd.rq2 - x2) : 0;
        // row pointers of every term at this item's combination (tiled coordinates at 0)
        const double* pa[NP0];
        const double* pe[NB > 0 ? NB : 1];
        const double* pt2;
#pragma unroll
        for (int t = 0; t < NP0; ++t) pa[t] = td[t].base;
#pragma unroll
        for (int t = 0; t < NB; ++t) pe[t] = td[TA + 1 + t].base;
        const double* pb = td[TA].base + (int64_t)x2 * sb;
        const double* ps = td[TS].base + (int64_t)x1 * ss;
        pt2 = NS2 ? td[TS + 1].base + (int64_t)x1 * ss2 : nullptr;
        int64_t obase = 0, ost = 1;
        for (int c = 0; c < vd.m; ++c) {                    // mixed-radix decode (lowest fastest)
            const uint32_t r = (uint32_t)vd.radix[c];
            if (c != q1 && c != q2) {
                const uint32_t qv = fdiv(rem, vd.rmul[c], vd.rsh[c]);
                const uint32_t v = rem - qv * r;
                rem = qv;
                obase += (int64_t)v * ost;
#pragma unroll
                for (int t = 0; t < NP0; ++t) pa[t] += (int64_t)v * td[t].stride[c];
#pragma unroll
                for (int t = 0; t < NB; ++t) pe[t] += (int64_t)v * td[TA + 1 + t].stride[c];
                pb += (int64_t)v * td[TA].stride[c];
                ps += (int64_t)v * td[TS].stride[c];
                if (NS2) pt2 += (int64_t)v * td[TS + 1].stride[c];
            }
            ost *= r;
        }
        const int m1 = nb1 > 0 ? nb1 - 1 : 0, m2 = nb2 > 0 ? nb2 - 1 : 0;
        const double* b[V2];
        const double* s[V1];
        const double* s2[NR2];
#pragma unroll
        for (int j = 0; j < V2; ++j) b[j] = pb + (int64_t)min(j, m2) * sb + lane;   // partial tiles
#pragma unroll
        for (int j = 0; j < V1; ++j) s[j] = ps + (int64_t)min(j, m1) * ss + lane;   // re-read a
#pragma unroll
        for (int j = 0; j < NR2; ++j) s2[j] = NS2 ? pt2 + (int64_t)min(j, m1) * ss2 + lane : nullptr;  // valid row
#pragma unroll
        for (int t = 0; t < NP0; ++t) pa[t] += lane;
#pragma unroll
        for (int t = 0; t < NB; ++t) pe[t] += lane;
        double best[V];
        int bestC[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        const int Kv = (nb1 > 0 && nb2 > 0) ? (live ? vd.K : min(vd.K, 2 * G)) : 0;   // warm: one trip
        // every row pointer starts at this lane's C and advances by 2G per double iteration;
        // the second iteration's loads carry +G as an immediate
        auto step = [&](auto off, int C) {
            constexpr int O = decltype(off)::value;
            double pre = ld_at<O>(pa[0]);
#pragma unroll
            for (int t = 1; t < NP0; ++t) pre = __dadd_rn(pre, ld_at<O>(pa[t]));
            double p1[V2], sv[V1], tv[NR2], ev[NB > 0 ? NB : 1];
#pragma unroll
            for (int j = 0; j < V2; ++j) p1[j] = ld_at<O>(b[j]);
#pragma unroll
            for (int t = 0; t < NB; ++t) ev[t] = ld_at<O>(pe[t]);
#pragma unroll
            for (int j = 0; j < V1; ++j) sv[j] = ld_at<O>(s[j]);
            if (NS2) {
#pragma unroll
                for (int j = 0; j < NR2; ++j) tv[j] = ld_at<O>(s2[j]);
            }
#pragma unroll
            for (int j = 0; j < V2; ++j) {
                p1[j] = __dadd_rn(pre, p1[j]);
#pragma unroll
                for (int t = 0; t < NB; ++t) p1[j] = __dadd_rn(p1[j], ev[t]);
            }
#pragma unroll
            for (int j1 = 0; j1 < V1; ++j1)
#pragma unroll
                for (int j2 = 0; j2 < V2; ++j2) {
                    double cost = __dadd_rn(p1[j2], sv[j1]);
                    if (NS2) cost = __dadd_rn(cost, tv[NS2 == 2 ? j1 : 0]);
                    const int j = j1 * V2 + j2;
                    if (cost < best[j]) { best[j] = cost; bestC[j] = C; }   // strict <: lowest C
                }
        };
        if (live) gate_wait(gate);
        int C = lane;
#pragma unroll 1
        for (; C + G < Kv; C += 2 * G) {
            step(std::integral_constant<int, 0>{}, C);
            step(std::integral_constant<int, G>{}, C + G);
#pragma unroll
            for (int t = 0; t < NP0; ++t) pa[t] += 2 * G;
#pragma unroll
            for (int t = 0; t < NB; ++t) pe[t] += 2 * G;
#pragma unroll
            for (int j = 0; j < V2; ++j) b[j] += 2 * G;
#pragma unroll
            for (int j = 0; j < V1; ++j) s[j] += 2 * G;
#pragma unroll
            for (int j = 0; j < NR2; ++j) s2[j] += NS2 ? 2 * G : 0;
        }
        if (C < Kv) step(std::integral_constant<int, 0>{}, C);
        // butterfly reduce-scatter across the G lanes of the group (as tile_items)
#pragma unroll
        for (int st = 0; st < S; ++st) {
            const int o = G >> (st + 1);
            const int half = V >> (st + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double sbv = up ? best[k] : best[k + half];
                const int sc = up ? bestC[k] : bestC[k + half];
                double kb = up ? best[k + half] : best[k];
                int kc = up ? bestC[k + half] : bestC[k];
                const double rb = __shfl_xor_sync(0xffffffffu, sbv, o);
                const int rc = __shfl_xor_sync(0xffffffffu, sc, o);
                combine(kb, kc, rb, rc);
                best[k] = kb;
                bestC[k] = kc;
            }
        }
#pragma unroll
        for (int o = G >> (S + 1); o >= 1; o >>= 1)
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const double rb = __shfl_xor_sync(0xffffffffu, best[k], o);
                const int rc = __shfl_xor_sync(0xffffffffu, bestC[k], o);
                combine(best[k], bestC[k], rb, rc);
            }
        int jbase = 0;
#pragma unroll
        for (int st = 0; st < S; ++st)
            if (lane & (G >> (st + 1))) jbase += V >> (st + 1);
        if (live && (lane & ((G >> S) - 1)) == 0) {
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const int j = jbase + k, j1 = j / V2, j2 = j % V2;
                if (j1 < nb1 && j2 < nb2)
                    st_out(vd, obase + (int64_t)(x1 + j1) * vd.ostride_q + (int64_t)(x2 + j2) * vd.ostride_q2,
                           best[k], bestC[k]);
            }
        }
        if (live) base += stride;
        live = true;
    }
}

// Generic path (any number of terms, 64-bit strides): one lane group per output phi,
// offsets recomputed per candidate.  Outputs [first + k*stride + sub, ...) < end.
__device__ __noinline__ void generic_items(const VertexDesc& vd, const TermDesc* __restrict__ tds, int glog,
                                           int64_t first, int64_t stride, int64_t end, Gate gate) {
    const int g = 1 << glog;
    const int lane = threadIdx.x & (g - 1);
    const int sub = (threadIdx.x & 31) >> glog;
    bool live = !(gate.warm && gate.p);                 // warm pass: see tile_items
    for (int64_t base = first; base < end;) {
        const int64_t phi = base + sub;
        const int K = phi < end ? (live ? vd.K : min(vd.K, g)) : 0;   // warm: one trip
        int32_t c[kMaxDep];
        int64_t rem = phi < end ? phi : 0;
        for (int q = 0; q < vd.m; ++q) { c[q] = (int32_t)(rem % vd.radix[q]); rem /= vd.radix[q]; }
        double best = __longlong_as_double(0x7ff0000000000000ll);
        int bestC = 0x7fffffff;
        if (live) gate_wait(gate);
        for (int C = lane; C < K; C += g) {
            double cost = 0.0;
            for (int t = 0; t < vd.nterms; ++t) {
                const TermDesc& d = tds[vd.term0 + t];
                int64_t off = 0;
                for (int q = 0; q < vd.m; ++q) off += (int64_t)c[q] * d.stride[q];
                const double x = ld(d.base + off + C);
                cost = t == 0 ? x : __dadd_rn(cost, x);
            }
            if (cost < best) { best = cost; bestC = C; }
        }
        for (int o = g >> 1; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bestC, o);
            combine(best, bestC, ob, oc);
        }
        if (live && lane == 0 && K > 0) st_out(vd, phi, best, bestC);
        if (live) base += stride;
        live = true;
    }
}


// =====================================================================================
// Streaming-regime tile: the vertex's last term is a child table
// spanning (sigma_i, D(i)), so every candidate reads one 8-B value that nothing else reads and
// the vertex is HBM-bound.  The rows of that term are STAGED INTO SHARED MEMORY BY TMA BULK
// COPIES (cp.async.bulk, completion on a per-stage mbarrier) in a kStreamStages-deep ring per
// warp over the reduction range: chunk c of an item = C in [32c, 32c + 32) of its kTile rows,
// so (kStreamStages - 1) chunks of every warp are in flight while it reduces the current one.
// Everything else is the 1-D tile with one item per warp (G = 32): the prefix terms [0, tstar)
// summed once per C, the suffix terms per output, the spanning term last, strict < over
// increasing C, butterfly argmin -- the canonical association, so results stay bit-identical.
// =====================================================================================
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(__cvta_generic_to_global(src)), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

constexpr int kStreamStages = 4;                         // chunks per warp ring
constexpr int kStreamRow = 34;                           // doubles per staged row chunk: 32 + alignment
constexpr int kStreamStage = kTile * kStreamRow;         // doubles per stage (kTile rows)
constexpr int kStreamWarps = 8;                          // warps per CTA (256 threads)
static_assert(kCtaSmemMax <= (size_t)kStreamWarps * kStreamStages * kStreamStage * 8, "CTA tile in the ring area");
constexpr size_t kStreamSmemBytes = (size_t)kStreamWarps * kStreamStages * kStreamStage * 8 +
                                    (size_t)kStreamWarps * kStreamStages * 8;

// ring of warp w: stages at dyn + w * stages * stage, barriers after all stages
__device__ __forceinline__ double* stream_buf(unsigned char* dyn, int w) {
    return reinterpret_cast<double*>(dyn) + (size_t)w * kStreamStages * kStreamStage;
}
__device__ __forceinline__ uint64_t* stream_bar(unsigned char* dyn, int w) {
    return reinterpret_cast<uint64_t*>(dyn + (size_t)kStreamWarps * kStreamStages * kStreamStage * 8) + w * kStreamStages;
}
__device__ __forceinline__ void stream_init(unsigned char* dyn) {      // once per CTA, before any use
    if (threadIdx.x < kStreamWarps * kStreamStages) mbar_init(stream_bar(dyn, 0) + threadIdx.x, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
}

// Decode of one item for the stream tile: output base, row pointers of every term at the
// item's combination (tiled coordinate at x0), rows in the tile.
template <int NP, int NS>
__device__ __forceinline__ void stream_decode(const VertexDesc& vd, const TermDesc* td, int64_t item,
                                              int64_t& obase, const double** pp, const double** sp, int& x0,
                                              int& nb) {
    const int q = vd.qstar;
    uint32_t rem, tix;
    split_item(vd, (uint32_t)item, rem, tix);
    x0 = (int)tix * kTile;
    nb = min(kTile, vd.rq - x0);
#pragma unroll
    for (int t = 0; t < NP; ++t) pp[t] = td[t].base;
#pragma unroll
    for (int t = 0; t < NS; ++t) sp[t] = td[NP + t].base + (int64_t)x0 * td[NP + t].stride[q];
    obase = 0;
    int64_t ost = 1;
    for (int c = 0; c < vd.m; ++c) {
        const uint32_t r = (uint32_t)vd.radix[c];
        if (c != q) {
            const uint32_t qv = fdiv(rem, vd.rmul[c], vd.rsh[c]);
            const uint32_t v = rem - qv * r;
            rem = qv;
            obase += (int64_t)v * ost;
#pragma unroll
            for (int t = 0; t < NP; ++t) pp[t] += (int64_t)v * td[t].stride[c];
#pragma unroll
            for (int t = 0; t < NS; ++t) sp[t] += (int64_t)v * td[NP + t].stride[c];
        }
        ost *= r;
    }
}

template <int NP, int NS>
__device__ __noinline__ uint32_t tile_stream_items(const VertexDesc& vd, const TermDesc* td, int64_t first,
                                                   int64_t stride, int64_t end, unsigned char* dyn, uint32_t seq,
                                                   Gate gate) {
    constexpr int V = kTile, S = 3, H = 1;               // G = 32: 3 halving steps, then 2 more
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & (kStreamWarps - 1);
    double* buf = stream_buf(dyn, w);
    uint64_t* bar = stream_bar(dyn, w);
    const int q = vd.qstar;
    const int K = vd.K;
    const int nch = (K + 31) >> 5;
    const int64_t sqs = td[NP + NS - 1].stride[q];       // row stride of the spanning term's tile
    int sq[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) sq[t] = (int)td[NP + t].stride[q];
    // producer cursor (warp-uniform): next (item, chunk) to stage; lanes < kTile hold its row
    int64_t pitem = first;
    int pch = 0;
    const double* prow = nullptr;
    auto prow_of = [&](int64_t item) {
        int64_t ob;
        const double* pp_[NP];
        const double* sp_[NS];
        int x0, nb;
        stream_decode<NP, NS>(vd, td, item, ob, pp_, sp_, x0, nb);
        return sp_[NS - 1] + (int64_t)min(lane, nb - 1) * sqs;
    };
    if (pitem < end && lane < V) prow = prow_of(pitem);
    gate_wait(gate);
    if (lane < V) fence_proxy_async_global();            // acquired child writes -> async-proxy reads
    uint32_t pseq = seq;
    auto produce = [&]() {                               // stage chunk (pitem, pch) as sequence pseq
        const int st = pseq % kStreamStages;
        double* dst = buf + st * kStreamStage;
        if (lane == 0) {
            fence_proxy_async_smem();                    // generic reads of this stage precede the refill
            mbar_expect_tx(bar + st, (uint32_t)(V * kStreamRow * 8));
        }
        __syncwarp();
        if (lane < V) {
            const double* a = prow + 32 * pch;
            a -= ((uintptr_t)a >> 3) & 1;                // 16-B aligned source, data at +0 or +1
            bulk_g2s(dst + lane * kStreamRow, a, kStreamRow * 8, bar + st);
        }
        ++pseq;
        if (++pch == nch) {
            pch = 0;
            pitem += stride;
            if (pitem < end && lane < V) prow = prow_of(pitem);
        }
    };
    for (int k = 0; k < kStreamStages - 1 && pitem < end; ++k) produce();
    for (int64_t item = first; item < end; item += stride) {
        int64_t obase;
        const double* pp[NP];
        const double* sp[NS];
        int x0, nb;
        stream_decode<NP, NS>(vd, td, item, obase, pp, sp, x0, nb);
        const int jmax = nb - 1;
        int sh[V];                                       // staged row j starts at +0 or +1
#pragma unroll
        for (int j = 0; j < V; ++j) sh[j] = (int)(((uintptr_t)(sp[NS - 1] + (int64_t)min(j, jmax) * sqs) >> 3) & 1);
        double best[V];
        int bestC[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        for (int ch = 0; ch < nch; ++ch) {
            if (pitem < end) produce();                  // keep kStreamStages - 1 chunks in flight
            const int st = seq % kStreamStages;
            mbar_wait(bar + st, (seq / kStreamStages) & 1);
            const double* sm = buf + st * kStreamStage;
            const int C = 32 * ch + lane;
            if (C < K) {
                double pre = ld(pp[0] + C);
#pragma unroll
                for (int t = 1; t < NP; ++t) pre = __dadd_rn(pre, ld(pp[t] + C));
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const int jj = j < jmax ? j : jmax;
                    double cost = pre;
#pragma unroll
                    for (int t = 0; t < NS - 1; ++t) cost = __dadd_rn(cost, ld(sp[t] + (int64_t)jj * sq[t] + C));
                    cost = __dadd_rn(cost, sm[jj * kStreamRow + sh[jj] + lane]);
                    if (cost < best[j]) { best[j] = cost; bestC[j] = C; }
                }
            }
            __syncwarp();                                // every lane is done with this stage
            ++seq;
        }
        // butterfly reduce-scatter across the warp (as tile_items with G = 32)
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
            const int o = 32 >> (s2 + 1);
            const int half = V >> (s2 + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double sb = up ? best[k] : best[k + half];
                const int sc = up ? bestC[k] : bestC[k + half];
                double kb = up ? best[k + half] : best[k];
                int kc = up ? bestC[k + half] : bestC[k];
                const double rb = __shfl_xor_sync(0xffffffffu, sb, o);
                const int rc = __shfl_xor_sync(0xffffffffu, sc, o);
                combine(kb, kc, rb, rc);
                best[k] = kb;
                bestC[k] = kc;
            }
        }
#pragma unroll
        for (int o = 32 >> (S + 1); o >= 1; o >>= 1) {
            const double rb = __shfl_xor_sync(0xffffffffu, best[0], o);
            const int rc = __shfl_xor_sync(0xffffffffu, bestC[0], o);
            combine(best[0], bestC[0], rb, rc);
        }
        int jbase = 0;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2)
            if (lane & (32 >> (s2 + 1))) jbase += V >> (s2 + 1);
        if ((lane & 3) == 0 && jbase < nb) st_out(vd, obase + (int64_t)(x0 + jbase) * vd.ostride_q, best[0], bestC[0]);
        (void)H;
    }
    return seq;
}

// Streaming-regime tile, L2-prefetch form: the 1-D tile with one item per warp (G = 32) reading
// the spanning rows with coalesced 256-B loads, while lanes 0..kTile-1 hand the NEXT item's rows
// to the TMA unit as bulk L2 prefetches (cp.async.bulk.prefetch.L2) -- the HBM stream runs one
// item ahead of the loads, with no shared-memory round trip and no per-chunk synchronisation.
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(bytes) : "memory");
}

template <int NP, int NS>
__device__ __noinline__ void tile_stream_pf(const VertexDesc& vd, const TermDesc* td, int64_t first,
                                            int64_t stride, int64_t end, Gate gate) {
    constexpr int V = kTile, S = 3;
    const int lane = threadIdx.x & 31;
    const int q = vd.qstar;
    const int K = vd.K;
    const int64_t sqs = td[NP + NS - 1].stride[q];
    int sq[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) sq[t] = (int)td[NP + t].stride[q];
    // one row = K doubles from an 8-B aligned start: prefetch the 16-B aligned cover
    auto prefetch_rows = [&](int64_t item) {
        int64_t ob;
        const double* pp_[NP];
        const double* sp_[NS];
        int x0, nb;
        stream_decode<NP, NS>(vd, td, item, ob, pp_, sp_, x0, nb);
        if (lane < nb) {
            const uintptr_t a = (uintptr_t)(sp_[NS - 1] + (int64_t)lane * sqs);
            const uintptr_t lo = a & ~(uintptr_t)15, hi = (a + (uintptr_t)K * 8 + 15) & ~(uintptr_t)15;
            bulk_prefetch_l2((const void*)lo, (uint32_t)(hi - lo));
        }
    };
    const int64_t ahead = (int64_t)vd.pf_ahead * stride;
    for (int64_t k = 0; k < ahead; k += stride)
        if (first + k < end && lane < V) prefetch_rows(first + k);
    for (int64_t item = first; item < end; item += stride) {
        if (item + ahead < end && lane < V) prefetch_rows(item + ahead);
        int64_t obase;
        const double* pp[NP];
        const double* sp[NS];
        int x0, nb;
        stream_decode<NP, NS>(vd, td, item, obase, pp, sp, x0, nb);
        const int jmax = nb - 1;
        double best[V];
        int bestC[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        gate_wait(gate);
#pragma unroll 2
        for (int C = lane; C < K; C += 32) {
            double pre = ld(pp[0] + C);
#pragma unroll
            for (int t = 1; t < NP; ++t) pre = __dadd_rn(pre, ld(pp[t] + C));
#pragma unroll
            for (int j = 0; j < V; ++j) {
                const int jj = j < jmax ? j : jmax;
                double cost = pre;
#pragma unroll
                for (int t = 0; t < NS - 1; ++t) cost = __dadd_rn(cost, ld(sp[t] + (int64_t)jj * sq[t] + C));
                cost = __dadd_rn(cost, ld(sp[NS - 1] + (int64_t)jj * sqs + C));
                if (cost < best[j]) { best[j] = cost; bestC[j] = C; }
            }
        }
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
            const int o = 32 >> (s2 + 1);
            const int half = V >> (s2 + 1);
            const bool up = (lane & o) != 0;
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const double sb = up ? best[k] : best[k + half];
                const int sc = up ? bestC[k] : bestC[k + half];
                double kb = up ? best[k + half] : best[k];
                int kc = up ? bestC[k + half] : bestC[k];
                const double rb = __shfl_xor_sync(0xffffffffu, sb, o);
                const int rc = __shfl_xor_sync(0xffffffffu, sc, o);
                combine(kb, kc, rb, rc);
                best[k] = kb;
                bestC[k] = kc;
            }
        }
#pragma unroll
        for (int o = 32 >> (S + 1); o >= 1; o >>= 1) {
            const double rb = __shfl_xor_sync(0xffffffffu, best[0], o);
            const int rc = __shfl_xor_sync(0xffffffffu, bestC[0], o);
            combine(best[0], bestC[0], rb, rc);
        }
        int jbase = 0;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2)
            if (lane & (32 >> (s2 + 1))) jbase += V >> (s2 + 1);
        if ((lane & 3) == 0 && jbase < nb) st_out(vd, obase + (int64_t)(x0 + jbase) * vd.ostride_q, best[0], bestC[0]);
    }
}

// CTA-tiled min-plus (shape kShapeCta): the single-suffix structure of tile2s
//   cost(j1, j2) = ((((P0 sum + A[j2]) + B) + S1[j1]) + S2)       (FORM as tile2s; canonical order)
// with one CTA item = one combination x a cb1 x cb2 block of (qstar, q2).  Rounds of kCtaG *
// kCtaCC values of C are staged in shared memory by cp.async (LDGSTS: no registers, every copy in
// flight), double-buffered: round r + 1 is copied while round r is reduced.  A pass per round
// forms p1[c][j2] = (P0 sum + A[j2]) (+ B) in place; then the CTA's kCtaG groups of 64 threads
// each reduce kCtaCC values of C, every thread a 4 x 4 block of outputs (8 shared loads per 16
// candidates, no address arithmetic, no cross-lane traffic).  The groups' (min, first argmin)
// pairs are combined lexicographically at the end -- the oracle's strict < over increasing C --
// so T, A stay bit-identical.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// shared doubles of one staging buffer (the host checks two of them fit kCtaSmemMax)
__host__ __device__ constexpr int cta_buffer_doubles(int cb1, int cb2) {
    return kCtaG * kCtaCC * ((kMaxP0 + 2) + (cb2 + 1) + 2 * (cb1 + 1));
}

template <int NP0, int FORM>
__device__ __noinline__ void cta_items(const VertexDesc& vd, const TermDesc* td, int64_t i0, int64_t stride,
                                       int64_t i1, unsigned char* dyn, Gate gate) {
    constexpr int NB = FORM == 1 ? 1 : 0, NS2 = FORM == 2 ? 1 : FORM == 3 ? 2 : 0;
    constexpr int TA = NP0, TS = NP0 + 1 + NB;
    constexpr int CR = kCtaG * kCtaCC;                   // values of C per round
    constexpr int NQ = NP0 + NB + (NS2 == 1 ? 1 : 0);    // per-C rows: P0 terms, B, constant S2
    const int cb1 = vd.cb1, cb2 = vd.cb2;
    const int T2 = cb2 >> 2, T1 = cb1 >> 2;
    const int ld2 = cb2 + 1, ld1 = cb1 + 1;              // odd row pitch (doubles)
    // buffer layout: q[NQ][CR] | p1[CR][ld2] | s1[CR][ld1] | s2[CR][ld1]
    const int bufd = cta_buffer_doubles(cb1, cb2);
    double* const base0 = reinterpret_cast<double*>(dyn);
    const int tid = threadIdx.x;
    const int grp = tid >> 6, u = tid & 63;
    const int t2 = u % T2, t1 = u / T2;
    const bool act = t1 < T1;
    const int q1 = vd.qstar, q2 = vd.q2;
    const int64_t sb = td[TA].stride[q2], ss = td[TS].stride[q1];
    const int64_t ss2 = NS2 == 2 ? td[TS + 1].stride[q1] : 0;
    const int K = vd.K;
    bool live = !(gate.warm && gate.p);
    for (int64_t it = i0; it < i1;) {
        const uint32_t combo = fdiv((uint32_t)it, vd.mul_tile, vd.sh_tile);
        const uint32_t blk = (uint32_t)it - combo * (uint32_t)vd.ntile;
        const uint32_t b1 = fdiv(blk, vd.mul_tile2, vd.sh_tile2);
        const int x1 = (int)b1 * cb1, x2 = (int)(blk - b1 * (uint32_t)vd.ntile2) * cb2;
        const int nb1 = min(cb1, vd.rq - x1), nb2 = min(cb2, vd.rq2 - x2);
        const double* pq[NQ > 0 ? NQ : 1];               // per-C rows: P0 terms, then B, then S2c
        const double* pb = td[TA].base + (int64_t)x2 * sb;
        const double* ps = td[TS].base + (int64_t)x1 * ss;
        const double* pt2 = NS2 == 2 ? td[TS + 1].base + (int64_t)x1 * ss2 : nullptr;
#pragma unroll
        for (int t = 0; t < NP0; ++t) pq[t] = td[t].base;
        if (NB) pq[NP0] = td[TA + 1].base;
        if (NS2 == 1) pq[NP0 + NB] = td[TS + 1].base;
        int64_t obase = 0, ost = 1;
        uint32_t rem = combo;
        for (int c = 0; c < vd.m; ++c) {                    // mixed-radix decode (lowest fastest)
            const uint32_t r = (uint32_t)vd.radix[c];
            if (c != q1 && c != q2) {
                const uint32_t qv = fdiv(rem, vd.rmul[c], vd.rsh[c]);
                const uint32_t v = rem - qv * r;
                rem = qv;
                obase += (int64_t)v * ost;
#pragma unroll
                for (int t = 0; t < NP0; ++t) pq[t] += (int64_t)v * td[t].stride[c];
                if (NB) pq[NP0] += (int64_t)v * td[TA + 1].stride[c];
                if (NS2 == 1) pq[NP0 + NB] += (int64_t)v * td[TS + 1].stride[c];
                pb += (int64_t)v * td[TA].stride[c];
                ps += (int64_t)v * td[TS].stride[c];
                if (NS2 == 2) pt2 += (int64_t)v * td[TS + 1].stride[c];
            }
            ost *= r;
        }
        double best[16];
        int bestC[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) { best[j] = __longlong_as_double(0x7ff0000000000000ll); bestC[j] = 0x7fffffff; }
        const int Kc = live ? K : min(K, CR);            // warm: one round
        const int nr = (Kc + CR - 1) / CR;
        // copy round r into buffer r & 1 (every thread issues its share; rows clamped to the block)
        auto issue = [&](int r) {
            double* B = base0 + (r & 1) * bufd;
            double* qs = B;
            double* as = qs + (kMaxP0 + 2) * CR;
            double* s1 = as + CR * ld2;
            double* s2 = s1 + CR * ld1;
            const int c0 = r * CR, nc = min(CR, Kc - c0);
            for (int x = tid; x < NQ * CR; x += blockDim.x) {
                const int c = x % CR, t = x / CR;
                if (c < nc) cp_async8(qs + t * CR + c, pq[t] + c0 + c);
            }
            for (int x = tid; x < CR * cb2; x += blockDim.x) {
                const int c = x % CR, jj = x / CR;
                if (c < nc) cp_async8(as + c * ld2 + jj, pb + (int64_t)min(jj, nb2 - 1) * sb + c0 + c);
            }
            for (int x = tid; x < CR * cb1; x += blockDim.x) {
                const int c = x % CR, jj = x / CR;
                if (c < nc) {
                    cp_async8(s1 + c * ld1 + jj, ps + (int64_t)min(jj, nb1 - 1) * ss + c0 + c);
                    if (NS2 == 2) cp_async8(s2 + c * ld1 + jj, pt2 + (int64_t)min(jj, nb1 - 1) * ss2 + c0 + c);
                }
            }
            cp_async_commit();
        };
        if (live) gate_wait(gate);                          // (each warp; the barrier below joins them)
        __syncthreads();                                    // the previous item's buffers are free
        if (nr > 0) issue(0);
        for (int r = 0; r < nr; ++r) {
            if (r + 1 < nr) { issue(r + 1); cp_async_wait<1>(); } else { cp_async_wait<0>(); }
            __syncthreads();                                // round r landed (every thread's copies)
            double* B = base0 + (r & 1) * bufd;
            double* qs = B;
            double* as = qs + (kMaxP0 + 2) * CR;
            double* s1 = as + CR * ld2;
            double* s2 = s1 + CR * ld1;
            const int c0 = r * CR, nc = min(CR, Kc - c0);
            // p1[c][j2] = ((P0 sum) + A[j2]) (+ B), in place over the staged A
            for (int x = tid; x < CR * cb2; x += blockDim.x) {
                const int c = x % CR, jj = x / CR;
                if (c < nc) {
                    double pre = qs[c];
#pragma unroll
                    for (int t = 1; t < NP0; ++t) pre = __dadd_rn(pre, qs[t * CR + c]);
                    double v = __dadd_rn(pre, as[c * ld2 + jj]);
                    if (NB) v = __dadd_rn(v, qs[NP0 * CR + c]);
                    as[c * ld2 + jj] = v;
                }
            }
            __syncthreads();
            const int ce = min(kCtaCC * (grp + 1), nc);
            if (act) {
#pragma unroll 2
                for (int c = kCtaCC * grp; c < ce; ++c) {
                    double p[4], sv[4], s2v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        p[k] = as[c * ld2 + 4 * t2 + k];
                        sv[k] = s1[c * ld1 + 4 * t1 + k];
                        if (NS2 == 2) s2v[k] = s2[c * ld1 + 4 * t1 + k];
                    }
                    const double s2c = NS2 == 1 ? qs[(NP0 + NB) * CR + c] : 0.0;
                    const int C = c0 + c;
#pragma unroll
                    for (int j1 = 0; j1 < 4; ++j1)
#pragma unroll
                        for (int j2 = 0; j2 < 4; ++j2) {
                            double cost = __dadd_rn(p[j2], sv[j1]);
                            if (NS2 == 1) cost = __dadd_rn(cost, s2c);
                            if (NS2 == 2) cost = __dadd_rn(cost, s2v[j1]);
                            const int j = j1 * 4 + j2;
                            if (cost < best[j]) { best[j] = cost; bestC[j] = C; }   // strict <: lowest C
                        }
                }
            }
            __syncthreads();                                // buffer r & 1 is refilled by round r + 2
        }
        // combine the groups' partial (min, argmin) per output: [g][j][u] in the staging area
        double* rb = base0;
        int* rc = reinterpret_cast<int*>(rb + kCtaG * 16 * 64);
        if (grp > 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                rb[(grp * 16 + j) * 64 + u] = best[j];
                rc[(grp * 16 + j) * 64 + u] = bestC[j];
            }
        }
        __syncthreads();
        if (grp == 0 && act) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                for (int g2 = 1; g2 < kCtaG; ++g2)
                    combine(best[j], bestC[j], rb[(g2 * 16 + j) * 64 + u], rc[(g2 * 16 + j) * 64 + u]);
            if (live) {
#pragma unroll
                for (int j1 = 0; j1 < 4; ++j1)
#pragma unroll
                    for (int j2 = 0; j2 < 4; ++j2) {
                        const int a1 = 4 * t1 + j1, a2 = 4 * t2 + j2;
                        if (a1 < nb1 && a2 < nb2)
                            st_out(vd, obase + (int64_t)(x1 + a1) * vd.ostride_q + (int64_t)(x2 + a2) * vd.ostride_q2,
                                   best[j1 * 4 + j2], bestC[j1 * 4 + j2]);
                    }
            }
        }
        if (live) it += stride;
        live = true;
    }
}

// shape index: 0..63 = tiled (NP-1)*16 + NS*4 + (log2 G - 2); -1 = generic
//   first_warp / nwarps: the calling warp's index / the warps sharing [i0, i1) (a CTA's warps
//   are consecutive).  Item slots per warp: 32/G (throughput mode) or 1/W (latency mode).
__device__ __forceinline__ void run_shape(int shape, const VertexDesc& vd, const TermDesc* td_sh,
                                          const TermDesc* tds_g, int64_t first_warp, int64_t nwarps,
                                          int64_t i0, int64_t i1, double* red_b, int* red_c,
                                          unsigned char* dyn, uint32_t& seq, Gate gate) {
    switch (shape) {
#define PASE_CASE(NP, NS, LGG)                                                                    \
    case (NP - 1) * 16 + NS * 4 + (LGG - 2): {                                                    \
        constexpr int G_ = 1 << LGG, GPW_ = 32 / G_;                                              \
        if (G_ == 32 && vd.wlog)                                                                  \
            tile_items<NP, NS, G_>(vd, td_sh, i0 + (first_warp >> vd.wlog), nwarps >> vd.wlog, i1,   \
                                   red_b, red_c, gate);                                           \
        else                                                                                      \
            tile_items<NP, NS, G_>(vd, td_sh, i0 + first_warp * GPW_, nwarps * GPW_, i1, red_b, red_c, gate); \
        return;                                                                                   \
    }
#define PASE_NS(NP, NS) PASE_CASE(NP, NS, 2) PASE_CASE(NP, NS, 3) PASE_CASE(NP, NS, 4) PASE_CASE(NP, NS, 5)
#define PASE_NP(NP) PASE_NS(NP, 0) PASE_NS(NP, 1) PASE_NS(NP, 2) PASE_NS(NP, 3)
        PASE_NP(1) PASE_NP(2) PASE_NP(3) PASE_NP(4)
#undef PASE_NP
#undef PASE_NS
#undef PASE_CASE
        // one lane per item (K <= 3): the whole reduction over C in one thread, 8 outputs per
        // thread, consecutive threads on consecutive items -- every store is a coalesced warp row
#define PASE_CASE1(NP, NS)                                                                        \
    case kShapeG1 + (NP - 1) * 4 + NS:                                                            \
        tile_items<NP, NS, 1>(vd, td_sh, i0 + first_warp * 32, nwarps * 32, i1, red_b, red_c, gate); \
        return;
#define PASE_NP1(NP) PASE_CASE1(NP, 0) PASE_CASE1(NP, 1) PASE_CASE1(NP, 2) PASE_CASE1(NP, 3)
        PASE_NP1(1) PASE_NP1(2) PASE_NP1(3) PASE_NP1(4)
#undef PASE_NP1
#undef PASE_CASE1
        // streaming regime: the spanning term staged by TMA bulk copies (one item per warp)
#define PASE_CASES(NP, NS)                                                                        \
    case kShapeStream + (NP - 1) * 4 + NS:                                                        \
        seq = tile_stream_items<NP, NS>(vd, td_sh, i0 + first_warp, nwarps, i1, dyn, seq, gate);  \
        return;
#define PASE_NPS(NP) PASE_CASES(NP, 1) PASE_CASES(NP, 2) PASE_CASES(NP, 3)
        PASE_NPS(1) PASE_NPS(2) PASE_NPS(3) PASE_NPS(4)
#undef PASE_NPS
#undef PASE_CASES
        // streaming regime: direct coalesced loads, the next item's rows bulk-prefetched into L2
#define PASE_CASEP(NP, NS)                                                                        \
    case kShapeStreamPF + (NP - 1) * 4 + NS:                                                      \
        tile_stream_pf<NP, NS>(vd, td_sh, i0 + first_warp, nwarps, i1, gate);                     \
        return;
#define PASE_NPP(NP) PASE_CASEP(NP, 1) PASE_CASEP(NP, 2) PASE_CASEP(NP, 3)
        PASE_NPP(1) PASE_NPP(2) PASE_NPP(3) PASE_NPP(4)
#undef PASE_NPP
#undef PASE_CASEP
#define PASE_CASE2(NS, LGG)                                                                       \
    case kShape2D + (NS - 1) * 4 + (LGG - 2): {                                                   \
        constexpr int G_ = 1 << LGG, GPW_ = 32 / G_;                                              \
        tile2_items<NS, G_>(vd, td_sh, i0 + first_warp * GPW_, nwarps * GPW_, i1, gate);          \
        return;                                                                                   \
    }
        PASE_CASE2(1, 2) PASE_CASE2(1, 3) PASE_CASE2(1, 4) PASE_CASE2(1, 5)
        PASE_CASE2(2, 2) PASE_CASE2(2, 3) PASE_CASE2(2, 4) PASE_CASE2(2, 5)
#undef PASE_CASE2
#define PASE_CASE2S(NP0, FORM, NB, NS2, LGG)                                                      \
    case kShape2S + ((NP0 - 1) * 4 + FORM) * 4 + (LGG - 2): {                                     \
        constexpr int G_ = 1 << LGG, GPW_ = 32 / G_;                                              \
        tile2s_items<NP0, NB, NS2, G_>(vd, td_sh, i0 + first_warp * GPW_, nwarps * GPW_, i1, gate); \
        return;                                                                                   \
    }
#define PASE_2S_G(NP0, FORM, NB, NS2)                                                             \
        PASE_CASE2S(NP0, FORM, NB, NS2, 2) PASE_CASE2S(NP0, FORM, NB, NS2, 3)                     \
        PASE_CASE2S(NP0, FORM, NB, NS2, 4) PASE_CASE2S(NP0, FORM, NB, NS2, 5)
#define PASE_2S_FORMS(NP0)                                                                        \
        PASE_2S_G(NP0, 0, 0, 0) PASE_2S_G(NP0, 1, 1, 0) PASE_2S_G(NP0, 2, 0, 1) PASE_2S_G(NP0, 3, 0, 2)
        PASE_2S_FORMS(1) PASE_2S_FORMS(2) PASE_2S_FORMS(3)
#undef PASE_2S_FORMS
#undef PASE_2S_G
#undef PASE_CASE2S
#define PASE_CASEC(NP0, FORM)                                                                     \
    case kShapeCta + (NP0 - 1) * 4 + FORM:                                                        \
        cta_items<NP0, FORM>(vd, td_sh, i0 + (first_warp >> 3), nwarps >> 3, i1, dyn, gate);      \
        return;
        PASE_CASEC(1, 0) PASE_CASEC(1, 1) PASE_CASEC(1, 2) PASE_CASEC(1, 3)
        PASE_CASEC(2, 0) PASE_CASEC(2, 1) PASE_CASEC(2, 2) PASE_CASEC(2, 3)
        PASE_CASEC(3, 0) PASE_CASEC(3, 1) PASE_CASEC(3, 2) PASE_CASEC(3, 3)
#undef PASE_CASEC
        default: {
            const int gpw = 32 >> vd.glog;
            generic_items(vd, tds_g, vd.glog, i0 + first_warp * gpw, nwarps * gpw, i1, gate);
        }
    }
}

// ---- per-vertex launch schedule (PASE_SCHEDULE=launches): one kernel per DP vertex ----
__global__ void __launch_bounds__(256, 2)
dp_fill_vertex(const VertexDesc* __restrict__ vds, const TermDesc* __restrict__ tds, int vtx) {
    __shared__ VertexDesc vd;
    __shared__ TermDesc td[kMaxTermsSh];
    __shared__ double red_b[8 * kTile];
    __shared__ int red_c[8 * kTile];
    extern __shared__ __align__(128) unsigned char dyn[];   // stream-tile rings (stream shapes only)
    if (threadIdx.x == 0) vd = vds[vtx];
    const int nt = min(vds[vtx].nterms, kMaxTermsSh);
    for (int t = threadIdx.x; t < nt; t += blockDim.x) td[t] = tds[vds[vtx].term0 + t];
    __syncthreads();
    if (stream_smem_shape(vd.shape)) stream_init(dyn);      // (the CTA tile uses the ring area's head)
    uint32_t seq = 0;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    run_shape(vd.shape, vd, td, tds, warp, nwarps, 0, vd.shape >= 0 ? vd.nitems : vd.nout, red_b, red_c, dyn, seq,
              Gate{nullptr, nullptr, 0, 0, nullptr, nullptr, 0, 0});
}

void launch_dp_vertex(const VertexDesc* vd_dev, const TermDesc* td_dev, int vertex,
                      const VertexDesc& vh, void* stream) {
    const int threads = 256;
    const int G = 1 << vh.glog;
    const int64_t units = vh.shape >= 0 ? vh.nitems : vh.nout;
    int64_t blocks = ((units * G << vh.wlog) + threads - 1) / threads;
    blocks = blocks > 148 * 8 ? 148 * 8 : (blocks < 1 ? 1 : blocks);
    const size_t dyn = (stream_smem_shape(vh.shape) || cta_shape(vh.shape)) ? kStreamSmemBytes : 0;
    if (dyn) {
        static bool attr = (cudaFuncSetAttribute(dp_fill_vertex, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)kStreamSmemBytes), true);
        (void)attr;
    }
    dp_fill_vertex<<<(unsigned)blocks, threads, dyn, (cudaStream_t)stream>>>(vd_dev, td_dev, vertex);
}

// ---- persistent schedule (default): one launch runs the whole elimination tree ----------
//   Tasks (item ranges of one vertex) are claimed in a static order computed on the host by
//   list-scheduling the task DAG on the CTAs of the grid with critical-path priority (a
//   topological order, so every task a CTA waits on is held by a running CTA: deadlock-free).
//   A claimed task waits until pending[vertex] -- the unfinished tasks of the vertex's
//   children -- reaches zero (relaxed spin, then fence.acq_rel: the PTX acquire pattern;
//   multi-GPU: ld.acquire.sys); its descriptors are fetched meanwhile.  A finished task decrements its parent's counter with an acq_rel RMW
//   after a CTA barrier, so a consumer that acquires the counter observes all child-table
//   writes (release sequence through pending[]).
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t smid() {
    uint32_t s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return s;
}
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
    // polling load: no acquire fence (an acquire invalidates the SM's L1 on every poll,
    // evicting the working set of the co-resident CTA)
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int atom_add_acq_rel(int32_t* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_add_release_gpu(int32_t* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_sys(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_sys(const int32_t* p) {
    int v;
    asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_add_release_sys(int32_t* p, int v) {
    asm volatile("red.release.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// a scheduler / group-barrier wait longer than the context's timeout (PASE_SPIN_TIMEOUT_MS,
// default 4 s; 0 = none) is reported through *err instead of hanging the GPU
__device__ __forceinline__ bool timed_out(uint64_t t0, uint64_t limit_ns) {
    return limit_ns != 0 && globaltimer() - t0 > limit_ns;
}

__device__ __forceinline__ void st_release(int32_t* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Claim modes.  STATIC (default): CTAs take tasks in the host's static topological order (a
// critical-path list schedule) and wait on each claimed task's pending counter.  READY QUEUE
// (single GPU, opt-in PASE_QUEUE=1; measured slower, profiles/r02_ab_queue.txt): only tasks whose
// dependencies are met are ever claimed -- the CTA that releases a
// vertex's last child task (its pending counter 1 -> 0) publishes all of the vertex's tasks into
// a ring (st.release of id + 1 per slot); CTAs claim ring slots with a fetch-and-add and wait
// only while the ring is empty.  No CTA ever sits on a claimed task whose children are still
// running, so ready work -- the critical path above all -- never queues behind blocked CTAs.
__global__ void __launch_bounds__(256, 2)
dp_persistent(const VertexDesc* __restrict__ vds, const TermDesc* __restrict__ tds,
              const TaskDesc* __restrict__ tasks, const int32_t* __restrict__ order, int ntasks,
              int32_t* __restrict__ sched, int32_t* __restrict__ err, Peers peers, CostArgs cost,
              int64_t* __restrict__ trace, uint64_t timeout_ns, int stream_smem, int32_t* __restrict__ ring,
              int32_t* __restrict__ ring_tail, int early_gate) {
    // sched: [0] claim counter / ring head (own 128-B line), [kSchedLine, +n) pending per vertex
    int32_t* head = sched;
    int32_t* pending = sched + kSchedLine;
    const bool queue = ring != nullptr;
    __shared__ int s_push;
    const bool multi = peers.world > 1;                     // peers: .sys scope
    __shared__ VertexDesc vd;
    __shared__ TermDesc td[kMaxTermsSh];
    __shared__ double red_b[8 * kTile];                     // latency-mode partial minima
    __shared__ int red_c[8 * kTile];
    __shared__ int s_task;
    __shared__ int s_warm;                                  // Gate::warm of the current task
    __shared__ int s_elect[2];                              // Gate::elect of the current task
    __shared__ CostSmem csm;                                // cost-table tasks
    extern __shared__ __align__(128) unsigned char dyn[];   // stream-tile rings (launched with them
    const bool stream = stream_smem != 0;                   // only when a vertex uses a stream shape)
    if (stream) stream_init(dyn);
    uint32_t seq = 0;                                       // this warp's staged-chunk sequence
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int cur = -1;
    // a group barrier that timed out (or any earlier failure of this solve) skips the DP: the
    // peers' tables may still be in use (the back-substitution skips its lookups too)
    if (ld_relaxed(err) != 0) return;
#if PASE_LAYOUT_PAD > 0
    // code-placement pad (build define; never executed: ntasks >= 0): shifts the placement of
    // the tile functions that follow in the kernel's code (placement moves the DP by
    // a few per cent between builds)
    if (ntasks < 0) {
#pragma unroll
        for (int k = 0; k < PASE_LAYOUT_PAD; ++k)
            asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_task)), "r"(k) : "memory");
    }
#endif
    for (;;) {
        int64_t t_claim = 0, t_start = 0;
        if (threadIdx.x == 0) {
            if (trace) t_claim = (int64_t)globaltimer();
            const int s = atomicAdd(head, 1);
            if (!queue) {
                s_task = s < ntasks ? order[s] : -1;
            } else if (s >= ntasks) {
                s_task = -1;
            } else {                                        // wait until slot s is published
                int v = ld_relaxed(ring + s);
                if (v == 0) {
                    const uint64_t t0 = globaltimer();
                    while ((v = ld_relaxed(ring + s)) == 0)
                        if (timed_out(t0, timeout_ns)) { atomicExch(err, 1); break; }
                }
                fence_acquire_gpu();                        // acquire: the children's tables
                s_task = v - 1;
                if (trace) t_start = (int64_t)globaltimer();
            }
        }
        __syncthreads();
        int task = s_task;
        if (task < 0) break;
        const TaskDesc tk = tasks[task];
        if (tk.vtx < 0) {                                   // cost-table chunk (no dependencies)
            const int c = -1 - tk.vtx;
            if (trace && threadIdx.x == 0) t_start = (int64_t)globaltimer();
            if (cost.enabled) cost_chunk(cost, c, csm);     // ends with a CTA barrier
            else __syncthreads();
            if (threadIdx.x == 0) {                         // its consumer's tasks may start
                int32_t* pc = pending + cost.chunks[c].consumer;
                if (multi) red_add_release_sys(pc, -1);
                else atom_add_acq_rel(pc, -1);
                if (trace) {
                    int64_t* tr = trace + (int64_t)kTraceWords * task;
                    tr[0] = ((int64_t)smid() << 32) | (uint32_t)tk.vtx;
                    tr[1] = t_claim;
                    tr[2] = t_start;
                    tr[3] = tr[4] = tr[5] = (int64_t)globaltimer();
                }
            }
            continue;
        }
        if (tk.vtx != cur) {                                // descriptors: static, fetch now
            stage_struct(&vd, vds + tk.vtx);                // one 4-B word per thread: one round of loads
            __syncthreads();
            const int nt = min(vd.nterms, kMaxTermsSh);
            for (int k = threadIdx.x; k < nt; k += blockDim.x) td[k] = tds[vd.term0 + k];
            cur = tk.vtx;
        }
        if (queue || early_gate) {
            // queue: ready by construction.  early gate: every warp waits at its tile's gate,
            // after its work-item decode (the gate fences; the stream tiles add the proxy fence).
            // early_gate bit 1: a task whose children still run warms its tile first (Gate::warm)
            if (early_gate && threadIdx.x == 0) {
                if (trace) t_start = (int64_t)globaltimer();
                s_elect[0] = s_elect[1] = 0;
                s_warm = !queue && (early_gate & 2) && !stream_smem_shape(vd.shape) &&
                         (multi ? ld_relaxed_sys(pending + tk.vtx) : ld_relaxed(pending + tk.vtx)) != 0;
            }
        } else if (threadIdx.x == 0) {                      // wait for the children's tasks
            int32_t* pv = pending + tk.vtx;
            if ((multi ? ld_relaxed_sys(pv) : ld_relaxed(pv)) != 0) {
                unsigned bo = 32;
                const uint64_t t0 = globaltimer();
                while ((multi ? ld_relaxed_sys(pv) : ld_relaxed(pv)) != 0) {
                    if (PASE_SPIN_SLEEP) {
                        __nanosleep(bo);
                        bo = bo < 256 ? 2 * bo : 256;
                    }
                    if (timed_out(t0, timeout_ns)) { atomicExch(err, 1); s_task = -1; break; }
                }
            }
            if (multi) (void)ld_acquire_sys(pv);
            else if (PASE_ACQ_FENCE) fence_acquire_gpu();      // relaxed read + fence = acquire pattern
            else (void)ld_acquire(pv);
            // the stream tile reads child tables through the async proxy (TMA): order the
            // acquired generic-proxy writes before those reads
            if (stream_smem_shape(vd.shape)) fence_proxy_async_global();
            if (trace) t_start = (int64_t)globaltimer();
        }
        __syncthreads();
        task = s_task;
        if (task < 0) break;                                // timed out (reported via *err)
        // wave-tail tasks (schedule.cpp) run the vertex's tile with wider lane groups: every
        // tile family encodes log2(G) - 2 in the shape's low 2 bits
        const int shape = tk.glog > 0 ? ((vd.shape & ~3) | (tk.glog - 2)) : vd.shape;
        const Gate gate{(early_gate && !queue) ? pending + tk.vtx : nullptr, err, timeout_ns, multi ? 1 : 0,
                        (early_gate & 4) ? s_elect : nullptr,
                        trace ? trace + (int64_t)kTraceWords * task + kTraceTaskWords : nullptr,
                        ((early_gate & 16) || ((early_gate & 8) && shape >= 0 && shape < kShape2D)) ? 1 : 0,
                        (early_gate && !queue) ? s_warm : 0};
        if (gate.stamp && (threadIdx.x & 31) == 0) gate.stamp[2 * warp] = gate.stamp[2 * warp + 1] = 0;
        run_shape(shape, vd, td, tds, warp, nwarps, tk.i0, tk.i1, red_b, red_c, dyn, seq, gate);
        int64_t t_comp = 0, t_sync = 0;
        if (trace && threadIdx.x == 0) t_comp = (int64_t)globaltimer();
        __syncthreads();                                    // task's stores precede the release
        if (queue) {
            if (threadIdx.x == 0) {
                if (trace) t_sync = (int64_t)globaltimer();
                s_push = -1;
                if (vd.parent >= 0 && atom_add_acq_rel(pending + vd.parent, -1) == 1) {
                    // last child task: the parent is ready -- reserve its slots
                    const int nt = vds[vd.parent].ntasks;
                    s_push = atomicAdd(ring_tail, nt);
                }
            }
            __syncthreads();
            if (s_push >= 0) {                              // publish the parent's tasks
                const int t0 = vds[vd.parent].task0, nt = vds[vd.parent].ntasks;
                for (int k = threadIdx.x; k < nt; k += blockDim.x) st_release(ring + s_push + k, t0 + k + 1);
            }
            if (threadIdx.x == 0 && trace) {
                int64_t* tr = trace + (int64_t)kTraceWords * task;
                tr[0] = ((int64_t)smid() << 32) | (uint32_t)tk.vtx;
                tr[1] = t_claim;
                tr[2] = t_start;
                tr[3] = t_comp;
                tr[4] = t_sync;
                tr[5] = (int64_t)globaltimer();
            }
            continue;
        }
        if (threadIdx.x == 0) {
            if (trace) t_sync = (int64_t)globaltimer();
            if (vd.parent >= 0) {
                if (vd.bcast & 1) {                         // every rank's copy of the parent waits
                    for (int q = 0; q < peers.world; ++q) red_add_release_sys(peers.pending[q] + vd.parent, -1);
                } else if (multi) {
                    red_add_release_sys(pending + vd.parent, -1);
                } else if (PASE_REL_RED || (early_gate & 32)) {   // runtime A/B: PASE_REL_RED=1
                    red_add_release_gpu(pending + vd.parent, -1);
                } else {
                    atom_add_acq_rel(pending + vd.parent, -1);
                }
            }
            if (trace) {                                    // PASE_TRACE: per-task timeline
                int64_t* tr = trace + (int64_t)kTraceWords * task;
                tr[0] = ((int64_t)smid() << 32) | (uint32_t)tk.vtx;
                tr[1] = t_claim;
                tr[2] = t_start;
                tr[3] = t_comp;
                tr[4] = t_sync;
                tr[5] = (int64_t)globaltimer();
            }
        }
    }
}

void launch_dp_persistent(const VertexDesc* vd_dev, const TermDesc* td_dev, const TaskDesc* tasks_dev,
                          const int32_t* order_dev, int ntasks, int32_t* sched_dev, int32_t* err_dev,
                          const Peers& peers, const CostArgs& cost, int nblocks, int64_t* trace_dev,
                          uint64_t timeout_ns, bool stream_tiles, int32_t* ring, int32_t* ring_tail,
                          int early_gate, void* stream) {
    const size_t dyn = stream_tiles ? kStreamSmemBytes : 0;
    dp_persistent<<<(unsigned)nblocks, 256, dyn, (cudaStream_t)stream>>>(vd_dev, td_dev, tasks_dev, order_dev,
                                                                           ntasks, sched_dev, err_dev, peers,
                                                                           cost, trace_dev, timeout_ns, (int)dyn,
                                                                           ring, ring_tail, early_gate);
}

// Group barrier between the ranks of a multi-GPU search (before and after the DP): every
// rank adds 1 to every rank's arrival counter (release.sys, peer atomics) and waits for
// epoch * world arrivals on its own.  bar[0] = arrivals, bar[kSchedLine] = local epoch.
__global__ void rank_barrier(Peers peers, int32_t* bar, int32_t* err, uint64_t timeout_ns) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int e = bar[kSchedLine] + 1;
    bar[kSchedLine] = e;
    for (int q = 0; q < peers.world; ++q) red_add_release_sys(peers.bar[q], 1);
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(bar) < e * peers.world) {
        __nanosleep(128);
        if (timed_out(t0, timeout_ns)) { atomicExch(err, 2); break; }
    }
}

void launch_rank_barrier(const Peers& peers, int32_t* bar_dev, int32_t* err_dev, uint64_t timeout_ns, void* stream) {
    rank_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(peers, bar_dev, err_dev, timeout_ns);
}

int persistent_blocks_per_sm() {
    // sized with the stream-tile rings reserved, so a context with stream shapes and one without
    // get the same grid (2 CTAs per SM: registers bound it either way)
    static bool attr = (cudaFuncSetAttribute(dp_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kStreamSmemBytes), true);
    (void)attr;
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dp_persistent, 256, kStreamSmemBytes);
    return nb;
}

// =====================================================================================
// K3: back-substitution: phi*(sigma_i) = A(i)[index(phi*|D(i))].  D(i) holds
// only ancestors of i in the elimination tree, so all vertices of one "back level"
// (1 + max back level over D(i); the root is level 0) are independent: one CTA walks the
// levels, a thread per vertex, choices in shared memory.  The records are staged once with
// 16-byte loads all in flight; a vertex's index is a branch-free sum over its (padded)
// dependent list, so each level costs one dependent A(i) load (L2) plus a barrier.
// =====================================================================================
__global__ void __launch_bounds__(256)
backtrack_kernel(const BtDesc* __restrict__ bt_g, const int32_t* __restrict__ bt_off_g, int nlev, int n,
                 const double* __restrict__ root_T, int32_t* __restrict__ choice, double* __restrict__ total,
                 int32_t* __restrict__ err, char* __restrict__ host_out, int smem_records) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // [choices: n int32][level offsets: nlev + 1][records (smem_records)]
    int32_t* ch = reinterpret_cast<int32_t*>(smem_raw);
    int32_t* off = ch + n;
    BtDesc* sh_bt = reinterpret_cast<BtDesc*>(smem_raw + (((size_t)n + nlev + 1) * 4 + 15) / 16 * 16);
    const BtDesc* bt = smem_records ? sh_bt : bt_g;
    if (smem_records) {                                     // 16-B words, 4 loads in flight per thread
        static_assert(sizeof(BtDesc) % 16 == 0, "record copy in 16-B words");
        const int words = (int)(sizeof(BtDesc) / 16) * n;
        const uint4* src = reinterpret_cast<const uint4*>(bt_g);
        uint4* dst = reinterpret_cast<uint4*>(sh_bt);
        for (int k0 = threadIdx.x; k0 < words; k0 += 4 * blockDim.x) {
            uint4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k0 + u * (int)blockDim.x < words) w[u] = src[k0 + u * blockDim.x];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k0 + u * (int)blockDim.x < words) dst[k0 + u * blockDim.x] = w[u];
        }
    }
    for (int k = threadIdx.x; k <= nlev; k += blockDim.x) off[k] = bt_off_g[k];
    for (int v = threadIdx.x; v < n; v += blockDim.x) ch[v] = 0;   // padding entries read ch[0]
    // a DP that reported an error (scheduler time-out) left tables unfinished: no lookups
    __shared__ int s_bad;
    if (threadIdx.x == 0) s_bad = 0;
    const int failed = *err;
    __syncthreads();
    for (int lev = 0; lev < (failed ? 0 : nlev); ++lev) {
        for (int k = off[lev] + threadIdx.x; k < off[lev + 1]; k += blockDim.x) {
            const BtDesc& d = bt[k];
            int c = 0;                                      // K = 1: A(i) is not stored
            if (d.K > 1) {
                int64_t idx = 0;
#pragma unroll
                for (int a = 0; a < kMaxDep; ++a) idx += (int64_t)ch[d.dep[a]] * d.stride[a];
                c = d.A[idx];
                if (c >= d.K) { s_bad = 1; c = 0; }        // no finite candidate: report, stay in range
            }
            ch[d.node] = c;
        }
        __syncthreads();
    }
    if (s_bad && threadIdx.x == 0) *err = 3;
    __syncthreads();
    // results: the device block (total | err | pad | choice[n]) and, when given, the same
    // layout straight into the caller's pinned host block (mapped: no copy-engine round trip)
    int32_t* hc = host_out ? reinterpret_cast<int32_t*>(host_out + 16) : nullptr;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        const int32_t c = failed ? 0 : ch[v];
        choice[v] = c;
        if (hc) hc[v] = c;
    }
    if (threadIdx.x == 0) {
        const double t = failed ? 0.0 : root_T[0];          // f(|V|, ∅); unwritten after a failure
        *total = t;
        if (host_out) {
            *reinterpret_cast<double*>(host_out) = t;
            *reinterpret_cast<int32_t*>(host_out + 8) = *err;
        }
    }
}

void launch_backtrack(const BtDesc* bt_dev, const int32_t* bt_off_dev, int nlev, int n,
                      const double* root_T, int32_t* choice_dev, double* total_dev, int32_t* err_dev,
                      void* host_out, void* stream) {
    const size_t head = (((size_t)n + nlev + 1) * 4 + 15) / 16 * 16;
    const size_t with_rec = head + sizeof(BtDesc) * (size_t)n;
    // opt-in dynamic shared memory: the device maximum minus the kernel's static shared memory
    static int max_dyn = [] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, backtrack_kernel);
        v -= (int)fa.sharedSizeBytes;
        cudaFuncSetAttribute(backtrack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, v);
        return v;
    }();
    const bool rec = with_rec <= (size_t)max_dyn;
    backtrack_kernel<<<1, 256, rec ? with_rec : head, (cudaStream_t)stream>>>(
        bt_dev, bt_off_dev, nlev, n, root_T, choice_dev, total_dev, err_dev, (char*)host_out, rec ? 1 : 0);
}

}  // namespace pase
