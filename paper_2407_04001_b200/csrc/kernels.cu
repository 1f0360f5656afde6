// kernels.cu -- sm_100a kernels of the PaSE hot path.
//   K1 cost_tables   (row a5): L_v[C] = t_l(v, C, r), W_e = r * t_x (Eq. 1)
//   K2 dp_fill       (row a6): Eq. 4 / Fig. 5 lines 8-20
//   K3 backtrack     (row a7): back-substitution from sigma_|V|.cfg
// Bit-exactness rules: every fp64 op is an explicit IEEE RN intrinsic
// (__dadd_rn / __dmul_rn / __ddiv_rn / __ull2double_rn), never contracted to FMA; the sum
// over the terms of Eq. 4 follows the canonical order L, W_e (E> order), T_j (rank order);
// ties in the min over C keep the lowest C (strict <, Fig. 5 line 17).
#include <cuda_runtime.h>

#include <cstdint>

#include "pase_internal.h"

namespace pase {

// =====================================================================================
// K1: cost tables
// =====================================================================================
__device__ __forceinline__ double d_allreduce(int64_t g, int64_t bytes) {
    // ring all-reduce over g participants: 2(g-1)B/g (DESIGN reading J)
    if (g <= 1) return 0.0;
    return __ddiv_rn(__ull2double_rn((unsigned long long)(2 * (g - 1) * bytes)), __ll2double_rn(g));
}

// t_l (DESIGN reading I): FLOPs of one (equal) shard + r * (reduction AR + gradient AR + halo)
__device__ double d_layer_cost(const pase_node& x, const int32_t* c, double r) {
    int64_t s[kMaxDims];
    for (int k = 0; k < x.n_dims; ++k) s[k] = x.size[k] / c[k];
    int64_t compute = x.flops_per_point;
    for (int k = 0; k < x.n_dims; ++k)
        if (x.flop_dims_mask == 0u || (x.flop_dims_mask >> k & 1u)) compute *= s[k];
    uint32_t out_m = 0, w_m = 0;
    int64_t out_elems = 1, w_elems = 1;
    for (int a = 0; a < x.n_out_axes; ++a) { out_m |= 1u << x.out_axes[a]; out_elems *= s[x.out_axes[a]]; }
    for (int a = 0; a < x.n_w_axes; ++a) { w_m |= 1u << x.w_axes[a]; w_elems *= s[x.w_axes[a]]; }
    int64_t g_red = 1, g_grad = 1;
    for (int k = 0; k < x.n_dims; ++k) {
        if (!(out_m >> k & 1u)) g_red *= c[k];
        if (!(w_m >> k & 1u)) g_grad *= c[k];
    }
    const int64_t out_bytes = (int64_t)x.elem_bytes * out_elems;
    const int64_t w_bytes = x.n_w_axes > 0 ? (int64_t)x.elem_bytes * w_elems : 0;
    if (x.n_w_axes == 0) g_grad = 1;
    int64_t halo = 0;
    for (int q = 0; q < x.n_halo; ++q) {
        const int h = x.halo_spatial[q], f = x.halo_filter[q];
        if (c[h] > 1 && x.size[f] > 1) {
            int64_t face = 1;
            for (int a = 0; a < x.n_out_axes; ++a)
                if (x.out_axes[a] != h) face *= s[x.out_axes[a]];
            halo += 2 * (int64_t)x.elem_bytes * (x.size[f] - 1) * face;
        }
    }
    double comm = d_allreduce(g_red, out_bytes);
    comm = __dadd_rn(comm, d_allreduce(g_grad, w_bytes));
    comm = __dadd_rn(comm, __ull2double_rn((unsigned long long)halo));
    return __dadd_rn(__ull2double_rn((unsigned long long)compute), __dmul_rn(r, comm));
}

// t_x bytes (DESIGN reading K): nested aligned layouts; per output axis of the producer
// held = ext / c_src, need = ceil(ext / c_dst[map]) (ext if unmapped), overlap = min.
__device__ int64_t d_transfer_bytes(const pase_node& u, const int32_t* cu, const int32_t* cv,
                                    const int32_t* amap) {
    int64_t need = 1, ov = 1;
    for (int a = 0; a < u.n_out_axes; ++a) {
        const int du = u.out_axes[a];
        const int64_t ext = u.size[du];
        const int64_t held = ext / cu[du];
        const int64_t nd = amap[a] < 0 ? ext : (ext + cv[amap[a]] - 1) / cv[amap[a]];
        need *= nd;
        ov *= nd < held ? nd : held;
    }
    return 2 * (int64_t)u.elem_bytes * (need - ov);
}

__global__ void __launch_bounds__(256)
cost_tables_kernel(const pase_node* __restrict__ nodes, const int32_t* __restrict__ K,
                   const int64_t* __restrict__ cfg_off, const int32_t* __restrict__ cfg,
                   const int64_t* __restrict__ loff, int n, const EdgeDesc* __restrict__ edges, int m,
                   const int64_t* __restrict__ item_off, int64_t total, double r,
                   double* __restrict__ L, double* __restrict__ W) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int lo = 0, hi = n + m;                       // item_off[lo] <= idx < item_off[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (item_off[mid] <= idx) lo = mid; else hi = mid;
        }
        const int64_t local = idx - item_off[lo];
        if (lo < n) {
            const int v = lo;
            L[loff[v] + local] = d_layer_cost(nodes[v], cfg + (cfg_off[v] + local) * kMaxDims, r);
        } else {
            const EdgeDesc& e = edges[lo - n];
            // W_e row = config of the later-ranked endpoint, column = earlier endpoint (stride 1)
            const int early = e.later_is_src ? e.dst : e.src;
            const int64_t row = local / K[early], col = local % K[early];
            const int64_t cs = e.later_is_src ? row : col, cd = e.later_is_src ? col : row;
            const int64_t b = d_transfer_bytes(nodes[e.src], cfg + (cfg_off[e.src] + cs) * kMaxDims,
                                               cfg + (cfg_off[e.dst] + cd) * kMaxDims, e.axis_map);
            W[e.woff + local] = __dmul_rn(r, __ull2double_rn((unsigned long long)b));
        }
    }
}

void launch_cost_tables(const pase_node* nodes_dev, const int32_t* K_dev, const int64_t* cfg_off_dev,
                        const int32_t* cfg_dev, const int64_t* loff_dev, int n,
                        const EdgeDesc* edges_dev, int m, const int64_t* item_off_dev,
                        int64_t total, double r, double* L_dev, double* W_dev, void* stream) {
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    cost_tables_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
        nodes_dev, K_dev, cfg_off_dev, cfg_dev, loff_dev, n, edges_dev, m, item_off_dev, total, r,
        L_dev, W_dev);
}

// =====================================================================================
// K2: DP fill, v1 (generic): a lane group of g = pow2 >= min(K, 32) lanes per output phi.
// =====================================================================================
template <int NT>
__global__ void __launch_bounds__(256)
dp_fill_kernel(const VertexDesc* __restrict__ vds, const TermDesc* __restrict__ tds, int vtx, int glog) {
    __shared__ VertexDesc vd;
    __shared__ TermDesc td[NT];
    if (threadIdx.x == 0) vd = vds[vtx];
    for (int t = threadIdx.x; t < NT; t += blockDim.x) td[t] = tds[vds[vtx].term0 + t];
    __syncthreads();
    const int g = 1 << glog;
    const int lane = threadIdx.x & (g - 1);
    const int gpw = 32 >> glog;                           // lane groups per warp
    const int sub = (threadIdx.x & 31) >> glog;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // warp-uniform loop (every lane reaches the shuffles); phi >= nout lanes idle
    for (int64_t base = warp * gpw; base < vd.nout; base += nwarps * gpw) {
        const int64_t phi = base + sub;
        const int K = phi < vd.nout ? vd.K : 0;
        // mixed-radix decode of phi over D(i) (ascending rank, lowest fastest)
        int64_t off[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) off[t] = 0;
        int64_t rem = phi < vd.nout ? phi : 0;
        for (int q = 0; q < vd.m; ++q) {
            const int64_t c = rem % vd.radix[q];
            rem /= vd.radix[q];
#pragma unroll
            for (int t = 0; t < NT; ++t) off[t] += c * td[t].stride[q];
        }
        const double* ptr[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) ptr[t] = td[t].base + off[t];
        double best = __longlong_as_double(0x7ff0000000000000ll);   // +inf
        int bestC = 0x7fffffff;
        for (int C = lane; C < K; C += g) {
            double cost = __ldg(ptr[0] + C);
#pragma unroll
            for (int t = 1; t < NT; ++t) cost = __dadd_rn(cost, __ldg(ptr[t] + C));
            if (cost < best) { best = cost; bestC = C; }          // strict <: lowest C in lane
        }
        // combine lanes: smaller cost, or equal cost and smaller C
        for (int o = g >> 1; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bestC, o);
            if (ob < best || (ob == best && oc < bestC)) { best = ob; bestC = oc; }
        }
        if (lane == 0 && K > 0) {
            vd.T[phi] = best;
            vd.A[phi] = (uint16_t)bestC;
        }
    }
}

// Fallback for vertices with more than kMaxTermsReg summands: offsets recomputed per candidate.
__global__ void __launch_bounds__(256)
dp_fill_kernel_many(const VertexDesc* __restrict__ vds, const TermDesc* __restrict__ tds, int vtx, int glog) {
    const VertexDesc& vd = vds[vtx];
    const int g = 1 << glog;
    const int lane = threadIdx.x & (g - 1);
    const int gpw = 32 >> glog;
    const int sub = (threadIdx.x & 31) >> glog;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * gpw; base < vd.nout; base += nwarps * gpw) {
        const int64_t phi = base + sub;
        const int K = phi < vd.nout ? vd.K : 0;
        int32_t c[kMaxDep];
        int64_t rem = phi < vd.nout ? phi : 0;
        for (int q = 0; q < vd.m; ++q) { c[q] = (int32_t)(rem % vd.radix[q]); rem /= vd.radix[q]; }
        double best = __longlong_as_double(0x7ff0000000000000ll);
        int bestC = 0x7fffffff;
        for (int C = lane; C < K; C += g) {
            double cost = 0.0;
            for (int t = 0; t < vd.nterms; ++t) {
                const TermDesc& d = tds[vd.term0 + t];
                int64_t off = 0;
                for (int q = 0; q < vd.m; ++q) off += (int64_t)c[q] * d.stride[q];
                const double x = __ldg(d.base + off + C);
                cost = t == 0 ? x : __dadd_rn(cost, x);
            }
            if (cost < best) { best = cost; bestC = C; }
        }
        for (int o = g >> 1; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bestC, o);
            if (ob < best || (ob == best && oc < bestC)) { best = ob; bestC = oc; }
        }
        if (lane == 0 && K > 0) {
            vd.T[phi] = best;
            vd.A[phi] = (uint16_t)bestC;
        }
    }
}

void launch_dp_vertex(const VertexDesc* vd_dev, const TermDesc* td_dev, int vertex,
                      const VertexDesc& vh, void* stream) {
    int glog = 0;
    while ((1 << glog) < vh.K && glog < 5) ++glog;
    const int threads = 256;
    int64_t blocks = (vh.nout * (1ll << glog) + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    cudaStream_t s = (cudaStream_t)stream;
    switch (vh.nterms) {
#define PASE_NT(N) case N: dp_fill_kernel<N><<<(unsigned)blocks, threads, 0, s>>>(vd_dev, td_dev, vertex, glog); break;
        PASE_NT(1) PASE_NT(2) PASE_NT(3) PASE_NT(4) PASE_NT(5) PASE_NT(6) PASE_NT(7) PASE_NT(8)
#undef PASE_NT
        default: dp_fill_kernel_many<<<(unsigned)blocks, threads, 0, s>>>(vd_dev, td_dev, vertex, glog);
    }
}

// =====================================================================================
// K3: back-substitution: phi*(sigma_i) = A(i)[index(phi*|D(i))], i = |V|..1
// =====================================================================================
__global__ void backtrack_kernel(const int32_t* __restrict__ sigma, const int32_t* __restrict__ dep_off,
                                 const int32_t* __restrict__ dep_ids, const VertexDesc* __restrict__ vds,
                                 int n, int32_t* __restrict__ choice, double* __restrict__ total) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    *total = vds[n - 1].T[0];                              // f(|V|, ∅)
    for (int i = n - 1; i >= 0; --i) {
        int64_t idx = 0, stride = 1;
        for (int a = dep_off[i]; a < dep_off[i + 1]; ++a) {
            idx += (int64_t)choice[dep_ids[a]] * stride;
            stride *= vds[i].radix[a - dep_off[i]];
        }
        choice[sigma[i]] = vds[i].A[idx];
    }
}

void launch_backtrack(const int32_t* sigma_dev, const int32_t* dep_off_dev, const int32_t* dep_ids_dev,
                      const VertexDesc* vd_dev, int n, int32_t* choice_dev, double* total_dev,
                      void* stream) {
    backtrack_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(sigma_dev, dep_off_dev, dep_ids_dev, vd_dev, n,
                                                         choice_dev, total_dev);
}

}  // namespace pase
