// eval.cu -- Eq. 1 on the GPU.
//   K4 eval_kernel   cost(G, phi) = sum_v t_l(v, phi(v), r) + sum_e r t_x(e, phi)  (Eq. 1)
//                    for a batch of given strategies (re-evaluation of phi*, data-parallel and
//                    other reference strategies: Table 2 checks).
//   K5 brute_kernel  the exhaustive search the DP replaces: min over all prod_v K_v
//                    strategies; by Theorem 1 its minimum equals the DP
//                    total, which makes it a check of the whole DP at sizes no CPU brute force
//                    reaches (~1e10-1e12 strategies).
// The sum is Eq. 1 written out in one fixed order -- 0 + L_v over node ids, then + W_e over
// edge ids, each an IEEE RN add (__dadd_rn, never contracted) -- and strategy indices are
// mixed radix over node ids, node 0 fastest; the minimum keeps the lowest index among equal
// costs.  Same definition as the CPU brute force of the test oracle, so the two agree bit
// for bit (tests/test_gpu_parity.py); no code is shared.
#include <cuda_runtime.h>

#include <cstdint>

#include "pase_internal.h"

namespace pase {

// W_e element for (c_row, c_col): W[off + c_row * kcol + c_col]; row = later-ranked endpoint
// (the DP layout of W_e).

__device__ __forceinline__ bool lex_less(double b, uint64_t i, double ob, uint64_t oi) {
    return ob < b || (ob == b && oi < i);
}

__global__ void __launch_bounds__(128)
eval_kernel(int n, int m, const int64_t* __restrict__ loff, const double* __restrict__ L,
            const EvalEdge* __restrict__ ed, const double* __restrict__ W,
            const int32_t* __restrict__ strat, int64_t ns, double* __restrict__ out) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ns) return;
    const int32_t* c = strat + s * n;
    double acc = 0.0;
    for (int v = 0; v < n; ++v) acc = __dadd_rn(acc, __ldg(L + loff[v] + c[v]));
    for (int e = 0; e < m; ++e) {
        const EvalEdge x = ed[e];
        acc = __dadd_rn(acc, __ldg(W + x.off + (int64_t)c[x.row] * x.kcol + c[x.col]));
    }
    out[s] = acc;
}

// One thread per contiguous index range [x0, x1): decode x0 once, then an odometer (node 0
// fastest).  The digits live in shared memory ([node][thread], conflict-free), so any edge can
// index them.
__global__ void __launch_bounds__(128)
brute_kernel(int n, int m, const int32_t* __restrict__ K, const int64_t* __restrict__ loff,
             const double* __restrict__ L, const EvalEdge* __restrict__ ed, const double* __restrict__ W,
             uint64_t total, uint64_t per, double* __restrict__ blk_b, uint64_t* __restrict__ blk_i) {
    extern __shared__ __align__(16) unsigned char smem[];
    EvalEdge* se = reinterpret_cast<EvalEdge*>(smem);
    int64_t* sl = reinterpret_cast<int64_t*>(se + m);
    int32_t* sk = reinterpret_cast<int32_t*>(sl + n);
    int32_t* cs = sk + n;                                   // [n][blockDim.x]
    for (int e = threadIdx.x; e < m; e += blockDim.x) se[e] = ed[e];
    for (int v = threadIdx.x; v < n; v += blockDim.x) { sl[v] = loff[v]; sk[v] = K[v]; }
    __syncthreads();
    const int B = blockDim.x, t = threadIdx.x;
    const uint64_t gt = (uint64_t)blockIdx.x * B + t;
    const uint64_t x0 = gt * per;
    const uint64_t x1 = x0 + per < total ? x0 + per : total;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint64_t bi = ~0ull;
    if (x0 < total) {
        uint64_t r = x0;
        for (int v = 0; v < n; ++v) { cs[v * B + t] = (int32_t)(r % (uint64_t)sk[v]); r /= (uint64_t)sk[v]; }
        for (uint64_t x = x0; x < x1; ++x) {
            double acc = 0.0;
            for (int v = 0; v < n; ++v) acc = __dadd_rn(acc, __ldg(L + sl[v] + cs[v * B + t]));
            for (int e = 0; e < m; ++e) {
                const EvalEdge& y = se[e];
                acc = __dadd_rn(acc, __ldg(W + y.off + (int64_t)cs[y.row * B + t] * y.kcol + cs[y.col * B + t]));
            }
            if (acc < best) { best = acc; bi = x; }          // strict <: first index in the range
            for (int v = 0; v < n; ++v) {                   // odometer, node 0 fastest
                const int c = cs[v * B + t] + 1;
                if (c < sk[v]) { cs[v * B + t] = c; break; }
                cs[v * B + t] = 0;
            }
        }
    }
    // (cost, index) lexicographic minimum over the block
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (lex_less(best, bi, ob, oi)) { best = ob; bi = oi; }
    }
    __shared__ double wb[32];
    __shared__ uint64_t wi[32];
    __syncthreads();                                        // cs no longer read
    if ((t & 31) == 0) { wb[t >> 5] = best; wi[t >> 5] = bi; }
    __syncthreads();
    if (t == 0) {
        for (int w = 1; w < (B >> 5); ++w)
            if (lex_less(best, bi, wb[w], wi[w])) { best = wb[w]; bi = wi[w]; }
        blk_b[blockIdx.x] = best;
        blk_i[blockIdx.x] = bi;
    }
}

__global__ void __launch_bounds__(1024)
brute_reduce(int nb, const double* __restrict__ blk_b, const uint64_t* __restrict__ blk_i,
             double* __restrict__ out_b, uint64_t* __restrict__ out_i) {
    double best = __longlong_as_double(0x7ff0000000000000ll);
    uint64_t bi = ~0ull;
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
        if (lex_less(best, bi, blk_b[k], blk_i[k])) { best = blk_b[k]; bi = blk_i[k]; }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (lex_less(best, bi, ob, oi)) { best = ob; bi = oi; }
    }
    __shared__ double wb[32];
    __shared__ uint64_t wi[32];
    if ((threadIdx.x & 31) == 0) { wb[threadIdx.x >> 5] = best; wi[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (lex_less(best, bi, wb[w], wi[w])) { best = wb[w]; bi = wi[w]; }
        *out_b = best;
        *out_i = bi;
    }
}

void launch_eval(int n, int m, const int64_t* loff_dev, const double* L_dev, const EvalEdge* ed_dev,
                 const double* W_dev, const int32_t* strat_dev, int64_t ns, double* out_dev, void* stream) {
    if (ns <= 0) return;
    eval_kernel<<<(unsigned)((ns + 127) / 128), 128, 0, (cudaStream_t)stream>>>(n, m, loff_dev, L_dev, ed_dev,
                                                                               W_dev, strat_dev, ns, out_dev);
}

size_t brute_smem_bytes(int n, int m) {
    return sizeof(EvalEdge) * (size_t)m + (sizeof(int64_t) + sizeof(int32_t)) * (size_t)n +
           sizeof(int32_t) * (size_t)n * kBruteThreads;
}

int launch_brute(int n, int m, const int32_t* K_dev, const int64_t* loff_dev, const double* L_dev,
                 const EvalEdge* ed_dev, const double* W_dev, uint64_t total, int nblocks,
                 double* blk_b, uint64_t* blk_i, double* out_b, uint64_t* out_i, void* stream) {
    const size_t smem = brute_smem_bytes(n, m);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(brute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    const uint64_t threads = (uint64_t)nblocks * kBruteThreads;
    const uint64_t per = (total + threads - 1) / threads;
    brute_kernel<<<(unsigned)nblocks, kBruteThreads, smem, (cudaStream_t)stream>>>(n, m, K_dev, loff_dev, L_dev, ed_dev,
                                                                                  W_dev, total, per, blk_b, blk_i);
    brute_reduce<<<1, 1024, 0, (cudaStream_t)stream>>>(nblocks, blk_b, blk_i, out_b, out_i);
    return 0;
}

}  // namespace pase
