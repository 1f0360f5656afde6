// capi.cu -- the C ABI of include/pase.h: context lifecycle, device memory, the solve
// schedule recorded once as a CUDA graph (cost tables -> [group barrier] -> persistent DP
// over the elimination tree -> [group barrier] -> back-substitution -> D2H of the strategy),
// multi-GPU peer connection, and the introspection hooks.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "pase_internal.h"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx (no-ops untraced)

namespace {
struct NvtxRange {               // RAII NVTX push/pop (tracing)
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using pase::EdgeDesc;
using pase::Plan;
using pase::TermDesc;
using pase::VertexDesc;

struct pase_ctx {
    Plan P;
    pase_machine mach{};
    std::string err;
    int dev = 0;
    int world = 1, rank = 0;
    bool virtual_ranks = false;             // all ranks of the group share this device
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool async_pools = false;               // pools from the library's stream-ordered mempool
    bool big_pinned = false;                // h_total came from cudaMallocHost, not the cache
    void* stage_block = nullptr;            // pinned upload image, returned after create's sync
    std::vector<cudaStream_t> aux;          // fork streams (per-vertex launch schedule)
    // pool 1: inputs, cost tables, DP tables (T/A written by peers), descriptors
    void* pool = nullptr;
    size_t pool_bytes = 0;
    pase_node* d_nodes = nullptr;
    int32_t* d_K = nullptr;
    int64_t* d_cfg_off = nullptr;
    int32_t* d_cfg = nullptr;
    int64_t* d_loff = nullptr;
    EdgeDesc* d_edges = nullptr;
    pase::CostChunk* d_chunks = nullptr;
    int nchunks = 0;
    double* d_L = nullptr;
    double* d_W = nullptr;
    double* d_T = nullptr;
    uint16_t* d_A = nullptr;
    VertexDesc* d_vd = nullptr;
    TermDesc* d_td = nullptr;
    pase::BtDesc* d_bt = nullptr;
    int32_t* d_bt_off = nullptr;
    int nbtlev = 0;                         // back-substitution levels
    int32_t* d_choice = nullptr;
    double* d_total = nullptr;
    int32_t* d_err = nullptr;               // scheduler time-out flag (inside the output block)
    // pool 2: scheduler (pending counters written by peers), tasks, claim order, trace
    void* pool2 = nullptr;
    size_t pool2_bytes = 0;
    int32_t* d_sched = nullptr;             // [0] claim counter / ring head | [kSchedLine, +n) pending |
                                            // ready queue: tail line, ring[ntasks]
    int32_t* d_ring = nullptr;              // ready-queue mode (nullptr: static claim order)
    int32_t* d_ring_tail = nullptr;
    bool queue = false;
    int32_t* d_sched_init = nullptr;        // its solve-start image
    size_t sched_bytes = 0;
    int32_t* d_bar = nullptr;               // [0] arrivals, [kSchedLine] epoch
    pase::TaskDesc* d_tasks = nullptr;
    int32_t* d_order = nullptr;
    int64_t* d_trace = nullptr;             // PASE_TRACE=1: kTraceWords int64 per persistent task
    int ntasks = 0, nblocks = 0;
    int64_t total_tasks = 0;
    uint64_t timeout_ns = 4000000000ull;    // scheduler / barrier wait limit (PASE_SPIN_TIMEOUT_MS)
    bool persistent = true;
    bool stream_tiles = false;              // some vertex uses the TMA-staged stream tile or the
                                            // CTA tile (the kernel gets the dynamic shared memory)
    bool cost_tasks = false;                // persistent: cost tables as tasks of the DP kernel
    // multi-GPU
    pase::Peers peers{};
    bool connected = false;
    std::vector<double*> peer_T;            // every rank's T pool (index = rank), after connect
    std::vector<void*> ipc_opened;
    // host mirrors
    std::vector<VertexDesc> vd;
    std::vector<TermDesc> td;
    pase::SchedPlan sp;
    int32_t* h_choice = nullptr;            // pinned
    double* h_total = nullptr;              // pinned
    void* h_total_dev = nullptr;            // its device-mapped address (nullptr: copy instead)
    int32_t* h_err = nullptr;               // pinned
    bool override_tables = false;
    bool solved = false;
    bool launched = false;
    bool no_graph = false;
    int direct_left = 1;                    // solves to issue directly before capturing
    int profiling = 0;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_mid = nullptr, ev_dp = nullptr;
    uint64_t h2d_bytes = 0;
    pase_stats stats{};
};

namespace {

thread_local std::string g_create_err;

#define CUDA_TRY(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
            return PASE_ERR_CUDA;                                                         \
        }                                                                                 \
    } while (0)

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Device memory of single-process contexts comes from one stream-ordered pool per device
// that keeps freed memory cached (release threshold = max): a create/solve/destroy cycle
// then costs no cudaMalloc/cudaFree (each of which maps/unmaps pages and synchronises).
// Contexts of a multi-process group use cudaMalloc (their pools are exported over CUDA IPC).
std::mutex g_pool_mu;
cudaMemPool_t g_mempool[64] = {};

cudaMemPool_t device_mempool(int dev) {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_mempool[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t mp = nullptr;
        if (cudaMemPoolCreate(&mp, &props) != cudaSuccess) return nullptr;
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
        g_mempool[dev] = mp;
    }
    return g_mempool[dev];
}

// Pinned result blocks (total | err | choice[n]) are recycled through a small process-wide
// cache: cudaMallocHost/cudaFreeHost cost milliseconds (and cudaFreeHost synchronises).
constexpr size_t kPinnedBlock = 64 << 10;
std::vector<void*> g_pinned_free;
std::map<void*, size_t> g_stage_size;

void* pinned_get(size_t bytes, bool* big) {
    *big = bytes > kPinnedBlock;
    if (!*big) {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_pinned_free.empty()) {
            void* p = g_pinned_free.back();
            g_pinned_free.pop_back();
            return p;
        }
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, *big ? bytes : kPinnedBlock) != cudaSuccess) return nullptr;
    return p;
}

// Pinned upload staging blocks (pase_create): recycled, grown to the largest request.
std::vector<std::pair<void*, size_t>> g_stage_free;

void* stage_get(size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t k = 0; k < g_stage_free.size(); ++k)
            if (g_stage_free[k].second >= bytes) {
                void* p = g_stage_free[k].first;
                g_stage_free.erase(g_stage_free.begin() + k);
                return p;
            }
    }
    const size_t sz = std::max<size_t>(bytes, 4 << 20);
    void* p = nullptr;
    if (cudaMallocHost(&p, sz) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_stage_size[p] = sz;
    return p;
}

void stage_put(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_stage_free.push_back({p, g_stage_size[p]});
}

void pinned_put(void* p, bool big) {
    if (!p) return;
    if (big) { cudaFreeHost(p); return; }
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pinned_free.push_back(p);
}

// Cost-table work list: edges first (row chunks of the later-endpoint configs), then vertices.
std::vector<pase::CostChunk> cost_chunks(const Plan& P) {
    std::vector<pase::CostChunk> ch;
    for (int e = 0; e < P.m; ++e) {
        const pase_edge& x = P.edges[e];
        const int late = P.rank[x.src] > P.rank[x.dst] ? x.src : x.dst;
        // W_e is read by its earlier-ranked endpoint (reading T)
        const int reader = std::min(P.rank[x.src], P.rank[x.dst]);
        for (int r0 = 0; r0 < P.K[late]; r0 += pase::kCostRows)
            ch.push_back({P.n + e, r0, std::min(pase::kCostRows, P.K[late] - r0), x.src, reader});
    }
    for (int v = 0; v < P.n; ++v) ch.push_back({v, 0, P.K[v], v, P.rank[v]});
    return ch;
}

pase::CostArgs cost_args(const pase_ctx* ctx) {
    pase::CostArgs a{};
    a.nodes = ctx->d_nodes;
    a.K = ctx->d_K;
    a.cfg_off = ctx->d_cfg_off;
    a.cfg = ctx->d_cfg;
    a.loff = ctx->d_loff;
    a.n = ctx->P.n;
    a.enabled = ctx->override_tables ? 0 : 1;
    a.edges = ctx->d_edges;
    a.chunks = ctx->d_chunks;
    a.r = ctx->P.r;
    a.L = ctx->d_L;
    a.W = ctx->d_W;
    return a;
}

bool trace_on() {
    const char* t = std::getenv("PASE_TRACE");
    return t && t[0] == '1';
}

// lane-group size: each lane should own >= ~8 values of C (K=28 -> 4 lanes, K=84 -> 8,
// K=205 -> 16, K=456 -> 32): fewer lanes per item amortise the per-item decode and the
// cross-lane reduction over more candidates.
bool no_2d() {
    const char* t = std::getenv("PASE_NO_2D");
    return t && t[0] == '1';
}

// 2-D register tile: pick q2 = the coordinate other than qstar (and the
// multi-GPU partition coordinate) whose first term is latest; use the 2-D tile when its
// segment structure fits the kernel and it cuts the loads per candidate by >= 20 % on a
// vertex whose 1-D form is load-heavy.
// Lane-group widening on the critical path.  Estimated vertex time = waves of
// one-round tasks x (3 us + candidates per task / 6000 per us); a vertex whose longest
// leaf-to-root path through it is >= 85 % of the longest is critical (re-evaluated after each
// round of widening).  A critical vertex whose
// one-round tasks do not fill the grid widens its lane groups (every tile family
// encodes log2 G in the shape's low 2 bits; >= 8 values of C per lane kept) until they do:
// its K/G serial iterations -- the latency on the chain -- shrink, and the idle CTAs take the
// extra tasks.  Non-critical vertices keep the efficient narrow groups (widening every
// few-task vertex was measured slower, profiles/r01_ab_scheduling.txt).
// widening keeps at least this many values of C per lane (PASE_WIDEN_MINC)
const int kWidenMinC = std::getenv("PASE_WIDEN_MINC") ? std::max(1, std::atoi(std::getenv("PASE_WIDEN_MINC"))) : 8;
// ... and 2 for vertices with K <= 64 (PASE_SMALLK_MINC): their reductions are short, so the
// latency of the serial C loop, not the butterfly, dominates a widened task; they are widened
// only while their tasks still fit one wave (GNMT -16 %, others neutral: profiles/r02_ab_warm.txt)
const int kSmallKMinC = std::getenv("PASE_SMALLK_MINC") ? std::max(1, std::atoi(std::getenv("PASE_SMALLK_MINC"))) : 2;
int widen_minc(int K) { return K <= 64 ? kSmallKMinC : kWidenMinC; }
void widen_critical(pase_ctx* ctx) {
    static const bool widen = !(std::getenv("PASE_WIDEN") && std::getenv("PASE_WIDEN")[0] == '0');
    if (!widen) return;
    const Plan& P = ctx->P;
    const int n = P.n;
    // task-length cap (A/B, PASE_MAX_LANE_CAND): a one-round task of a big vertex occupies its CTA
    // for outputs-per-item x K/G serial candidates per lane; while that exceeds the cap, widen
    // the lane groups (shorter, more numerous tasks: a ready critical task waits less for a CTA)
    static const int64_t cap = std::getenv("PASE_MAX_LANE_CAND") ? std::atoll(std::getenv("PASE_MAX_LANE_CAND")) : 0;
    if (cap > 0)
        for (VertexDesc& d : ctx->vd) {
            if (d.shape < 0 || d.shape >= pase::kShapeG1 || d.wlog != 0) continue;
            const int64_t outs = d.q2 >= 0 ? pase::kTile1 * pase::kTile2 : pase::kTile;
            while (d.glog < 5 && (widen_minc(d.K) << (d.glog + 1)) <= d.K &&
                   outs * ((d.K + (1 << d.glog) - 1) >> d.glog) > cap) {
                ++d.glog;
                d.shape = (d.shape & ~3) | (d.glog - 2);
            }
        }
    const int64_t nb = ctx->nblocks;
    auto tasks_of = [&](const VertexDesc& d) -> int64_t {
        const int64_t items = std::max<int64_t>(1, d.nitems / (d.part ? ctx->world : 1));
        return std::max<int64_t>(1, ((items << d.glog) + 255) / 256);
    };
    // (rates from PASE_TRACE timelines: ~6000 candidates per us per CTA for the tiled
    // shapes; one-round latency-mode / generic tasks ~5.5 us)
    auto est = [&](const VertexDesc& d) -> double {
        const double cand = (double)d.nout * d.K / (d.part ? ctx->world : 1);
        if (d.shape < 0 || d.wlog > 0) return 5.5 + cand / 6000.0 / (double)nb;
        const int64_t T = tasks_of(d);
        return (double)((T + nb - 1) / nb) * (3.0 + cand / (double)T / 6000.0);
    };
    // a few rounds: widening the critical chain can make another chain critical
    for (int round = 0; round < 4; ++round) {
        std::vector<double> w(n), top(n), bot(n);
        for (int i = 0; i < n; ++i) w[i] = est(ctx->vd[i]) + 1.0;      // + dependency latency
        for (int i = 0; i < n; ++i) {                                  // children: lower ranks
            double mx = 0.0;
            for (int j : P.children[i]) mx = std::max(mx, top[j]);
            top[i] = w[i] + mx;
        }
        for (int i = n - 1; i >= 0; --i) bot[i] = w[i] + (P.parent[i] >= 0 ? bot[P.parent[i]] : 0.0);
        const double cp = top[n - 1];
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            VertexDesc& d = ctx->vd[i];
            static const double crit = std::getenv("PASE_CRIT_FRAC") ? std::atof(std::getenv("PASE_CRIT_FRAC")) : 0.85;
            if (top[i] + bot[i] - w[i] < crit * cp || d.shape < 0 || d.shape >= pase::kShapeG1 || d.wlog != 0) continue;
            while (d.glog < 5 && (widen_minc(d.K) << (d.glog + 1)) <= d.K && tasks_of(d) < nb) {
                // a short reduction (K <= 64) is widened only while its tasks still fit one wave
                if (d.K <= 64) {
                    VertexDesc w = d;
                    ++w.glog;
                    if (tasks_of(w) > nb) break;
                }
                ++d.glog;
                d.shape = (d.shape & ~3) | (d.glog - 2);
                changed = true;
            }
        }
        if (!changed) break;
    }
}

// single-suffix 2-D tile only for vertices with at least this many candidates (round 2 sweep,
// profiles/r02_ab_tiles.txt: 2^22 instead of 2^24 cuts the north-star DP 8 %, LE_P 1.4 %, neutral
// on InceptionV3 / GNMT / RNNLM; 2^18 hurts InceptionV3 and GNMT)
const int64_t kMin2S = std::getenv("PASE_MIN_2S") ? std::atoll(std::getenv("PASE_MIN_2S")) : (int64_t(1) << 22);

void set_tile2(VertexDesc& d, int q2, int f2) {
    d.q2 = q2;
    d.rq2 = d.radix[q2];
    d.t2star = f2;
    d.ostride_q2 = 1;
    for (int q = 0; q < q2; ++q) d.ostride_q2 *= d.radix[q];
    d.ntile2 = (d.rq2 + pase::kTile2 - 1) / pase::kTile2;
    d.ntile = ((d.rq + pase::kTile1 - 1) / pase::kTile1) * d.ntile2;
    d.ncombo = d.nout / ((int64_t)d.rq * d.rq2);
    d.nitems = d.ncombo * d.ntile;
}

void try_tile2(pase_ctx* ctx, VertexDesc& d, const TermDesc* tv, int top) {
    (void)ctx;
    if (d.qstar < 0 || d.m < 2 || d.rq < 2) return;
    // measured (profiles/r01_ab_*.txt): the general 2-D tile is faster than the 1-D one only
    // with >= 2 suffix terms; one suffix term takes the single-suffix 2-D form when the terms
    // have its structure (below)
    static const bool single = !(std::getenv("PASE_2S") && std::getenv("PASE_2S")[0] == '0');
    const int NSd = d.nterms - d.tstar;
    // candidate q2 coordinates, best first: latest first term (longest scalar prefix), then
    // larger radix
    std::vector<std::pair<int, int>> cand;                 // (first term, q)
    for (int q = 0; q < d.m; ++q) {
        if (q == d.qstar || (d.part && q == top) || d.radix[q] < 2) continue;
        int first = -1;
        for (int t = 0; t < d.nterms && first < 0; ++t)
            if (tv[t].stride[q] != 0) first = t;
        cand.push_back({first, q});
    }
    std::sort(cand.begin(), cand.end(), [&](const std::pair<int, int>& x, const std::pair<int, int>& y) {
        return x.first != y.first ? x.first > y.first : d.radix[x.second] > d.radix[y.second];
    });
    if (cand.empty()) return;
    // single-suffix form (tile2s_items): P0 = [0, f2) on neither coordinate; P1 = the first
    // term on q2 plus NB <= 1 terms not on q2; S = one term on qstar (not q2), optionally one
    // more not on q2 (on qstar or constant).  Small vertices keep the 1-D tile: twice the
    // items, i.e. twice the parallelism a latency-bound vertex needs (measured on InceptionV3).
    // Below kMin2S a 4-lane vertex with K >= 128 takes the 2-D form with 8-lane groups: half
    // the items of the 1-D tile but twice the lanes per item, so the same parallelism, half the
    // serial C iterations (still >= 16 per lane) and fewer loads per candidate (measured:
    // Transformer EXACT_P DP 0.571 -> 0.539 ms; with K < 128 the reduction dominates: GNMT
    // 0.633 -> 0.678 ms, hence the bound).
    static const bool wide = !(std::getenv("PASE_2S_WIDE") && std::getenv("PASE_2S_WIDE")[0] == '0');
    const bool big = d.nout * d.K >= kMin2S;
    static const int max2s = std::getenv("PASE_2S_MAXG") ? std::atoi(std::getenv("PASE_2S_MAXG")) : 5;
    if (single && (big || (wide && d.glog == 2 && d.K >= 128)) && NSd <= 2 && d.glog <= max2s) {
        for (const auto& cq : cand) {
            const int q2 = cq.second, f2 = cq.first;
            const int nb = d.tstar - f2 - 1;
            if (f2 < 1 || f2 > 3 || nb < 0 || nb > 1 || (NSd == 2 && nb != 0)) continue;
            bool ok = true;
            for (int t = f2 + 1; t < d.nterms; ++t) ok = ok && tv[t].stride[q2] == 0;
            for (int t = 0; t < d.nterms; ++t) ok = ok && tv[t].stride[q2] < (int64_t(1) << 31) / 16;
            if (!ok) continue;
            const int form = NSd == 1 ? nb : (tv[d.tstar + 1].stride[d.qstar] != 0 ? 3 : 2);
            if (!big) d.glog = 3;
            set_tile2(d, q2, f2);
            d.shape = pase::kShape2S + ((f2 - 1) * 4 + form) * 4 + (d.glog - 2);
            // CTA-tiled min-plus (PASE_CTA=1, single GPU): 4 groups of 64 threads, a 4 x 4 block
            // of outputs per thread: cb2 = q2 values (<= 64), cb1 = qstar values balanced over the
            // blocks; staged rounds of 32 values of C must fit the kernel's dynamic shared memory
            static const bool cta = std::getenv("PASE_CTA") && std::getenv("PASE_CTA")[0] == '1';
            if (cta && big && ctx->world == 1 && !d.part) {
                const int rq = d.rq, rq2 = d.rq2;
                const int cb2 = std::min(64, (rq2 + 3) / 4 * 4), T2 = cb2 / 4;
                const int T1 = std::min(16, 64 / T2);
                const int nblk1 = (rq + 4 * T1 - 1) / (4 * T1);
                const int cb1 = ((rq + nblk1 - 1) / nblk1 + 3) / 4 * 4;
                // two staging buffers and the final combine area in the kernel's dynamic smem
                const size_t need = std::max<size_t>(2 * sizeof(double) * (size_t)pase::kCtaG * pase::kCtaCC *
                                                     ((pase::kMaxP0 + 2) + (cb2 + 1) + 2 * (cb1 + 1)),
                                                     (size_t)pase::kCtaG * 16 * 64 * 12);
                if (T1 >= 1 && need <= pase::kCtaSmemMax) {
                    d.cb1 = cb1;
                    d.cb2 = cb2;
                    d.ntile2 = (rq2 + cb2 - 1) / cb2;
                    d.ntile = nblk1 * d.ntile2;
                    d.nitems = d.ncombo * d.ntile;
                    d.glog = 8;                           // one item per CTA round
                    d.shape = pase::kShapeCta + (f2 - 1) * 4 + form;
                }
            }
            return;
        }
    }
    // measured (profiles/r01_ab_*.txt): the general 2-D tile is faster than the 1-D one only
    // with >= 2 suffix terms
    if (NSd < 2) return;
    const int q2 = cand[0].second, f2 = cand[0].first;
    if (q2 < 0 || f2 < 1) return;
    const int nP0 = f2, nP1 = d.tstar - f2, NS = d.nterms - d.tstar;
    if (nP0 > pase::kMaxP0 || nP1 > pase::kMaxP1 || NS < 1 || NS > 2) return;
    if (NS == 2 && (tv[d.tstar].stride[q2] != 0 || tv[d.tstar + 1].stride[q2] != 0)) return;
    for (int t = 0; t < d.nterms; ++t)
        if (tv[t].stride[q2] >= (int64_t(1) << 31) / 16) return;
    double l2 = nP0;
    for (int t = f2; t < d.tstar; ++t) l2 += tv[t].stride[q2] ? pase::kTile2 : 1;
    for (int t = d.tstar; t < d.nterms; ++t) l2 += tv[t].stride[q2] ? pase::kTile1 * pase::kTile2 : pase::kTile1;
    const double per2 = l2 / (pase::kTile1 * pase::kTile2);
    const double per1 = (double)(d.tstar + pase::kTile * NS) / pase::kTile;
    static const double gain2 = std::getenv("PASE_2D_GAIN") ? std::atof(std::getenv("PASE_2D_GAIN")) : 0.8;
    if (per2 > gain2 * per1) return;
    set_tile2(d, q2, f2);
    d.shape = pase::kShape2D + (NS - 1) * 4 + (d.glog - 2);
}

// dependency wait at each warp's tile gate, after its work-item decode (PASE_EARLY_GATE=0: one
// thread per CTA waits before the tile starts)
// thread per CTA waits before the tile starts).  Bit 1 (PASE_WARM, default on): a task whose
// children are still running when it is claimed runs its first work item once without stores
// before the gate, so its tile's code is in this SM's instruction caches when the gate opens.
// Bit 2 (PASE_GATE_ELECT=1): one warp per CTA polls the counter, the others a shared flag.
int early_gate() {
    static const int mode = [] {
        const char* e = std::getenv("PASE_EARLY_GATE");
        if (e && e[0] == '0') return 0;
        const char* w = std::getenv("PASE_WARM");
        const char* el = std::getenv("PASE_GATE_ELECT");
        // bits 3 / 4: acquire by ld.acquire of the counter instead of fence.acq_rel at the gates of
        // 1-D tiles (PASE_GATE_LDACQ=1) / of every tile (2, the default: no MEMBAR.GPU per gate;
        // same-binary A/B, profiles/r02_ab_reentry.txt: -4 % DP on Transformer, -6..-12 % on
        // GNMT / RNNLM / InceptionV3 / AlexNet, -0.7 % on LE_P); 0 = the fence everywhere
        const char* la = std::getenv("PASE_GATE_LDACQ");
        const int ldacq = la ? std::atoi(la) : 2;
        // bit 5 (default; PASE_REL_RED=0 turns it off): a finished task releases its parent with
        // red.release (no return value to wait for) instead of atom.acq_rel -- its CTA claims the
        // next task ~1 us sooner (same-binary A/B: -0.9 % DP on Transformer, -1.4 % GNMT, +0.8 % RNNLM)
        const char* rr = std::getenv("PASE_REL_RED");
        return ((w && w[0] == '0') ? 1 : 3) | ((el && el[0] == '1') ? 4 : 0) | (ldacq == 1 ? 8 : ldacq == 2 ? 16 : 0) |
               ((rr && rr[0] == '0') ? 0 : 32);
    }();
    return mode;
}

// streaming-vertex form (PASE_STREAM_TMA): 0 = direct full-warp loads, 1 = rows TMA-staged in a
// shared-memory ring, 2 = direct loads with the next item's rows TMA-prefetched into L2
int stream_tma() {
    static const int mode = std::getenv("PASE_STREAM_TMA") ? std::atoi(std::getenv("PASE_STREAM_TMA")) : 2;
    return mode;
}

// streaming-regime vertices: spanning child tables of at least this many bytes
const uint64_t kStreamBytes = std::getenv("PASE_STREAM_MB") ? (uint64_t)std::atoll(std::getenv("PASE_STREAM_MB")) << 20 : (64ull << 20);

// latency mode: vertices with at most this many candidates (N_i * K)
const int64_t kLatencyCand = std::getenv("PASE_LATENCY_CAND") ? std::atoll(std::getenv("PASE_LATENCY_CAND")) : (1 << 18);

int lane_group_log2(int K) {
    static const int per_lane = std::getenv("PASE_C_PER_LANE") ? std::atoi(std::getenv("PASE_C_PER_LANE")) : 32;
    int g = 2;
    while (g < 5 && (1 << (g + 1)) * per_lane <= K) ++g;
    return g;
}

struct Item { void** ptr; size_t bytes; };

// Carve items out of one allocation (base == nullptr for host-only contexts: offsets only).
pase_status carve(pase_ctx* ctx, std::vector<Item>& items, void** base, size_t* bytes, bool device) {
    size_t total = 0;
    for (auto& it : items) total += align_up(it.bytes);
    total = std::max<size_t>(total, 256);
    if (device) {
        cudaError_t e = cudaErrorMemoryAllocation;
        if (ctx->async_pools) {
            cudaMemPool_t mp = device_mempool(ctx->dev);
            e = mp ? cudaMallocFromPoolAsync(base, total, mp, ctx->stream) : cudaErrorMemoryAllocation;
        } else {
            e = cudaMalloc(base, total);
        }
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaMalloc of ") + std::to_string(total) + " bytes failed: " + cudaGetErrorString(e);
            return PASE_ERR_RESOURCE;
        }
    } else {
        *base = nullptr;
    }
    *bytes = total;
    char* p = (char*)*base;
    for (auto& it : items) { *it.ptr = p; p += align_up(it.bytes); }
    return PASE_OK;
}

// Pool 1: everything whose size the plan fixes.
pase_status allocate(pase_ctx* ctx, bool device) {
    const Plan& P = ctx->P;
    const int n = P.n, m = P.m;
    int64_t nterms_total = 0;
    for (int i = 0; i < n; ++i) nterms_total += 1 + (int64_t)P.egt[i].size() + (int64_t)P.children[i].size();
    const int64_t ncfg = P.cfg_off[n];
    ctx->nchunks = (int)cost_chunks(P).size();
    // uploaded items first: prepare() stages them in one host image and copies it once
    std::vector<Item> items = {
        {(void**)&ctx->d_nodes, sizeof(pase_node) * n},
        {(void**)&ctx->d_K, sizeof(int32_t) * n},
        {(void**)&ctx->d_cfg_off, sizeof(int64_t) * (n + 1)},
        {(void**)&ctx->d_cfg, sizeof(int32_t) * pase::kMaxDims * ncfg},
        {(void**)&ctx->d_loff, sizeof(int64_t) * (n + 1)},
        {(void**)&ctx->d_edges, sizeof(EdgeDesc) * std::max(m, 1)},
        {(void**)&ctx->d_chunks, sizeof(pase::CostChunk) * (size_t)ctx->nchunks},
        {(void**)&ctx->d_vd, sizeof(VertexDesc) * n},
        {(void**)&ctx->d_td, sizeof(TermDesc) * nterms_total},
        {(void**)&ctx->d_bt, sizeof(pase::BtDesc) * n},
        {(void**)&ctx->d_bt_off, sizeof(int32_t) * (n + 1)},
        {(void**)&ctx->d_L, sizeof(double) * P.loff[n]},
        {(void**)&ctx->d_W, sizeof(double) * std::max<int64_t>(P.woff[m], 1)},
        {(void**)&ctx->d_T, sizeof(double) * P.toff[n]},
        {(void**)&ctx->d_A, sizeof(uint16_t) * P.toff[n]},
        // solve outputs, laid out as the pinned host block: total | err | pad | choice[n]
        // (one D2H copy per solve)
        {(void**)&ctx->d_total, 16 + sizeof(int32_t) * n},
    };
    size_t total = 0;
    for (auto& it : items) total += align_up(it.bytes);
    const uint64_t budget = ctx->mach.table_budget_bytes ? ctx->mach.table_budget_bytes : (64ull << 30);
    if (total > budget) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "size guard: %.3f GB of tables/state exceeds the budget of %.3f GB (M = %d, K = %d)",
                      total / 1e9, budget / 1e9, P.max_dep, P.max_k);
        ctx->err = buf;
        return PASE_ERR_RESOURCE;
    }
    pase_status st = carve(ctx, items, &ctx->pool, &ctx->pool_bytes, device);
    ctx->d_err = (int32_t*)((char*)ctx->d_total + 8);
    ctx->d_choice = (int32_t*)((char*)ctx->d_total + 16);
    return st;
}

// Vertex/term descriptors, the task schedule (schedule.cpp), pool 2, upload.
pase_status prepare(pase_ctx* ctx, bool device) {
    using clk = std::chrono::steady_clock;
    const auto p0 = clk::now();
    const Plan& P = ctx->P;
    const int n = P.n, m = P.m;
    std::vector<EdgeDesc> ed(std::max(m, 1));
    for (int e = 0; e < m; ++e) {
        EdgeDesc& d = ed[e];
        d.src = P.edges[e].src;
        d.dst = P.edges[e].dst;
        d.later_is_src = P.rank[d.src] > P.rank[d.dst];
        d.pad = 0;
        for (int a = 0; a < pase::kMaxDims; ++a) d.axis_map[a] = P.edges[e].axis_map[a];
        d.woff = P.woff[e];
    }
    const std::vector<pase::CostChunk> chunks = cost_chunks(P);
    const uint64_t redundant_below = ctx->mach.redundant_below_bytes;

    ctx->vd.assign(n, VertexDesc{});
    ctx->td.clear();
    for (int i = 0; i < n; ++i) {
        const int v = P.sigma[i];
        VertexDesc& d = ctx->vd[i];
        d.K = P.K[v];
        d.m = (int32_t)P.dep[i].size();
        d.term0 = (int32_t)ctx->td.size();
        d.nout = P.tsize[i];
        for (int q = 0; q < pase::kMaxDep; ++q) d.radix[q] = q < d.m ? P.K[P.dep[i][q]] : 1;
        d.T = ctx->d_T + P.toff[i];
        d.A = ctx->d_A + P.toff[i];
        d.parent = P.parent[i];
        auto pos_of = [&](int node) {
            for (int q = 0; q < d.m; ++q) if (P.dep[i][q] == node) return q;
            return -1;
        };
        TermDesc t{};
        t.base = ctx->d_L + P.loff[v];                    // term 0: L_{sigma_i}[C]
        ctx->td.push_back(t);
        for (int e : P.egt[i]) {                          // edges to later neighbours (E> order)
            TermDesc te{};
            const int other = P.edges[e].src == v ? P.edges[e].dst : P.edges[e].src;
            const int q = pos_of(other);
            if (q < 0) { ctx->err = "internal: E>(sigma_i) endpoint outside D(i)"; return PASE_ERR_STATE; }
            te.base = ctx->d_W + P.woff[e];               // row = config of the other endpoint
            te.stride[q] = d.K;
            ctx->td.push_back(te);
        }
        for (int j : P.children[i]) {                     // children, ascending rank
            TermDesc tc{};                                // T_j coords (sigma_i, w_1, ...), sigma_i fastest
            tc.base = ctx->d_T + P.toff[j];
            int64_t st = P.K[v];
            for (size_t a = 1; a < P.dep[j].size(); ++a) {
                const int q = pos_of(P.dep[j][a]);
                if (q < 0 || P.dep[j][0] != v) { ctx->err = "internal: child table not nested"; return PASE_ERR_STATE; }
                tc.stride[q] += st;
                st *= P.K[P.dep[j][a]];
            }
            ctx->td.push_back(tc);
        }
        d.nterms = (int32_t)ctx->td.size() - d.term0;
        // multi-GPU partition by the top coordinate: big tables only
        const int top = d.m - 1;
        d.part = (ctx->world > 1 && d.m >= 2 && (uint64_t)d.nout * 8ull >= redundant_below &&
                  d.radix[top] >= 2) ? 1 : 0;
        // qstar = the coordinate whose first term is latest in the canonical order (longest
        // hoistable prefix); ties -> larger radix, lower q; never the partition coordinate.
        const TermDesc* tv = ctx->td.data() + d.term0;
        d.qstar = -1;
        d.tstar = d.nterms;
        int best_first = -1;
        for (int q = 0; q < d.m; ++q) {
            int first = -1;
            for (int t = 0; t < d.nterms && first < 0; ++t)
                if (tv[t].stride[q] != 0) first = t;
            if (first < 1) { ctx->err = "internal: D(i) coordinate not used by any term"; return PASE_ERR_STATE; }
            if (d.part && q == top) continue;
            if (first > best_first || (first == best_first && d.radix[q] > d.radix[d.qstar])) {
                best_first = first;
                d.qstar = q;
            }
        }
        if (d.qstar >= 0) d.tstar = best_first;
        d.rq = d.qstar >= 0 ? d.radix[d.qstar] : 1;
        d.ntile = (d.rq + pase::kTile - 1) / pase::kTile;
        d.ostride_q = 1;
        for (int q = 0; q < d.qstar; ++q) d.ostride_q *= d.radix[q];
        if (d.qstar < 0) d.ostride_q = 0;
        d.ncombo = d.nout / d.rq;
        d.nitems = d.ncombo * d.ntile;
        bool wide = d.nitems >= (int64_t(1) << 31);       // 32-bit item decode
        for (int t = 0; t < d.nterms; ++t)
            for (int q = 0; q < d.m; ++q)
                if (tv[t].stride[q] >= (int64_t(1) << 31) / 16) wide = true;
        const int NP = d.tstar, NS = d.nterms - d.tstar;
        d.wlog = 0;
        d.q2 = -1;
        d.rq2 = 1;
        d.ntile2 = 1;
        d.t2star = d.tstar;
        d.ostride_q2 = 0;
        // streaming regime: a child table spanning (sigma_i, D(i)) gives every
        // candidate one 8-B value nobody else reads; with L2-exceeding tables the vertex is
        // HBM-bound, so full-warp lane groups read each row as 256-B coalesced segments (narrow
        // groups would scatter a warp's loads over 8 rows: L1-wavefront bound, measured)
        bool streaming = false, last_spans = false;
        for (int j : P.children[i])
            if (P.tsize[j] == (int64_t)d.K * d.nout && (uint64_t)P.tsize[j] * 8ull >= kStreamBytes) {
                streaming = true;
                last_spans = j == P.children[i].back();   // the spanning table is the last term
            }
        if (!wide && NP >= 1 && NP <= 4 && NS >= 0 && NS <= 3) {
            d.glog = lane_group_log2(d.K);
            // latency mode: a small vertex (<= kLatencyCand candidates) is
            // latency-bound -- on a critical-path chain its few items cannot fill the GPU --
            // so each item gets L = pow2 >= K/2 lanes (W = L/32 full warps when L > 32): every
            // lane reduces <= 2 values of C, i.e. one round of loads.  (Measured: widening the
            // lane groups of mid-size vertices too -- up to a warp, or to K/2 lanes, whenever
            // their items cannot fill the grid -- is slower overall: 0.58 -> 0.76 / 1.42 ms DP
            // on Transformer p=64; the extra tasks cost more than the shorter chains save.)
            if ((int64_t)d.nout * d.K <= kLatencyCand) {
                // values of C per lane (PASE_LAT_CPL, default 2: one round of loads)
                static const int cpl = std::getenv("PASE_LAT_CPL") ? std::max(1, std::atoi(std::getenv("PASE_LAT_CPL"))) : 2;
                int ll = 2;
                while (ll < 8 && (cpl << ll) < d.K) ++ll;
                // one value of C per lane (twice the lanes) while that needs <= PASE_LAT_ONE_LANES
                // lanes (default 16: K <= 16, the group stays inside a warp) and the vertex's tasks
                // number <= PASE_LAT_ONE_TASKS (default unbounded; 0 = off).  Same-binary A/B
                // (profiles/r02_ab_reentry.txt): InceptionV3 -14 % DP (87 K = 6 vertices), others
                // +-0.1 %; wider limits (32+ lanes) cost Transformer / RNNLM 3-6 %.
                static const int64_t one_tasks = std::getenv("PASE_LAT_ONE_TASKS") ? std::atoll(std::getenv("PASE_LAT_ONE_TASKS")) : (int64_t(1) << 40);
                static const int one_lanes = std::getenv("PASE_LAT_ONE_LANES") ? std::atoi(std::getenv("PASE_LAT_ONE_LANES")) : 16;
                if (one_tasks > 0 && ll < 8 && (2 << ll) >= d.K && (2 << ll) <= one_lanes &&
                    (d.nitems << (ll + 1)) <= one_tasks * 256) ++ll;
                d.glog = std::min(ll, 5);
                d.wlog = ll - d.glog;
            }
            d.shape = (NP - 1) * 16 + NS * 4 + (d.glog - 2);
            if (d.wlog == 0 && streaming) {
                d.glog = 5;
                d.shape = (NP - 1) * 16 + NS * 4 + 3;
                // its rows staged into shared memory by TMA bulk copies
                if (last_spans && NS >= 1 && stream_tma() == 1) d.shape = pase::kShapeStream + (NP - 1) * 4 + NS;
                if (last_spans && NS >= 1 && stream_tma() == 2) d.shape = pase::kShapeStreamPF + (NP - 1) * 4 + NS;
                static const int ahead = std::getenv("PASE_STREAM_PF_AHEAD") ? std::atoi(std::getenv("PASE_STREAM_PF_AHEAD")) : 0;
                d.pf_ahead = ahead;
            } else if (d.wlog == 0 && d.K <= 3) {             // one lane per item
                d.glog = 0;
                d.shape = pase::kShapeG1 + (NP - 1) * 4 + NS;
            } else if (d.wlog == 0 && !no_2d()) {
                try_tile2(ctx, d, tv, top);
            }
        } else {                                          // generic kernel
            d.glog = d.K <= 4 ? 2 : d.K <= 8 ? 3 : d.K <= 16 ? 4 : 5;
            d.shape = -1;
        }
    }
    const auto p1 = clk::now();
    widen_critical(ctx);
    ctx->stream_tiles = false;
    for (const VertexDesc& d : ctx->vd)
        ctx->stream_tiles = ctx->stream_tiles || pase::stream_smem_shape(d.shape) || pase::cta_shape(d.shape);
    for (VertexDesc& d : ctx->vd) {                       // partitioned item order (split_item)
        d.psub = (d.part && d.shape >= 0) ? (int32_t)(d.ncombo / d.radix[d.m - 1]) : 1;
        // magic numbers of the work-item decode (division by invariant integers)
        for (int q = 0; q < pase::kMaxDep; ++q) pase::fastdiv_magic((uint32_t)std::max(1, d.radix[q]), d.rmul[q], d.rsh[q]);
        pase::fastdiv_magic((uint32_t)std::max<int64_t>(1, std::min<int64_t>(d.ncombo, INT32_MAX)), d.mul_combo, d.sh_combo);
        pase::fastdiv_magic((uint32_t)std::max(1, d.ntile), d.mul_tile, d.sh_tile);
        pase::fastdiv_magic((uint32_t)std::max(1, d.ntile2), d.mul_tile2, d.sh_tile2);
        pase::fastdiv_magic((uint32_t)std::max(1, d.psub), d.mul_psub, d.sh_psub);
    }
    const auto p2 = clk::now();
    // tasks, broadcast flags, pending counters, claim order (schedule.cpp)
    std::vector<int32_t> consumer(chunks.size());
    for (size_t k = 0; k < chunks.size(); ++k) consumer[k] = chunks[k].consumer;
    // ready queue (single GPU, opt-in PASE_QUEUE=1): measured SLOWER than the static critical-path
    // order on every workload (profiles/r02_ab_queue.txt: FIFO publication loses the priority, and
    // non-critical ready work competes with the critical chain for the SMs)
    const char* qv = std::getenv("PASE_QUEUE");
    ctx->queue = ctx->world == 1 && !ctx->cost_tasks && qv && qv[0] == '1';
    pase_status st = pase::build_schedule(P, ctx->vd, ctx->world, ctx->rank, ctx->nblocks, ctx->sp, ctx->err,
                                          ctx->cost_tasks ? &consumer : nullptr, !ctx->queue);
    if (st) return st;
    ctx->ntasks = (int)ctx->sp.tasks.size();
    ctx->total_tasks = ctx->sp.total_tasks;
    for (VertexDesc& d : ctx->vd) d.npeer = d.bcast ? ctx->world - 1 : 0;
    const auto p3 = clk::now();
    // pool 2
    // ready queue: tail on its own line after the pending counters, then one ring slot per
    // task; reset with the rest of the block
    const size_t pend_words = ((size_t)n + pase::kSchedLine - 1) / pase::kSchedLine * pase::kSchedLine;
    const size_t ring_off = pase::kSchedLine + pend_words + pase::kSchedLine;
    const size_t sched_words = ctx->queue ? ring_off + std::max<size_t>(ctx->sp.tasks.size(), 1) : pase::kSchedLine + (size_t)n;

    ctx->sched_bytes = sizeof(int32_t) * sched_words;
    std::vector<Item> items2 = {                          // uploaded items first, as pool 1
        {(void**)&ctx->d_sched_init, ctx->sched_bytes},
        {(void**)&ctx->d_tasks, sizeof(pase::TaskDesc) * std::max<size_t>(ctx->sp.tasks.size(), 1)},
        {(void**)&ctx->d_order, sizeof(int32_t) * std::max<size_t>(ctx->sp.order.size(), 1)},
        {(void**)&ctx->d_sched, ctx->sched_bytes},
        {(void**)&ctx->d_bar, sizeof(int32_t) * 3 * pase::kSchedLine},
        {(void**)&ctx->d_trace, trace_on() ? sizeof(int64_t) * pase::kTraceWords * std::max<size_t>(ctx->sp.tasks.size(), 1) : 0},
    };
    if ((st = carve(ctx, items2, &ctx->pool2, &ctx->pool2_bytes, device))) return st;
    std::vector<int32_t> sched(sched_words, 0);
    for (int i = 0; i < n; ++i) sched[pase::kSchedLine + i] = ctx->sp.pending[i];
    ctx->d_ring = ctx->d_ring_tail = nullptr;
    if (ctx->queue) {                           // the leaves' tasks are published from the start
        for (size_t k = 0; k < ctx->sp.ready0.size(); ++k) sched[ring_off + k] = ctx->sp.ready0[k] + 1;
        sched[ring_off - pase::kSchedLine] = (int32_t)ctx->sp.ready0.size();
        if (ctx->d_sched) {
            ctx->d_ring = ctx->d_sched + ring_off;
            ctx->d_ring_tail = ctx->d_sched + ring_off - pase::kSchedLine;
        }
    }
    // single-rank peer table (connect() fills the group's)
    ctx->peers = pase::Peers{};
    ctx->peers.world = ctx->world;
    ctx->peers.rank = ctx->rank;
    ctx->peers.pending[ctx->rank] = ctx->d_sched + pase::kSchedLine;
    ctx->peers.bar[ctx->rank] = ctx->d_bar;
    // back-substitution: levels lev(root) = 0, lev(i) = 1 + max lev over D(i);
    // the vertices of one level are independent, records in level order
    std::vector<int> blev(n, 0);
    int nlev = 0;
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int u : P.dep[i]) l = std::max(l, blev[P.rank[u]] + 1);
        blev[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<int32_t> bt_off(nlev + 1, 0);
    for (int i = 0; i < n; ++i) bt_off[blev[i] + 1]++;
    for (int l = 0; l < nlev; ++l) bt_off[l + 1] += bt_off[l];
    std::vector<pase::BtDesc> bt(n);
    {
        std::vector<int32_t> fill(bt_off.begin(), bt_off.end() - 1);
        for (int i = n - 1; i >= 0; --i) {
            pase::BtDesc& b = bt[fill[blev[i]]++];
            b = pase::BtDesc{};
            b.A = ctx->vd[i].A;
            b.node = P.sigma[i];
            b.K = P.K[P.sigma[i]];
            int64_t st = 1;
            for (size_t a = 0; a < P.dep[i].size(); ++a) {
                b.dep[a] = P.dep[i][a];
                b.stride[a] = st;
                st *= P.K[P.dep[i][a]];
            }
        }
    }
    const int ngroups = nlev;
    ctx->nbtlev = ngroups;
    // one host image per pool (the uploaded prefix), one copy each
    // one upload image per pool (the uploaded prefix of each), staged in PINNED host memory
    // (a recycled process-wide block) so both copies run asynchronously at full PCIe rate;
    // host-only contexts only size them
    const size_t size1 = (size_t)((char*)ctx->d_L - (char*)ctx->pool);
    const size_t size2 = (size_t)((char*)ctx->d_sched - (char*)ctx->pool2);
    ctx->h2d_bytes = size1 + size2;
    if (const char* tv = std::getenv("PASE_TIMING"); tv && tv[0] == '1') {
        auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[pase] prepare: descriptors %.3f ms, widen %.3f ms, schedule %.3f ms, pool2+bt %.3f ms\n",
                     ms(p0, p1), ms(p1, p2), ms(p2, p3), ms(p3, clk::now()));
    }
    if (!device) return PASE_OK;
    char* img = (char*)stage_get(size1 + size2);
    if (!img) { ctx->err = "cudaMallocHost of the upload image failed"; return PASE_ERR_RESOURCE; }
    ctx->stage_block = img;
    auto stage = [&](char* base, void* pool, void* dst, const void* src, size_t bytes) {
        if (bytes) std::memcpy(base + ((char*)dst - (char*)pool), src, bytes);
    };
    char* img1 = img;
    char* img2 = img + size1;
    stage(img1, ctx->pool, ctx->d_nodes, P.nodes.data(), sizeof(pase_node) * n);
    stage(img1, ctx->pool, ctx->d_K, P.K.data(), sizeof(int32_t) * n);
    stage(img1, ctx->pool, ctx->d_cfg_off, P.cfg_off.data(), sizeof(int64_t) * (n + 1));
    stage(img1, ctx->pool, ctx->d_cfg, P.cfg.data(), sizeof(int32_t) * P.cfg.size());
    stage(img1, ctx->pool, ctx->d_loff, P.loff.data(), sizeof(int64_t) * (n + 1));
    stage(img1, ctx->pool, ctx->d_edges, ed.data(), sizeof(EdgeDesc) * ed.size());
    stage(img1, ctx->pool, ctx->d_chunks, chunks.data(), sizeof(pase::CostChunk) * chunks.size());
    stage(img1, ctx->pool, ctx->d_vd, ctx->vd.data(), sizeof(VertexDesc) * n);
    stage(img1, ctx->pool, ctx->d_td, ctx->td.data(), sizeof(TermDesc) * ctx->td.size());
    stage(img1, ctx->pool, ctx->d_bt, bt.data(), sizeof(pase::BtDesc) * n);
    stage(img1, ctx->pool, ctx->d_bt_off, bt_off.data(), sizeof(int32_t) * bt_off.size());
    stage(img2, ctx->pool2, ctx->d_sched_init, sched.data(), ctx->sched_bytes);
    stage(img2, ctx->pool2, ctx->d_tasks, ctx->sp.tasks.data(), sizeof(pase::TaskDesc) * ctx->sp.tasks.size());
    stage(img2, ctx->pool2, ctx->d_order, ctx->sp.order.data(), sizeof(int32_t) * ctx->sp.order.size());
    // the block returns to the cache once pase_create has synchronised the stream
    CUDA_TRY(cudaMemcpyAsync(ctx->pool, img1, size1, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->pool2, img2, size2, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->d_bar, 0, sizeof(int32_t) * 3 * pase::kSchedLine, ctx->stream));
    return PASE_OK;
}

// Issue (or capture) the whole solve.  Persistent schedule: cost tables -> reset scheduler
// -> [group barrier] -> dp_persistent -> [group barrier] -> back-substitution -> D2H.
// PASE_SCHEDULE=launches: one kernel per vertex, children -> parent event edges.
pase_status issue_schedule(pase_ctx* ctx, bool capture) {
    const Plan& P = ctx->P;
    const int n = P.n;
    if (capture && ctx->exec) { cudaGraphExecDestroy(ctx->exec); ctx->exec = nullptr; }
    const int nstreams = ctx->persistent ? 0 : 4;
    if (ctx->aux.empty() && nstreams) {
        ctx->aux.resize(nstreams);
        for (auto& s : ctx->aux) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    std::vector<cudaEvent_t> done(ctx->persistent ? 0 : n);
    for (auto& e : done) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t start = nullptr;
    if (!ctx->persistent) CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    std::vector<cudaEvent_t> join(nstreams);
    for (auto& e : join) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t s = ctx->stream;
    if (capture) CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const unsigned ext = capture ? cudaEventRecordExternal : cudaEventRecordDefault;
    int32_t* d_err = ctx->d_err;
    // the cost-table kernel also resets the error flag and the persistent scheduler's state
    // (claim counter, pending counters) before the DP kernel starts: no memset / copy nodes
    const bool fold = !ctx->override_tables && !ctx->cost_tasks;
    if (fold) {
        pase::CostArgs ca = cost_args(ctx);
        ca.err = d_err;
        if (ctx->persistent) {
            ca.sched = ctx->d_sched;
            ca.sched_init = ctx->d_sched_init;
            ca.sched_words = (int32_t)(ctx->sched_bytes / sizeof(int32_t));
        }
        pase::launch_cost_tables(ca, ctx->nchunks, s);
    } else {
        CUDA_TRY(cudaMemsetAsync(d_err, 0, sizeof(int32_t), s));
    }
    // phase split: external event nodes (plain records would only become capture edges)
    CUDA_TRY(cudaEventRecordWithFlags(ctx->ev_mid, s, ext));
    std::vector<char> used(nstreams, 0);
    if (ctx->persistent) {
        if (!fold)
            CUDA_TRY(cudaMemcpyAsync(ctx->d_sched, ctx->d_sched_init, ctx->sched_bytes, cudaMemcpyDeviceToDevice, s));
        if (ctx->world > 1) pase::launch_rank_barrier(ctx->peers, ctx->d_bar, d_err, ctx->timeout_ns, s);
        pase::launch_dp_persistent(ctx->d_vd, ctx->d_td, ctx->d_tasks, ctx->d_order, ctx->ntasks, ctx->d_sched,
                                   d_err, ctx->peers, cost_args(ctx), ctx->nblocks,
                                   trace_on() ? ctx->d_trace : nullptr, ctx->timeout_ns, ctx->stream_tiles,
                                   ctx->d_ring, ctx->d_ring_tail, early_gate(), s);
        if (ctx->world > 1) pase::launch_rank_barrier(ctx->peers, ctx->d_bar, d_err, ctx->timeout_ns, s);
    } else {
        CUDA_TRY(cudaEventRecord(start, s));
        std::vector<int> sid(n, -1);                      // a chain stays on one stream
        int rr = 0;
        for (int i = 0; i < n; ++i) {
            sid[i] = P.children[i].empty() ? (rr++ % nstreams) : sid[P.children[i][0]];
            cudaStream_t si = ctx->aux[sid[i]];
            if (!used[sid[i]]) { CUDA_TRY(cudaStreamWaitEvent(si, start, 0)); used[sid[i]] = 1; }
            for (int j : P.children[i])
                if (sid[j] != sid[i]) CUDA_TRY(cudaStreamWaitEvent(si, done[j], 0));
            pase::launch_dp_vertex(ctx->d_vd, ctx->d_td, i, ctx->vd[i], si);
            CUDA_TRY(cudaEventRecord(done[i], si));
        }
        for (int k = 0; k < nstreams; ++k)
            if (used[k]) {
                CUDA_TRY(cudaEventRecord(join[k], ctx->aux[k]));
                CUDA_TRY(cudaStreamWaitEvent(s, join[k], 0));
            }
    }
    CUDA_TRY(cudaEventRecordWithFlags(ctx->ev_dp, s, ext));
    // the back-substitution kernel stores the result block straight into the pinned host block
    // (device-mapped); without a mapping, one D2H copy of it
    pase::launch_backtrack(ctx->d_bt, ctx->d_bt_off, ctx->nbtlev, n, ctx->vd[n - 1].T, ctx->d_choice,
                           ctx->d_total, ctx->d_err, ctx->h_total_dev, s);
    if (!ctx->h_total_dev)
        CUDA_TRY(cudaMemcpyAsync(ctx->h_total, ctx->d_total, 16 + sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    cudaError_t ce = cudaSuccess;
    cudaGraph_t graph = nullptr;
    if (capture) ce = cudaStreamEndCapture(s, &graph);
    for (auto& e : done) cudaEventDestroy(e);
    for (auto& e : join) cudaEventDestroy(e);
    if (start) cudaEventDestroy(start);
    if (ce != cudaSuccess) { ctx->err = std::string("stream capture: ") + cudaGetErrorString(ce); return PASE_ERR_CUDA; }
    if (capture) {
        ce = cudaGraphInstantiate(&ctx->exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) { ctx->err = std::string("graph instantiate: ") + cudaGetErrorString(ce); return PASE_ERR_CUDA; }
    }
    return PASE_OK;
}

// The solve schedule is issued directly at the first solve after a (re)configuration and
// recorded as a CUDA graph at the second (a context solved once -- the create/solve/destroy
// pattern -- never pays for capture and instantiation); PASE_NO_GRAPH=1 issues it directly
// at every solve.
pase_status record_graph(pase_ctx* ctx) {
    const int dp_launches = ctx->persistent ? 1 + (ctx->world > 1 ? 2 : 0) : ctx->P.n;
    ctx->stats.n_launches = (ctx->override_tables || ctx->cost_tasks ? 0 : 1) + dp_launches + 1;
    const char* ng = std::getenv("PASE_NO_GRAPH");
    ctx->no_graph = ng && ng[0] == '1';
    if (ctx->exec) { cudaGraphExecDestroy(ctx->exec); ctx->exec = nullptr; }
    ctx->direct_left = 1;
    return PASE_OK;
}

void fill_stats(pase_ctx* ctx) {
    const Plan& P = ctx->P;
    pase_stats& s = ctx->stats;
    s.n_vertices = P.n;
    s.n_edges = P.m;
    s.max_dep = P.max_dep;
    s.max_configs = P.max_k;
    s.tree_levels = P.levels;
    s.candidates = P.candidates;
    s.table_entries = P.entries;
    s.cost_entries = (uint64_t)(P.loff[P.n] + P.woff[P.m]);
    // each table written once (8 B value + 2 B argmin) and read once by its parent;
    // W_e rows and L read by the vertex that owns them.
    uint64_t b = 0, ops = 0, comm = 0;
    for (int i = 0; i < P.n; ++i) {
        const int v = P.sigma[i];
        const uint64_t terms = 1 + P.egt[i].size() + P.children[i].size();
        ops += (uint64_t)P.tsize[i] * (uint64_t)P.K[v] * terms;
        b += (uint64_t)P.tsize[i] * (P.K[v] > 1 ? 10u : 8u);     // K = 1: no argmin table
        for (int j : P.children[i]) b += (uint64_t)P.tsize[j] * 8u;
        for (int e : P.egt[i]) b += 8ull * (uint64_t)P.K[P.edges[e].src] * (uint64_t)P.K[P.edges[e].dst];
        b += 8ull * (uint64_t)P.K[v];
        if (i < (int)ctx->vd.size() && ctx->vd[i].bcast) {   // peer bytes this rank writes
            const uint64_t mine = (uint64_t)P.tsize[i] / std::max(ctx->world, 1);
            comm += mine * ((ctx->vd[i].bcast & 1 ? 8u : 0u) + 2u) * (uint64_t)(ctx->world - 1);
        }
    }
    s.alg_bytes_dp = b;
    s.dp_fp64_ops = ops;
    s.alg_bytes_tables = 8ull * s.cost_entries;
    s.comm_bytes = comm;
    s.h2d_bytes = ctx->h2d_bytes;
    s.d2h_bytes = 16 + sizeof(int32_t) * P.n;     // one copy: total | err | pad | choice[n]
}

// Group handle blob (PASE_HANDLE_BYTES): how a peer reaches this context's pools.
struct HandleBlob {
    uint32_t magic;
    int32_t version;
    uint64_t nonce;                     // random per process: same-process peers (virtual ranks)
    int32_t device, world, rank, n;
    int64_t total_tasks;
    cudaIpcMemHandle_t h1, h2;
    uint64_t raw1, raw2;
    uint64_t off_T, off_A, off_pending, off_bar;
};
static_assert(sizeof(HandleBlob) <= PASE_HANDLE_BYTES, "handle blob too large");
constexpr uint32_t kMagic = 0x50415345;   // "PASE"

// Identifies this process among the group's (a bare pid can repeat across PID namespaces on one
// node): drawn once from the OS entropy source, mixed with the pid and the clock.
uint64_t process_nonce() {
    static const uint64_t nonce = [] {
        uint64_t x = 0;
        if (FILE* f = std::fopen("/dev/urandom", "rb")) {
            if (std::fread(&x, sizeof x, 1, f) != 1) x = 0;
            std::fclose(f);
        }
        x ^= (uint64_t)getpid() * 0x9e3779b97f4a7c15ull;
        x ^= (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
        return x | 1ull;
    }();
    return nonce;
}

}  // namespace

extern "C" {

pase_status pase_create(const pase_graph* g, int32_t p, const pase_machine* m, pase_ctx** out) {
    if (!out) return PASE_ERR_INVALID;
    *out = nullptr;
    auto t0 = std::chrono::steady_clock::now();
    pase_ctx* ctx = new (std::nothrow) pase_ctx();
    if (!ctx) { g_create_err = "out of host memory"; return PASE_ERR_RESOURCE; }
    if (!m) { g_create_err = "machine is NULL"; delete ctx; return PASE_ERR_INVALID; }
    ctx->mach = *m;
    ctx->world = std::max(1, m->world);
    ctx->rank = m->rank;
    ctx->virtual_ranks = m->virtual_ranks != 0;
    if (ctx->world > pase::kMaxWorld || ctx->rank < 0 || ctx->rank >= ctx->world) {
        g_create_err = "world must be in [1, 8] and 0 <= rank < world";
        delete ctx;
        return PASE_ERR_INVALID;
    }
    ctx->dev = m->cuda_device;
    if (const char* to = std::getenv("PASE_SPIN_TIMEOUT_MS"))      // 0 = wait without limit
        ctx->timeout_ns = (uint64_t)std::max(0ll, std::atoll(to)) * 1000000ull;
    auto fail = [&](pase_status code) {
        g_create_err = ctx->err;
        pase_destroy(ctx);
        return code;
    };
    pase_status st;
    {
        NvtxRange r("pase_create/plan (a1-a4)");
        st = pase::build_plan(g, p, m, ctx->P, ctx->err);
    }
    if (st) return fail(st);
    const bool device = ctx->dev >= 0;
    {
        const char* sc = std::getenv("PASE_SCHEDULE");
        ctx->persistent = !(sc && std::strcmp(sc, "launches") == 0) || ctx->world > 1;
        // PASE_COST_TASKS=1: the cost tables run as tasks of the persistent DP kernel instead of
        // their own kernel first (measured slower on Transformer p=64: 0.699 vs 0.682 ms per
        // solve; neutral to 2 % faster elsewhere -- profiles/r01_ab_scheduling.txt)
        const char* ct = std::getenv("PASE_COST_TASKS");
        ctx->cost_tasks = ctx->persistent && ct && ct[0] == '1';
    }
    if (!device) {                          // host-only planning context (no device work)
        ctx->nblocks = std::max(1, 2 * 148 / (ctx->virtual_ranks ? ctx->world : 1));
        auto ta = std::chrono::steady_clock::now();
        if ((st = allocate(ctx, false))) return fail(st);
        if ((st = prepare(ctx, false))) return fail(st);
        if (const char* tv = std::getenv("PASE_TIMING"); tv && tv[0] == '1')
            std::fprintf(stderr, "[pase] host-only create: plan %.3f ms, prepare %.3f ms\n",
                         std::chrono::duration<double, std::milli>(ta - t0).count(),
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count());
        fill_stats(ctx);
        ctx->stats.n_launches = 0;
        ctx->stats.ms_create =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *out = ctx;
        return PASE_OK;
    }
    {
        cudaError_t e = cudaSetDevice(ctx->dev);
        if (e != cudaSuccess) { ctx->err = std::string("cudaSetDevice: ") + cudaGetErrorString(e); return fail(PASE_ERR_CUDA); }
    }
    if (m->cuda_stream) {
        ctx->stream = (cudaStream_t)m->cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
            ctx->err = "cudaStreamCreate failed";
            return fail(PASE_ERR_CUDA);
        }
        ctx->own_stream = true;
    }
    {                                       // one pinned block: total | err | choice[n]
        void* h = pinned_get(16 + sizeof(int32_t) * ctx->P.n, &ctx->big_pinned);
        if (!h) {
            ctx->err = "cudaMallocHost failed";
            return fail(PASE_ERR_CUDA);
        }
        ctx->h_total = (double*)h;
        ctx->h_err = (int32_t*)((char*)h + 8);
        ctx->h_choice = (int32_t*)((char*)h + 16);
        const char* mo = std::getenv("PASE_MAPPED_OUT");
        if ((mo && mo[0] == '0') || cudaHostGetDevicePointer(&ctx->h_total_dev, h, 0) != cudaSuccess) {
            ctx->h_total_dev = nullptr;
            cudaGetLastError();
        }
    }
    if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        cudaEventCreate(&ctx->ev_mid) != cudaSuccess || cudaEventCreate(&ctx->ev_dp) != cudaSuccess) {
        ctx->err = "cudaEventCreate failed";
        return fail(PASE_ERR_CUDA);
    }
    {
        int sms = 0;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev) != cudaSuccess || sms < 1) {
            ctx->err = "cudaDeviceGetAttribute(MultiProcessorCount) failed";
            return fail(PASE_ERR_CUDA);
        }
        // virtual ranks share one device: each persistent grid gets 1/world of its CTA slots,
        // so all ranks' grids are co-resident (they wait on each other)
        ctx->nblocks = std::max(1, std::max(1, pase::persistent_blocks_per_sm()) * sms /
                                       (ctx->virtual_ranks ? ctx->world : 1));
    }
    ctx->async_pools = ctx->world == 1;     // groups export their pools (CUDA IPC / peer access)
    auto t_plan = std::chrono::steady_clock::now();
    if ((st = allocate(ctx, true))) return fail(st);
    auto t_alloc = std::chrono::steady_clock::now();
    {
        NvtxRange r("pase_create/prepare+upload");
        st = prepare(ctx, true);
    }
    if (st) return fail(st);
    auto t_upload = std::chrono::steady_clock::now();
    if ((st = record_graph(ctx))) return fail(st);
    // A group's pools are read by the peers' kernels (their own streams): complete them before
    // returning.  A single-GPU context touches its pools only through its own stream (solves and
    // every hook are ordered there), so the upload stays asynchronous and the pinned image goes
    // back to the cache once the first solve (or destroy) has synchronised the stream.
    if (ctx->world > 1) {
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) { ctx->err = "cudaStreamSynchronize failed"; return fail(PASE_ERR_CUDA); }
        stage_put(ctx->stage_block);
        ctx->stage_block = nullptr;
    }
    auto t_graph = std::chrono::steady_clock::now();
    fill_stats(ctx);
    using ms = std::chrono::duration<double, std::milli>;
    ctx->stats.ms_create = ms(t_graph - t0).count();
    if (const char* tv = std::getenv("PASE_TIMING"); tv && tv[0] == '1') {
        std::fprintf(stderr, "[pase] pools %p (%zu B) %p (%zu B), T at %p\n", ctx->pool, ctx->pool_bytes, ctx->pool2,
                     ctx->pool2_bytes, (void*)ctx->d_T);
        std::fprintf(stderr, "[pase] create: plan+setup %.3f ms, alloc %.3f ms, upload %.3f ms, graph %.3f ms\n",
                     ms(t_plan - t0).count(), ms(t_alloc - t_plan).count(), ms(t_upload - t_alloc).count(),
                     ms(t_graph - t_upload).count());
    }
    *out = ctx;
    return PASE_OK;
}

pase_status pase_launch(pase_ctx* ctx) {
    if (!ctx) return PASE_ERR_INVALID;
    NvtxRange r("pase_launch (a5-a8 enqueue)");
    if (ctx->dev < 0) { ctx->err = "host-only planning context: no solve"; return PASE_ERR_STATE; }
    if (ctx->world > 1 && !ctx->connected) { ctx->err = "multi-GPU context: call pase_connect first"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_launch called twice without pase_finish"; return PASE_ERR_STATE; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    const bool direct = ctx->no_graph || ctx->direct_left > 0;
    if (!direct && !ctx->exec) {
        pase_status st = issue_schedule(ctx, true);
        if (st) return st;
    }
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    if (direct) {
        pase_status st = issue_schedule(ctx, false);
        if (st) return st;
        if (ctx->direct_left > 0) --ctx->direct_left;
    } else {
        CUDA_TRY(cudaGraphLaunch(ctx->exec, ctx->stream));
    }
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    ctx->launched = true;
    return PASE_OK;
}

pase_status pase_finish(pase_ctx* ctx, int32_t* configs_out, int32_t* config_index_out, double* total_cost_out) {
    if (!ctx) return PASE_ERR_INVALID;
    if (!ctx->launched) { ctx->err = "pase_finish without pase_launch"; return PASE_ERR_STATE; }
    ctx->launched = false;
    NvtxRange r("pase_finish (wait + strategy)");
    CUDA_TRY(cudaSetDevice(ctx->dev));
    // wait for THIS solve only (its end event): work queued behind it on the same stream -- e.g.
    // the next search of a pipelined caller -- keeps running
    CUDA_TRY(cudaEventSynchronize(ctx->ev1));
    if (ctx->stage_block) {                     // the create-time upload has completed
        stage_put(ctx->stage_block);
        ctx->stage_block = nullptr;
    }
    if (*ctx->h_err) {
        const int code = *ctx->h_err;
        ctx->err = code == 3 ? std::string("DP entry without a finite candidate (cost overflow): no strategy")
                             : std::string("scheduler wait timed out after PASE_SPIN_TIMEOUT_MS (code ") +
                                   std::to_string(code) + "): ranks of the group not running concurrently?";
        return code == 3 ? PASE_ERR_RESOURCE : PASE_ERR_STATE;
    }
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    ctx->stats.ms_solve = ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev_mid));
    ctx->stats.ms_tables = ms;
    CUDA_TRY(cudaEventElapsedTime(&ms, ctx->ev_mid, ctx->ev_dp));
    ctx->stats.ms_dp = ms;
    const Plan& P = ctx->P;
    for (int v = 0; v < P.n; ++v) {
        const int c = ctx->h_choice[v];
        if (c < 0 || c >= P.K[v]) { ctx->err = "internal: back-substitution produced an invalid config"; return PASE_ERR_STATE; }
        if (config_index_out) config_index_out[v] = c;
        if (configs_out)
            for (int k = 0; k < pase::kMaxDims; ++k)
                configs_out[(size_t)v * pase::kMaxDims + k] = P.cfg[(size_t)(P.cfg_off[v] + c) * pase::kMaxDims + k];
    }
    if (total_cost_out) *total_cost_out = *ctx->h_total;
    ctx->solved = true;
    return PASE_OK;
}

pase_status pase_solve(pase_ctx* ctx, int32_t* configs_out, int32_t* config_index_out, double* total_cost_out) {
    pase_status st = pase_launch(ctx);
    if (st) return st;
    return pase_finish(ctx, configs_out, config_index_out, total_cost_out);
}

pase_status pase_export_handle(const pase_ctx* ctx_c, void* blob) {
    pase_ctx* ctx = const_cast<pase_ctx*>(ctx_c);
    if (!ctx || !blob) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context has no device memory"; return PASE_ERR_STATE; }
    HandleBlob h{};
    h.magic = kMagic;
    h.version = 1;
    h.nonce = process_nonce();
    h.device = ctx->dev;
    h.world = ctx->world;
    h.rank = ctx->rank;
    h.n = ctx->P.n;
    h.total_tasks = ctx->total_tasks;
    CUDA_TRY(cudaSetDevice(ctx->dev));
    if (!ctx->async_pools) {
        CUDA_TRY(cudaIpcGetMemHandle(&h.h1, ctx->pool));
        CUDA_TRY(cudaIpcGetMemHandle(&h.h2, ctx->pool2));
    }
    h.raw1 = (uint64_t)(uintptr_t)ctx->pool;
    h.raw2 = (uint64_t)(uintptr_t)ctx->pool2;
    h.off_T = (uint64_t)((char*)ctx->d_T - (char*)ctx->pool);
    h.off_A = (uint64_t)((char*)ctx->d_A - (char*)ctx->pool);
    h.off_pending = (uint64_t)((char*)(ctx->d_sched + pase::kSchedLine) - (char*)ctx->pool2);
    h.off_bar = (uint64_t)((char*)ctx->d_bar - (char*)ctx->pool2);
    std::memset(blob, 0, PASE_HANDLE_BYTES);
    std::memcpy(blob, &h, sizeof h);
    return PASE_OK;
}

pase_status pase_connect(pase_ctx* ctx, const void* blobs) {
    if (!ctx || !blobs) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context cannot connect"; return PASE_ERR_STATE; }
    if (ctx->connected) { ctx->err = "already connected"; return PASE_ERR_STATE; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    std::vector<double*> Tb(ctx->world);
    std::vector<uint16_t*> Ab(ctx->world);
    for (int q = 0; q < ctx->world; ++q) {
        HandleBlob h;
        std::memcpy(&h, (const char*)blobs + (size_t)q * PASE_HANDLE_BYTES, sizeof h);
        if (h.magic != kMagic || h.world != ctx->world || h.rank != q || h.n != ctx->P.n ||
            h.total_tasks != ctx->total_tasks) {
            ctx->err = "pase_connect: handle " + std::to_string(q) + " does not belong to this group / plan";
            return PASE_ERR_INVALID;
        }
        char *b1, *b2;
        if (q == ctx->rank) {
            b1 = (char*)ctx->pool;
            b2 = (char*)ctx->pool2;
        } else if (h.nonce == process_nonce()) {        // virtual ranks in one process
            b1 = (char*)(uintptr_t)h.raw1;
            b2 = (char*)(uintptr_t)h.raw2;
            if (h.device != ctx->dev) {
                cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    ctx->err = std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
                    return PASE_ERR_CUDA;
                }
                cudaGetLastError();
            }
        } else {                                        // another process: IPC over NVLink
            void *p1 = nullptr, *p2 = nullptr;
            CUDA_TRY(cudaIpcOpenMemHandle(&p1, h.h1, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_opened.push_back(p1);
            CUDA_TRY(cudaIpcOpenMemHandle(&p2, h.h2, cudaIpcMemLazyEnablePeerAccess));
            ctx->ipc_opened.push_back(p2);
            b1 = (char*)p1;
            b2 = (char*)p2;
        }
        Tb[q] = (double*)(b1 + h.off_T);
        Ab[q] = (uint16_t*)(b1 + h.off_A);
        ctx->peers.pending[q] = (int32_t*)(b2 + h.off_pending);
        ctx->peers.bar[q] = (int32_t*)(b2 + h.off_bar);
    }
    for (int i = 0; i < ctx->P.n; ++i) {
        VertexDesc& d = ctx->vd[i];
        int k = 0;
        for (int q = 0; q < ctx->world; ++q) {
            if (q == ctx->rank) continue;
            d.Tpeer[k] = Tb[q] + ctx->P.toff[i];
            d.Apeer[k] = Ab[q] + ctx->P.toff[i];
            ++k;
        }
    }
    // ordered on the context's stream (the solves run there), complete before return: vd is
    // pageable host memory
    CUDA_TRY(cudaMemcpyAsync(ctx->d_vd, ctx->vd.data(), sizeof(VertexDesc) * ctx->P.n, cudaMemcpyHostToDevice,
                             ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->peer_T = Tb;
    ctx->connected = true;
    return record_graph(ctx);
}

int64_t pase_get_schedule(const pase_ctx* ctx, int32_t* vinfo, int64_t* tasks, int32_t* order) {
    if (!ctx) return -1;
    const int n = ctx->P.n;
    if (vinfo)
        for (int i = 0; i < n; ++i) {
            int32_t* o = vinfo + 8 * i;
            o[0] = ctx->vd[i].part;
            o[1] = ctx->vd[i].bcast;
            o[2] = ctx->vd[i].ntasks;
            o[3] = ctx->sp.pending[i];
            o[4] = ctx->vd[i].shape;
            o[5] = ctx->vd[i].glog;
            o[6] = ctx->vd[i].wlog;
            o[7] = ctx->vd[i].q2;
        }
    if (tasks)
        for (size_t t = 0; t < ctx->sp.tasks.size(); ++t) {
            tasks[4 * t + 0] = ctx->sp.tasks[t].vtx;
            tasks[4 * t + 1] = ctx->sp.tasks[t].i0;
            tasks[4 * t + 2] = ctx->sp.tasks[t].i1;
            tasks[4 * t + 3] = ctx->sp.tasks[t].glog;
        }
    if (order) std::copy(ctx->sp.order.begin(), ctx->sp.order.end(), order);
    return (int64_t)ctx->sp.tasks.size();
}

pase_status pase_get_stats(const pase_ctx* ctx, pase_stats* out) {
    if (!ctx || !out) return PASE_ERR_INVALID;
    *out = ctx->stats;
    return PASE_OK;
}

const char* pase_last_error(const pase_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

void pase_destroy(pase_ctx* ctx) {
    if (!ctx) return;
    if (ctx->dev < 0) { delete ctx; return; }
    cudaSetDevice(ctx->dev);
    if ((ctx->launched || ctx->stage_block) && ctx->stream) cudaStreamSynchronize(ctx->stream);
    stage_put(ctx->stage_block);                // failed create: upload image back to the cache
    if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
    for (auto s : ctx->aux) cudaStreamDestroy(s);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev_mid) cudaEventDestroy(ctx->ev_mid);
    if (ctx->ev_dp) cudaEventDestroy(ctx->ev_dp);
    for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    if (ctx->async_pools) {                 // back to the cached pool, ordered after our work
        if (ctx->pool) cudaFreeAsync(ctx->pool, ctx->stream);
        if (ctx->pool2) cudaFreeAsync(ctx->pool2, ctx->stream);
    } else {
        if (ctx->pool) cudaFree(ctx->pool);
        if (ctx->pool2) cudaFree(ctx->pool2);
    }
    pinned_put(ctx->h_total, ctx->big_pinned);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

pase_status pase_get_configs(const pase_ctx* ctx, int32_t* counts, int32_t* tuples) {
    if (!ctx) return PASE_ERR_INVALID;
    const Plan& P = ctx->P;
    if (counts) std::copy(P.K.begin(), P.K.end(), counts);
    if (tuples)                                   // per node in id order (shared blocks expanded)
        for (int v = 0, o = 0; v < P.n; o += P.K[v], ++v)
            std::copy(P.cfg.begin() + P.cfg_off[v] * pase::kMaxDims, P.cfg.begin() + (P.cfg_off[v] + P.K[v]) * pase::kMaxDims,
                      tuples + (size_t)o * pase::kMaxDims);
    return PASE_OK;
}

pase_status pase_get_order(const pase_ctx* ctx, int32_t* sigma, int32_t* dep_off, int32_t* dep_ids,
                           int32_t* parent) {
    if (!ctx) return PASE_ERR_INVALID;
    const Plan& P = ctx->P;
    if (sigma) std::copy(P.sigma.begin(), P.sigma.end(), sigma);
    if (parent) std::copy(P.parent.begin(), P.parent.end(), parent);
    int pos = 0;
    for (int i = 0; i < P.n; ++i) {
        if (dep_off) dep_off[i] = pos;
        for (int u : P.dep[i]) {
            if (dep_ids) dep_ids[pos] = u;
            ++pos;
        }
    }
    if (dep_off) dep_off[P.n] = pos;
    return PASE_OK;
}

pase_status pase_get_cost_tables(const pase_ctx* ctx_c, int32_t index, int32_t is_edge, double* out) {
    pase_ctx* ctx = const_cast<pase_ctx*>(ctx_c);
    if (!ctx || !out) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context has no device tables"; return PASE_ERR_STATE; }
    const Plan& P = ctx->P;
    if (!ctx->solved && !ctx->override_tables) { ctx->err = "call pase_solve first"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_get_cost_tables during a launched solve"; return PASE_ERR_STATE; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    if (!is_edge) {
        if (index < 0 || index >= P.n) return PASE_ERR_INVALID;
        CUDA_TRY(cudaMemcpyAsync(out, ctx->d_L + P.loff[index], sizeof(double) * P.K[index], cudaMemcpyDeviceToHost,
                                 ctx->stream));
        CUDA_TRY(cudaStreamSynchronize(ctx->stream));
        return PASE_OK;
    }
    if (index < 0 || index >= P.m) return PASE_ERR_INVALID;
    const pase_edge& e = P.edges[index];
    const int ks = P.K[e.src], kd = P.K[e.dst];
    std::vector<double> buf((size_t)ks * kd);
    CUDA_TRY(cudaMemcpyAsync(buf.data(), ctx->d_W + P.woff[index], sizeof(double) * buf.size(), cudaMemcpyDeviceToHost,
                             ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const bool later_is_src = P.rank[e.src] > P.rank[e.dst];
    for (int cs = 0; cs < ks; ++cs)
        for (int cd = 0; cd < kd; ++cd)
            out[(size_t)cs * kd + cd] = later_is_src ? buf[(size_t)cs * kd + cd] : buf[(size_t)cd * ks + cs];
    return PASE_OK;
}

int64_t pase_table_entries(const pase_ctx* ctx, int32_t rank) {
    if (!ctx || rank < 0 || rank >= ctx->P.n) return -1;
    return ctx->P.tsize[rank];
}

pase_status pase_get_dp_table(const pase_ctx* ctx_c, int32_t rank, double* T_out, uint16_t* A_out) {
    pase_ctx* ctx = const_cast<pase_ctx*>(ctx_c);
    if (!ctx || rank < 0 || rank >= ctx->P.n) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context has no device tables"; return PASE_ERR_STATE; }
    if (!ctx->solved) { ctx->err = "call pase_solve first"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_get_dp_table during a launched solve"; return PASE_ERR_STATE; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    const int64_t sz = ctx->P.tsize[rank], off = ctx->P.toff[rank];
    if (T_out) CUDA_TRY(cudaMemcpyAsync(T_out, ctx->d_T + off, sizeof(double) * sz, cudaMemcpyDeviceToHost, ctx->stream));
    if (A_out && ctx->vd[rank].K == 1) std::memset(A_out, 0, sizeof(uint16_t) * sz);   // not stored
    else if (A_out) CUDA_TRY(cudaMemcpyAsync(A_out, ctx->d_A + off, sizeof(uint16_t) * sz, cudaMemcpyDeviceToHost, ctx->stream));
    // multi-GPU: a partitioned table whose T is not broadcast holds only this rank's slice
    // (configs [q K/G, (q+1) K/G) of its top coordinate, the slowest): gather the others'
    // slices from their pools through the peer mappings (argmin tables are always complete)
    const VertexDesc& d = ctx->vd[rank];
    if (T_out && ctx->world > 1 && d.part && !(d.bcast & 1) && ctx->connected) {
        const int64_t Kt = d.radix[d.m - 1], S = sz / Kt;
        for (int q = 0; q < ctx->world; ++q) {
            if (q == ctx->rank) continue;
            const int64_t lo = q * Kt / ctx->world * S, hi = (q + 1) * Kt / ctx->world * S;
            if (hi > lo)
                CUDA_TRY(cudaMemcpyAsync(T_out + lo, ctx->peer_T[q] + off + lo, sizeof(double) * (hi - lo),
                                         cudaMemcpyDefault, ctx->stream));
        }
    }
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return PASE_OK;
}

pase_status pase_set_cost_tables(pase_ctx* ctx, const double* L, const double* W) {
    if (!ctx || !L || (!W && ctx->P.m > 0)) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context has no device tables"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_set_cost_tables during a launched solve"; return PASE_ERR_STATE; }
    const Plan& P = ctx->P;
    // Eq. 1 costs are finite (a non-finite candidate would leave a DP entry without argmin)
    for (int64_t k = 0; k < P.loff[P.n]; ++k)
        if (!std::isfinite(L[k])) { ctx->err = "pase_set_cost_tables: L[" + std::to_string(k) + "] is not finite"; return PASE_ERR_INVALID; }
    for (int64_t k = 0; k < P.woff[P.m]; ++k)
        if (!std::isfinite(W[k])) { ctx->err = "pase_set_cost_tables: W[" + std::to_string(k) + "] is not finite"; return PASE_ERR_INVALID; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    // one pageable staging buffer in the device layout, copied on the context's stream (the
    // solves' stream) and complete before return
    std::vector<double> buf((size_t)(P.loff[P.n] + P.woff[P.m]));
    std::memcpy(buf.data(), L, sizeof(double) * P.loff[P.n]);
    for (int e = 0; e < P.m; ++e) {          // src-major input -> [later][earlier] device layout
        const pase_edge& x = P.edges[e];
        const int ks = P.K[x.src], kd = P.K[x.dst];
        const double* w = W + P.woff[e];
        double* o = buf.data() + P.loff[P.n] + P.woff[e];
        const bool later_is_src = P.rank[x.src] > P.rank[x.dst];
        for (int cs = 0; cs < ks; ++cs)
            for (int cd = 0; cd < kd; ++cd)
                (later_is_src ? o[(size_t)cs * kd + cd] : o[(size_t)cd * ks + cs]) = w[(size_t)cs * kd + cd];
    }
    CUDA_TRY(cudaMemcpyAsync(ctx->d_L, buf.data(), sizeof(double) * P.loff[P.n], cudaMemcpyHostToDevice, ctx->stream));
    if (P.m > 0)
        CUDA_TRY(cudaMemcpyAsync(ctx->d_W, buf.data() + P.loff[P.n], sizeof(double) * P.woff[P.m],
                                 cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (!ctx->override_tables) {
        ctx->override_tables = true;
        pase_status st = record_graph(ctx);
        if (st) return st;
    }
    return PASE_OK;
}

int64_t pase_get_trace(const pase_ctx* ctx_c, int64_t* out, int64_t cap) {
    pase_ctx* ctx = const_cast<pase_ctx*>(ctx_c);
    if (!ctx || ctx->dev < 0 || !ctx->d_trace || !trace_on()) return 0;
    const int64_t nt = std::min<int64_t>(ctx->ntasks, cap);
    if (out && nt > 0 && (cudaMemcpyAsync(out, ctx->d_trace, sizeof(int64_t) * pase::kTraceWords * nt,
                                          cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
                          cudaStreamSynchronize(ctx->stream) != cudaSuccess))
        return -1;
    return ctx->ntasks;
}

pase_status pase_set_profiling(pase_ctx* ctx, int32_t enable) {
    if (!ctx) return PASE_ERR_INVALID;
    ctx->profiling = enable;
    return PASE_OK;
}

// ---- row f2: Eq. 1 on the GPU (eval.cu) ----------------------------------------------------
namespace {
// The cost tables the Eq. 1 kernels read: the cost-table kernel's output (recomputed on the
// context's stream) unless pase_set_cost_tables replaced them.  Also uploads the W_e index
// records (row = later endpoint: the DP layout) into a stream-ordered temporary.
pase_status eq1_prepare(pase_ctx* ctx, pase::EvalEdge** ed_dev) {
    const Plan& P = ctx->P;
    CUDA_TRY(cudaSetDevice(ctx->dev));
    if (!ctx->override_tables) pase::launch_cost_tables(cost_args(ctx), ctx->nchunks, ctx->stream);
    std::vector<pase::EvalEdge> ed(std::max(P.m, 1));
    for (int e = 0; e < P.m; ++e) {
        const pase_edge& x = P.edges[e];
        const bool later_is_src = P.rank[x.src] > P.rank[x.dst];
        ed[e].row = later_is_src ? x.src : x.dst;
        ed[e].col = later_is_src ? x.dst : x.src;
        ed[e].kcol = P.K[ed[e].col];
        ed[e].pad = 0;
        ed[e].off = P.woff[e];
    }
    CUDA_TRY(cudaMallocAsync((void**)ed_dev, sizeof(pase::EvalEdge) * ed.size(), ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(*ed_dev, ed.data(), sizeof(pase::EvalEdge) * ed.size(), cudaMemcpyHostToDevice,
                             ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));         // ed (pageable) consumed
    return PASE_OK;
}
}  // namespace

pase_status pase_evaluate(pase_ctx* ctx, const int32_t* config_index, int64_t n_strategies, double* cost_out) {
    if (!ctx || n_strategies < 0 || (n_strategies > 0 && (!config_index || !cost_out))) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context: no device evaluation"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_evaluate during a launched solve"; return PASE_ERR_STATE; }
    const Plan& P = ctx->P;
    for (int64_t s = 0; s < n_strategies; ++s)
        for (int v = 0; v < P.n; ++v) {
            const int32_t c = config_index[s * P.n + v];
            if (c < 0 || c >= P.K[v]) {
                ctx->err = "pase_evaluate: strategy " + std::to_string(s) + ", node " + std::to_string(v) +
                           ": config index " + std::to_string(c) + " outside [0, " + std::to_string(P.K[v]) + ")";
                return PASE_ERR_INVALID;
            }
        }
    pase::EvalEdge* ed = nullptr;
    pase_status st = eq1_prepare(ctx, &ed);
    if (st) return st;
    if (n_strategies > 0) {
        int32_t* d_s = nullptr;
        double* d_c = nullptr;
        const size_t sb = sizeof(int32_t) * (size_t)n_strategies * P.n, cb = sizeof(double) * (size_t)n_strategies;
        CUDA_TRY(cudaMallocAsync((void**)&d_s, sb, ctx->stream));
        CUDA_TRY(cudaMallocAsync((void**)&d_c, cb, ctx->stream));
        CUDA_TRY(cudaMemcpyAsync(d_s, config_index, sb, cudaMemcpyHostToDevice, ctx->stream));
        pase::launch_eval(P.n, P.m, ctx->d_loff, ctx->d_L, ed, ctx->d_W, d_s, n_strategies, d_c, ctx->stream);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaMemcpyAsync(cost_out, d_c, cb, cudaMemcpyDeviceToHost, ctx->stream));
        CUDA_TRY(cudaFreeAsync(d_s, ctx->stream));
        CUDA_TRY(cudaFreeAsync(d_c, ctx->stream));
    }
    CUDA_TRY(cudaFreeAsync(ed, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return PASE_OK;
}

pase_status pase_brute_force(pase_ctx* ctx, uint64_t max_strategies, int32_t* config_index_out,
                             double* total_cost_out, uint64_t* n_strategies_out) {
    if (!ctx) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context: no device search"; return PASE_ERR_STATE; }
    if (ctx->launched) { ctx->err = "pase_brute_force during a launched solve"; return PASE_ERR_STATE; }
    const Plan& P = ctx->P;
    const uint64_t cap = max_strategies ? max_strategies : (1ull << 40);
    uint64_t total = 1;
    for (int v = 0; v < P.n; ++v) {
        if (total > cap / (uint64_t)P.K[v]) {
            ctx->err = "brute force: prod_v K_v exceeds the limit of " + std::to_string(cap) + " strategies";
            return PASE_ERR_RESOURCE;
        }
        total *= (uint64_t)P.K[v];
    }
    if (n_strategies_out) *n_strategies_out = total;
    int maxsm = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->dev));
    if (pase::brute_smem_bytes(P.n, P.m) > (size_t)maxsm) {
        ctx->err = "brute force: graph too large for the shared-memory odometer (" + std::to_string(P.n) + " nodes)";
        return PASE_ERR_RESOURCE;
    }
    pase::EvalEdge* ed = nullptr;
    pase_status st = eq1_prepare(ctx, &ed);
    if (st) return st;
    int sms = 148;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
    const uint64_t want = (total + pase::kBruteThreads - 1) / pase::kBruteThreads;
    const int nblocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * 16, want));
    double* d_b = nullptr;
    uint64_t* d_i = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&d_b, sizeof(double) * (nblocks + 1), ctx->stream));
    CUDA_TRY(cudaMallocAsync((void**)&d_i, sizeof(uint64_t) * (nblocks + 1), ctx->stream));
    if (pase::launch_brute(P.n, P.m, ctx->d_K, ctx->d_loff, ctx->d_L, ed, ctx->d_W, total, nblocks, d_b, d_i,
                           d_b + nblocks, d_i + nblocks, ctx->stream)) {
        ctx->err = "brute force: cannot reserve shared memory";
        return PASE_ERR_CUDA;
    }
    CUDA_TRY(cudaGetLastError());
    double best = 0.0;
    uint64_t bi = 0;
    CUDA_TRY(cudaMemcpyAsync(&best, d_b + nblocks, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(&bi, d_i + nblocks, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaFreeAsync(d_b, ctx->stream));
    CUDA_TRY(cudaFreeAsync(d_i, ctx->stream));
    CUDA_TRY(cudaFreeAsync(ed, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (bi >= total) { ctx->err = "internal: brute force found no strategy"; return PASE_ERR_STATE; }
    for (int v = 0; v < P.n; ++v) {                          // mixed radix, node 0 fastest
        if (config_index_out) config_index_out[v] = (int32_t)(bi % (uint64_t)P.K[v]);
        bi /= (uint64_t)P.K[v];
    }
    if (total_cost_out) *total_cost_out = best;
    return PASE_OK;
}

// ---- row f3: device assignment (assign.cpp) ------------------------------------------------
pase_status pase_assign_devices(const pase_ctx* ctx_c, const int32_t* config_index, int32_t* device_out,
                                double* tx_out) {
    pase_ctx* ctx = const_cast<pase_ctx*>(ctx_c);
    if (!ctx || !config_index) return PASE_ERR_INVALID;
    return pase::assign_devices(ctx->P, config_index, device_out, tx_out, ctx->err);
}

}  // extern "C"
