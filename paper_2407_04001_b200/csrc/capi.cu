// capi.cu -- the C ABI of include/pase.h: context lifecycle, device memory, the solve
// schedule recorded once as a CUDA graph (cost tables -> DP fill over the elimination
// tree, children before parents, independent subtrees concurrent -> back-substitution ->
// D2H of the strategy), and the introspection hooks.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "pase_internal.h"

using pase::EdgeDesc;
using pase::Plan;
using pase::TermDesc;
using pase::VertexDesc;

struct pase_ctx {
    Plan P;
    pase_machine mach{};
    std::string err;
    int dev = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::vector<cudaStream_t> aux;          // fork streams for concurrent subtrees
    // device memory
    void* pool = nullptr;
    size_t pool_bytes = 0;
    pase_node* d_nodes = nullptr;
    int32_t* d_K = nullptr;
    int64_t* d_cfg_off = nullptr;
    int32_t* d_cfg = nullptr;
    int64_t* d_loff = nullptr;
    EdgeDesc* d_edges = nullptr;
    int64_t* d_item_off = nullptr;
    double* d_L = nullptr;
    double* d_W = nullptr;
    double* d_T = nullptr;
    uint16_t* d_A = nullptr;
    VertexDesc* d_vd = nullptr;
    TermDesc* d_td = nullptr;
    int32_t* d_sigma = nullptr;
    int32_t* d_dep_off = nullptr;
    int32_t* d_dep_ids = nullptr;
    int32_t* d_choice = nullptr;
    double* d_total = nullptr;
    // host mirrors
    std::vector<VertexDesc> vd;
    std::vector<TermDesc> td;
    int32_t* h_choice = nullptr;            // pinned
    double* h_total = nullptr;              // pinned
    int64_t cost_total = 0;
    bool override_tables = false;
    bool solved = false;
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

// Carve all device buffers out of one allocation.
pase_status allocate(pase_ctx* ctx) {
    const Plan& P = ctx->P;
    const int n = P.n, m = P.m;
    const int64_t nterms_total = [&] {
        int64_t t = 0;
        for (int i = 0; i < n; ++i) t += 1 + (int64_t)P.egt[i].size() + (int64_t)P.children[i].size();
        return t;
    }();
    struct Item { void** ptr; size_t bytes; };
    const int64_t ncfg = P.cfg_off[n];
    std::vector<Item> items = {
        {(void**)&ctx->d_nodes, sizeof(pase_node) * n},
        {(void**)&ctx->d_K, sizeof(int32_t) * n},
        {(void**)&ctx->d_cfg_off, sizeof(int64_t) * (n + 1)},
        {(void**)&ctx->d_cfg, sizeof(int32_t) * pase::kMaxDims * ncfg},
        {(void**)&ctx->d_loff, sizeof(int64_t) * (n + 1)},
        {(void**)&ctx->d_edges, sizeof(EdgeDesc) * std::max(m, 1)},
        {(void**)&ctx->d_item_off, sizeof(int64_t) * (n + m + 1)},
        {(void**)&ctx->d_L, sizeof(double) * P.loff[n]},
        {(void**)&ctx->d_W, sizeof(double) * std::max<int64_t>(P.woff[m], 1)},
        {(void**)&ctx->d_T, sizeof(double) * P.toff[n]},
        {(void**)&ctx->d_A, sizeof(uint16_t) * P.toff[n]},
        {(void**)&ctx->d_vd, sizeof(VertexDesc) * n},
        {(void**)&ctx->d_td, sizeof(TermDesc) * nterms_total},
        {(void**)&ctx->d_sigma, sizeof(int32_t) * n},
        {(void**)&ctx->d_dep_off, sizeof(int32_t) * (n + 1)},
        {(void**)&ctx->d_dep_ids, sizeof(int32_t) * std::max<int64_t>((int64_t)n * pase::kMaxDep, 1)},
        {(void**)&ctx->d_choice, sizeof(int32_t) * n},
        {(void**)&ctx->d_total, sizeof(double)},
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
    cudaError_t e = cudaMalloc(&ctx->pool, total);
    if (e != cudaSuccess) {
        ctx->err = std::string("cudaMalloc of ") + std::to_string(total) + " bytes failed: " + cudaGetErrorString(e);
        return PASE_ERR_RESOURCE;
    }
    ctx->pool_bytes = total;
    char* p = (char*)ctx->pool;
    for (auto& it : items) { *it.ptr = p; p += align_up(it.bytes); }
    return PASE_OK;
}

// Build vertex/term descriptors (DESIGN §4 layout) and upload all static inputs.
pase_status upload(pase_ctx* ctx) {
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
    std::vector<int64_t> item_off(n + m + 1, 0);
    for (int v = 0; v < n; ++v) item_off[v + 1] = item_off[v] + P.K[v];
    for (int e = 0; e < m; ++e)
        item_off[n + e + 1] = item_off[n + e] + (int64_t)P.K[P.edges[e].src] * P.K[P.edges[e].dst];
    ctx->cost_total = item_off[n + m];

    ctx->vd.assign(n, VertexDesc{});
    ctx->td.clear();
    std::vector<int32_t> dep_off(n + 1, 0), dep_ids;
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
        auto pos_of = [&](int node) {
            for (int q = 0; q < d.m; ++q) if (P.dep[i][q] == node) return q;
            return -1;
        };
        TermDesc t{};
        // term 0: L_{sigma_i}[C]
        t.base = ctx->d_L + P.loff[v];
        ctx->td.push_back(t);
        // edges to later neighbours, canonical order: row = config of the other endpoint
        for (int e : P.egt[i]) {
            TermDesc te{};
            const int other = P.edges[e].src == v ? P.edges[e].dst : P.edges[e].src;
            const int q = pos_of(other);
            if (q < 0) { ctx->err = "internal: E>(sigma_i) endpoint outside D(i)"; return PASE_ERR_STATE; }
            te.base = ctx->d_W + P.woff[e];
            te.stride[q] = d.K;
            ctx->td.push_back(te);
        }
        // children ascending rank: T_j coordinates (sigma_i, w_1, ...) with sigma_i fastest
        for (int j : P.children[i]) {
            TermDesc tc{};
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
        dep_off[i] = (int32_t)dep_ids.size();
        dep_ids.insert(dep_ids.end(), P.dep[i].begin(), P.dep[i].end());
    }
    dep_off[n] = (int32_t)dep_ids.size();
    if (dep_ids.empty()) dep_ids.push_back(0);
    cudaStream_t s = ctx->stream;
    ctx->h2d_bytes = sizeof(pase_node) * n + sizeof(int32_t) * n + sizeof(int64_t) * (n + 1) * 2 +
                     sizeof(int32_t) * P.cfg.size() + sizeof(EdgeDesc) * ed.size() +
                     sizeof(int64_t) * (n + m + 1) + sizeof(VertexDesc) * n + sizeof(TermDesc) * ctx->td.size() +
                     sizeof(int32_t) * (2 * n + 1 + dep_ids.size());
    CUDA_TRY(cudaMemcpyAsync(ctx->d_nodes, P.nodes.data(), sizeof(pase_node) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_K, P.K.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_cfg_off, P.cfg_off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_cfg, P.cfg.data(), sizeof(int32_t) * P.cfg.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_loff, P.loff.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_edges, ed.data(), sizeof(EdgeDesc) * ed.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_item_off, item_off.data(), sizeof(int64_t) * (n + m + 1), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_vd, ctx->vd.data(), sizeof(VertexDesc) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_td, ctx->td.data(), sizeof(TermDesc) * ctx->td.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_sigma, P.sigma.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_dep_off, dep_off.data(), sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->d_dep_ids, dep_ids.data(), sizeof(int32_t) * dep_ids.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaStreamSynchronize(s));   // host vectors above are stack-local
    return PASE_OK;
}

// Record the whole solve as one CUDA graph.  DP kernels are issued in rank order; a vertex
// waits on its children's events only, so independent subtrees overlap.
pase_status record_graph(pase_ctx* ctx) {
    const Plan& P = ctx->P;
    const int n = P.n;
    if (ctx->exec) { cudaGraphExecDestroy(ctx->exec); ctx->exec = nullptr; }
    const int nstreams = 4;
    if (ctx->aux.empty()) {
        ctx->aux.resize(nstreams);
        for (auto& s : ctx->aux) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    std::vector<cudaEvent_t> done(n);
    for (auto& e : done) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t start;
    CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    std::vector<cudaEvent_t> join(nstreams);
    for (auto& e : join) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaStream_t s = ctx->stream;
    CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    if (!ctx->override_tables)
        pase::launch_cost_tables(ctx->d_nodes, ctx->d_K, ctx->d_cfg_off, ctx->d_cfg, ctx->d_loff, n,
                                 ctx->d_edges, P.m, ctx->d_item_off, ctx->cost_total, P.r, ctx->d_L,
                                 ctx->d_W, s);
    // phase split: external event nodes (plain records would only become capture edges)
    CUDA_TRY(cudaEventRecordWithFlags(ctx->ev_mid, s, cudaEventRecordExternal));
    CUDA_TRY(cudaEventRecord(start, s));
    std::vector<char> used(nstreams, 0);
    // assign each vertex the stream of its first child (chains stay on one stream)
    std::vector<int> sid(n, -1);
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
    CUDA_TRY(cudaEventRecordWithFlags(ctx->ev_dp, s, cudaEventRecordExternal));
    pase::launch_backtrack(ctx->d_sigma, ctx->d_dep_off, ctx->d_dep_ids, ctx->d_vd, n, ctx->d_choice,
                           ctx->d_total, s);
    CUDA_TRY(cudaMemcpyAsync(ctx->h_choice, ctx->d_choice, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(ctx->h_total, ctx->d_total, sizeof(double), cudaMemcpyDeviceToHost, s));
    cudaGraph_t graph;
    cudaError_t ce = cudaStreamEndCapture(s, &graph);
    for (auto& e : done) cudaEventDestroy(e);
    for (auto& e : join) cudaEventDestroy(e);
    cudaEventDestroy(start);
    if (ce != cudaSuccess) { ctx->err = std::string("stream capture: ") + cudaGetErrorString(ce); return PASE_ERR_CUDA; }
    ce = cudaGraphInstantiate(&ctx->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) { ctx->err = std::string("graph instantiate: ") + cudaGetErrorString(ce); return PASE_ERR_CUDA; }
    ctx->stats.n_launches = (ctx->override_tables ? 0 : 1) + n + 1;
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
    uint64_t b = 0, ops = 0;
    for (int i = 0; i < P.n; ++i) {
        const int v = P.sigma[i];
        const uint64_t terms = 1 + P.egt[i].size() + P.children[i].size();
        ops += (uint64_t)P.tsize[i] * (uint64_t)P.K[v] * terms;
        b += (uint64_t)P.tsize[i] * 10u;
        for (int j : P.children[i]) b += (uint64_t)P.tsize[j] * 8u;
        for (int e : P.egt[i]) b += 8ull * (uint64_t)P.K[P.edges[e].src] * (uint64_t)P.K[P.edges[e].dst];
        b += 8ull * (uint64_t)P.K[v];
    }
    s.alg_bytes_dp = b;
    s.dp_fp64_ops = ops;
    s.alg_bytes_tables = 8ull * s.cost_entries;
    s.comm_bytes = 0;
    s.h2d_bytes = ctx->h2d_bytes;
    s.d2h_bytes = sizeof(int32_t) * P.n + sizeof(double);
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
    if (m->world > 1) {
        g_create_err = "multi-GPU contexts (world > 1) are not supported by this build";
        delete ctx;
        return PASE_ERR_INVALID;
    }
    pase_status st = pase::build_plan(g, p, m, ctx->P, ctx->err);
    auto fail = [&](pase_status code) {
        g_create_err = ctx->err;
        pase_destroy(ctx);
        return code;
    };
    if (st) return fail(st);
    ctx->dev = m->cuda_device;
    if (ctx->dev < 0) {                      // host-only planning context (no device work)
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
    if (cudaMallocHost(&ctx->h_choice, sizeof(int32_t) * ctx->P.n) != cudaSuccess ||
        cudaMallocHost(&ctx->h_total, sizeof(double)) != cudaSuccess) {
        ctx->err = "cudaMallocHost failed";
        return fail(PASE_ERR_CUDA);
    }
    if (cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        cudaEventCreate(&ctx->ev_mid) != cudaSuccess || cudaEventCreate(&ctx->ev_dp) != cudaSuccess) {
        ctx->err = "cudaEventCreate failed";
        return fail(PASE_ERR_CUDA);
    }
    if ((st = allocate(ctx))) return fail(st);
    if ((st = upload(ctx))) return fail(st);
    if ((st = record_graph(ctx))) return fail(st);
    fill_stats(ctx);
    ctx->stats.ms_create =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *out = ctx;
    return PASE_OK;
}

pase_status pase_solve(pase_ctx* ctx, int32_t* configs_out, int32_t* config_index_out, double* total_cost_out) {
    if (!ctx) return PASE_ERR_INVALID;
    if (!ctx->exec) { ctx->err = "context has no solve schedule (host-only planning context?)"; return PASE_ERR_STATE; }
    CUDA_TRY(cudaSetDevice(ctx->dev));
    CUDA_TRY(cudaEventRecord(ctx->ev0, ctx->stream));
    CUDA_TRY(cudaGraphLaunch(ctx->exec, ctx->stream));
    CUDA_TRY(cudaEventRecord(ctx->ev1, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
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
    if (ctx->exec) cudaGraphExecDestroy(ctx->exec);
    for (auto s : ctx->aux) cudaStreamDestroy(s);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev_mid) cudaEventDestroy(ctx->ev_mid);
    if (ctx->ev_dp) cudaEventDestroy(ctx->ev_dp);
    if (ctx->pool) cudaFree(ctx->pool);
    if (ctx->h_choice) cudaFreeHost(ctx->h_choice);
    if (ctx->h_total) cudaFreeHost(ctx->h_total);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

pase_status pase_get_configs(const pase_ctx* ctx, int32_t* counts, int32_t* tuples) {
    if (!ctx) return PASE_ERR_INVALID;
    const Plan& P = ctx->P;
    if (counts) std::copy(P.K.begin(), P.K.end(), counts);
    if (tuples) std::copy(P.cfg.begin(), P.cfg.end(), tuples);
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
    CUDA_TRY(cudaSetDevice(ctx->dev));
    if (!is_edge) {
        if (index < 0 || index >= P.n) return PASE_ERR_INVALID;
        CUDA_TRY(cudaMemcpy(out, ctx->d_L + P.loff[index], sizeof(double) * P.K[index], cudaMemcpyDeviceToHost));
        return PASE_OK;
    }
    if (index < 0 || index >= P.m) return PASE_ERR_INVALID;
    const pase_edge& e = P.edges[index];
    const int ks = P.K[e.src], kd = P.K[e.dst];
    std::vector<double> buf((size_t)ks * kd);
    CUDA_TRY(cudaMemcpy(buf.data(), ctx->d_W + P.woff[index], sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
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
    CUDA_TRY(cudaSetDevice(ctx->dev));
    const int64_t sz = ctx->P.tsize[rank], off = ctx->P.toff[rank];
    if (T_out) CUDA_TRY(cudaMemcpy(T_out, ctx->d_T + off, sizeof(double) * sz, cudaMemcpyDeviceToHost));
    if (A_out) CUDA_TRY(cudaMemcpy(A_out, ctx->d_A + off, sizeof(uint16_t) * sz, cudaMemcpyDeviceToHost));
    return PASE_OK;
}

pase_status pase_set_cost_tables(pase_ctx* ctx, const double* L, const double* W) {
    if (!ctx || !L || (!W && ctx->P.m > 0)) return PASE_ERR_INVALID;
    if (ctx->dev < 0) { ctx->err = "host-only planning context has no device tables"; return PASE_ERR_STATE; }
    const Plan& P = ctx->P;
    CUDA_TRY(cudaSetDevice(ctx->dev));
    CUDA_TRY(cudaMemcpy(ctx->d_L, L, sizeof(double) * P.loff[P.n], cudaMemcpyHostToDevice));
    std::vector<double> buf;
    for (int e = 0; e < P.m; ++e) {          // src-major input -> [later][earlier] device layout
        const pase_edge& x = P.edges[e];
        const int ks = P.K[x.src], kd = P.K[x.dst];
        const double* w = W + P.woff[e];
        buf.resize((size_t)ks * kd);
        const bool later_is_src = P.rank[x.src] > P.rank[x.dst];
        for (int cs = 0; cs < ks; ++cs)
            for (int cd = 0; cd < kd; ++cd)
                (later_is_src ? buf[(size_t)cs * kd + cd] : buf[(size_t)cd * ks + cs]) = w[(size_t)cs * kd + cd];
        CUDA_TRY(cudaMemcpy(ctx->d_W + P.woff[e], buf.data(), sizeof(double) * buf.size(), cudaMemcpyHostToDevice));
    }
    if (!ctx->override_tables) {
        ctx->override_tables = true;
        pase_status st = record_graph(ctx);
        if (st) return st;
    }
    return PASE_OK;
}

pase_status pase_set_profiling(pase_ctx* ctx, int32_t enable) {
    if (!ctx) return PASE_ERR_INVALID;
    ctx->profiling = enable;
    return PASE_OK;
}

pase_status pase_get_unique_id(void* uid_out) {
    (void)uid_out;
    return PASE_ERR_STATE;   // multi-GPU not built in this configuration
}

}  // extern "C"
