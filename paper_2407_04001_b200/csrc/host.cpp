// host.cpp -- host core of the hot path (rows a1-a4 of SURVEY §8):
//   a1 ingest + validation, a2 C(v) enumeration,
//   a3 SortNodes with incremental dependent sets (Fig. 4),
//   a4 elimination tree (children(i) = {j : min-rank D(j) = i}) and layouts.
// Written independently of oracle/ (bitset d-sets, tree rule instead of dfs).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <map>
#include <cmath>
#include <cstdio>
#include <numeric>

#include "pase_internal.h"

namespace pase {
namespace {

std::string fmt(const char* f, long long a = 0, long long b = 0, long long c = 0) {
    char buf[256];
    std::snprintf(buf, sizeof buf, f, a, b, c);
    return buf;
}

// ---------------------------------------------------------------- a1
pase_status validate(const pase_graph* g, std::string& err) {
    if (!g || g->n_nodes < 1 || !g->nodes) { err = "graph has no nodes"; return PASE_ERR_INVALID; }
    if (g->n_edges < 0 || (g->n_edges > 0 && !g->edges)) { err = "bad edge array"; return PASE_ERR_INVALID; }
    const int n = g->n_nodes;
    for (int v = 0; v < n; ++v) {
        const pase_node& x = g->nodes[v];
        if (x.n_dims < 1 || x.n_dims > kMaxDims) { err = fmt("node %lld: n_dims %lld out of range", v, x.n_dims); return PASE_ERR_INVALID; }
        for (int k = 0; k < x.n_dims; ++k)
            if (x.size[k] < 1 || x.size[k] > 0x7fffffff) {
                err = fmt("node %lld: dim %lld size out of range [1, 2^31)", v, k);
                return PASE_ERR_INVALID;
            }
        if (x.n_out_axes < 1 || x.n_out_axes > x.n_dims) { err = fmt("node %lld: bad n_out_axes", v); return PASE_ERR_INVALID; }
        if (x.n_w_axes < 0 || x.n_w_axes > x.n_dims) { err = fmt("node %lld: bad n_w_axes", v); return PASE_ERR_INVALID; }
        uint32_t seen = 0;
        for (int a = 0; a < x.n_out_axes; ++a) {
            int d = x.out_axes[a];
            if (d < 0 || d >= x.n_dims || (seen >> d & 1u)) { err = fmt("node %lld: bad out axis %lld", v, a); return PASE_ERR_INVALID; }
            seen |= 1u << d;
        }
        seen = 0;
        for (int a = 0; a < x.n_w_axes; ++a) {
            int d = x.w_axes[a];
            if (d < 0 || d >= x.n_dims || (seen >> d & 1u)) { err = fmt("node %lld: bad weight axis %lld", v, a); return PASE_ERR_INVALID; }
            seen |= 1u << d;
        }
        if (x.n_in_axes < 0 || x.n_in_axes > x.n_dims) { err = fmt("node %lld: bad n_in_axes", v); return PASE_ERR_INVALID; }
        seen = 0;
        for (int a = 0; a < x.n_in_axes; ++a) {
            int d = x.in_axes[a];
            if (d < 0 || d >= x.n_dims || (seen >> d & 1u)) { err = fmt("node %lld: bad input axis %lld", v, a); return PASE_ERR_INVALID; }
            seen |= 1u << d;
        }
        if (x.n_halo < 0 || x.n_halo > PASE_MAX_HALO) { err = fmt("node %lld: bad n_halo", v); return PASE_ERR_INVALID; }
        for (int q = 0; q < x.n_halo; ++q) {
            if (x.halo_spatial[q] < 0 || x.halo_spatial[q] >= x.n_dims || x.halo_filter[q] < 0 ||
                x.halo_filter[q] >= x.n_dims) { err = fmt("node %lld: bad halo pair %lld", v, q); return PASE_ERR_INVALID; }
            if (!(seen >> x.halo_spatial[q] & 1u)) {        // reading L: the halo face is the input's
                err = fmt("node %lld: halo pair %lld: spatial dim %lld is not an input-tensor axis", v, q, x.halo_spatial[q]);
                return PASE_ERR_INVALID;
            }
        }
        if (x.elem_bytes < 1 || x.flops_per_point < 0) { err = fmt("node %lld: bad elem_bytes / flops", v); return PASE_ERR_INVALID; }
        if (x.flop_dims_mask >> x.n_dims) { err = fmt("node %lld: flop_dims_mask names missing dims", v); return PASE_ERR_INVALID; }
    }
    for (int e = 0; e < g->n_edges; ++e) {
        const pase_edge& x = g->edges[e];
        if (x.src < 0 || x.src >= n || x.dst < 0 || x.dst >= n) { err = fmt("edge %lld: endpoint out of range", e); return PASE_ERR_INVALID; }
        if (x.src == x.dst) { err = fmt("edge %lld: self-loop on node %lld", e, x.src); return PASE_ERR_INVALID; }
        for (int a = 0; a < g->nodes[x.src].n_out_axes; ++a)
            if (x.axis_map[a] < -1 || x.axis_map[a] >= g->nodes[x.dst].n_dims) {
                err = fmt("edge %lld: axis_map[%lld] out of range", e, a);
                return PASE_ERR_INVALID;
            }
    }
    // weak connectivity (DESIGN reading N): union-find
    std::vector<int> uf(n);
    std::iota(uf.begin(), uf.end(), 0);
    auto find = [&](int x) { while (uf[x] != x) x = uf[x] = uf[uf[x]]; return x; };
    int comps = n;
    for (int e = 0; e < g->n_edges; ++e) {
        int a = find(g->edges[e].src), b = find(g->edges[e].dst);
        if (a != b) { uf[a] = b; --comps; }
    }
    if (comps != 1) { err = fmt("graph is not weakly connected (%lld components)", comps); return PASE_ERR_INVALID; }
    return PASE_OK;
}

// ---------------------------------------------------------------- a2
// Splits of dim k: values c | p with c | size_k (equal parts), ascending.
void splits_of(const pase_node& x, int k, int p, std::vector<int>& out) {
    out.clear();
    if (!(x.splittable_mask >> k & 1u)) { out.push_back(1); return; }
    for (int c = 1; c <= p; ++c)
        if (p % c == 0 && x.size[k] % c == 0) out.push_back(c);
}

// Lexicographic product (dim 0 most significant) filtered by the policy.  Depth-first over
// the ascending split lists, pruned by the running product; no per-tuple allocation.
// EXACT_P: `target` = the largest achievable product <= p; only branches that can still reach
// it exactly are walked (maxrem[k] = product of the largest splits of dims k..).
struct Enum {
    int nd, p;
    int64_t target = 0;                        // 0: LE_P (every product <= p)
    int opt[kMaxDims][64], nopt[kMaxDims];
    int64_t maxrem[kMaxDims + 1];
    int32_t cur[kMaxDims];
    std::vector<int32_t>* rows;
    void rec(int k, int64_t prod) {
        if (k == nd) {
            if (target == 0 || prod == target) rows->insert(rows->end(), cur, cur + kMaxDims);
            return;
        }
        for (int i = 0; i < nopt[k]; ++i) {
            const int c = opt[k][i];
            const int64_t q = prod * c;
            if (q > (target ? target : p)) break;       // ascending: larger splits exceed it too
            if (target && q * maxrem[k + 1] < target) continue;
            cur[k] = c;
            rec(k + 1, q);
        }
        cur[k] = 1;
    }
    int64_t best(int k, int64_t prod) const {          // largest reachable product <= p
        if (k == nd) return prod;
        int64_t b = 0;
        for (int i = 0; i < nopt[k] && prod * opt[k][i] <= p; ++i) {
            if (prod * opt[k][i] * maxrem[k + 1] <= b) continue;
            b = std::max(b, best(k + 1, prod * opt[k][i]));
            if (b == p) break;
        }
        return b;
    }
};

void enumerate(const pase_node& x, int p, int policy, std::vector<int32_t>& rows) {
    Enum E;
    E.nd = x.n_dims;
    E.p = p;
    std::vector<int> tmp;
    for (int k = 0; k < x.n_dims; ++k) {
        splits_of(x, k, p, tmp);
        E.nopt[k] = (int)tmp.size();
        for (int i = 0; i < E.nopt[k]; ++i) E.opt[k][i] = tmp[i];
    }
    E.maxrem[x.n_dims] = 1;
    for (int k = x.n_dims - 1; k >= 0; --k)
        E.maxrem[k] = std::min<int64_t>((int64_t)p, E.maxrem[k + 1] * E.opt[k][E.nopt[k] - 1]);
    for (int k = 0; k < kMaxDims; ++k) E.cur[k] = 1;
    rows.clear();
    E.rows = &rows;
    if (policy == PASE_CFG_EXACT_P) E.target = E.best(0, 1);   // the tuples of that product only
    E.rec(0, 1);
}

// ---------------------------------------------------------------- a3
// SortNodes (Fig. 4) with bitset d-sets.  Reading C: v.d <- (v.d ∪ sigma_i.d) - {sigma_i, v};
// reading D: ties -> smallest node id.
// Breadth-first order: source = smallest node id, neighbours by increasing id.
std::vector<int32_t> bfs_order(int n, const std::vector<pase_edge>& edges) {
    std::vector<std::vector<int32_t>> nb(n);
    for (const pase_edge& e : edges) { nb[e.src].push_back(e.dst); nb[e.dst].push_back(e.src); }
    for (auto& l : nb) { std::sort(l.begin(), l.end()); l.erase(std::unique(l.begin(), l.end()), l.end()); }
    std::vector<int32_t> order;
    std::vector<char> seen(n, 0);
    order.push_back(0);
    seen[0] = 1;
    for (size_t h = 0; h < order.size(); ++h)
        for (int y : nb[order[h]])
            if (!seen[y]) { seen[y] = 1; order.push_back(y); }
    return order;
}

// SortNodes (Fig. 4).  With `fixed` non-empty, the vertex of step i is fixed[i] instead of
// the argmin of line 5: the update of line 8 then yields D(i) for that ordering too
// (Theorem 2's induction, does not use the argmin) -- the BFS baseline.
void sort_nodes(int n, const std::vector<pase_edge>& edges, std::vector<int32_t>& sigma,
                std::vector<std::vector<int32_t>>& dep_nodes, const std::vector<int32_t>& fixed = {}) {
    const int W = (n + 63) / 64;
    std::vector<uint64_t> d((size_t)n * W, 0);
    auto bit = [&](int v, int x) -> uint64_t& { return d[(size_t)v * W + x / 64]; };
    for (const pase_edge& e : edges) {                    // line 1: v.d <- N(v)
        bit(e.src, e.dst) |= 1ull << (e.dst % 64);
        bit(e.dst, e.src) |= 1ull << (e.src % 64);
    }
    std::vector<int> card(n, 0);
    auto recount = [&](int v) {
        int c = 0;
        for (int w = 0; w < W; ++w) c += __builtin_popcountll(d[(size_t)v * W + w]);
        card[v] = c;
    };
    for (int v = 0; v < n; ++v) recount(v);
    std::vector<char> unseq(n, 1);                        // line 2: U <- V
    sigma.assign(n, -1);
    dep_nodes.assign(n, {});
    std::vector<uint64_t> di(W);
    for (int i = 0; i < n; ++i) {                         // line 4
        int u = -1;
        if (!fixed.empty()) u = fixed[i];
        else
            for (int v = 0; v < n; ++v)                   // line 5: argmin |u.d|, smallest id first
                if (unseq[v] && (u < 0 || card[v] < card[u])) u = v;
        sigma[i] = u;
        unseq[u] = 0;                                     // line 6
        std::copy(d.begin() + (size_t)u * W, d.begin() + (size_t)(u + 1) * W, di.begin());
        for (int w = 0; w < W; ++w)
            for (uint64_t b = di[w]; b; b &= b - 1) {
                int v = w * 64 + __builtin_ctzll(b);      // line 7: v in sigma_i.d
                dep_nodes[i].push_back(v);
                uint64_t* dv = &d[(size_t)v * W];
                for (int q = 0; q < W; ++q) dv[q] |= di[q];   // line 8
                dv[u / 64] &= ~(1ull << (u % 64));
                dv[v / 64] &= ~(1ull << (v % 64));
                recount(v);
            }
    }
}

}  // namespace

pase_status build_plan(const pase_graph* g, int32_t p, const pase_machine* mach, Plan& P,
                       std::string& err) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    if (p < 1 || p > 4096) { err = fmt("p = %lld out of range [1, 4096]", p); return PASE_ERR_INVALID; }
    if (!mach) { err = "machine is NULL"; return PASE_ERR_INVALID; }
    if (mach->cfg_policy != PASE_CFG_EXACT_P && mach->cfg_policy != PASE_CFG_LE_P) { err = "bad cfg_policy"; return PASE_ERR_INVALID; }
    if (mach->ordering != PASE_ORDER_SORTNODES && mach->ordering != PASE_ORDER_BFS) { err = "bad ordering"; return PASE_ERR_INVALID; }
    if (!(mach->flops_per_device > 0) || !(mach->link_bandwidth > 0)) { err = "F and B must be > 0"; return PASE_ERR_INVALID; }
    pase_status st = validate(g, err);
    if (st) return st;
    P.n = g->n_nodes;
    P.m = g->n_edges;
    P.p = p;
    P.policy = mach->cfg_policy;
    P.r = mach->flops_per_device / mach->link_bandwidth;    // r = F/B, once, fp64
    if (!std::isfinite(P.r) || !std::isfinite(mach->flops_per_device)) {
        err = "F must be finite and r = F/B finite (B may be +inf: r = 0)";
        return PASE_ERR_INVALID;
    }
    P.nodes.assign(g->nodes, g->nodes + P.n);
    P.edges.assign(g->edges, g->edges + P.m);
    for (pase_edge& e : P.edges)                            // canonicalise unused map slots
        for (int a = P.nodes[e.src].n_out_axes; a < kMaxDims; ++a) e.axis_map[a] = -1;
    const int n = P.n, m = P.m;

    const auto ta = clk::now();
    // a2
    P.K.assign(n, 0);
    P.cfg_off.assign(n + 1, 0);
    P.cfg.clear();
    std::vector<int32_t> rows;
    // C(v) depends only on (n_dims, size[], splittable_mask, p, policy): each distinct
    // iteration space is enumerated once and stored once (the zoo's layers repeat per block /
    // time step); nodes of the same space share its rows (cfg_off = start of the shared block)
    std::map<std::vector<int64_t>, std::pair<int64_t, int32_t>> memo;   // key -> (offset, K)
    std::vector<int64_t> key;
    for (int v = 0; v < n; ++v) {
        const pase_node& x = P.nodes[v];
        key.assign(x.size, x.size + x.n_dims);
        key.push_back(x.splittable_mask);
        auto it = memo.find(key);
        if (it == memo.end()) {
            enumerate(x, p, P.policy, rows);
            const int64_t k = (int64_t)rows.size() / kMaxDims;
            if (k < 1 || k > 65535) { err = fmt("node %lld: %lld configurations (supported 1..65535)", v, k); return PASE_ERR_RESOURCE; }
            it = memo.emplace(key, std::make_pair((int64_t)P.cfg.size() / kMaxDims, (int32_t)k)).first;
            P.cfg.insert(P.cfg.end(), rows.begin(), rows.end());
        }
        P.K[v] = it->second.second;
        P.cfg_off[v] = it->second.first;
    }
    P.cfg_off[n] = (int64_t)P.cfg.size() / kMaxDims;          // rows in the shared pool
    P.max_k = *std::max_element(P.K.begin(), P.K.end());

    const auto tb = clk::now();
    // a3
    std::vector<std::vector<int32_t>> dn;
    if (mach->ordering == PASE_ORDER_BFS) sort_nodes(n, P.edges, P.sigma, dn, bfs_order(n, P.edges));
    else sort_nodes(n, P.edges, P.sigma, dn);
    P.rank.assign(n, 0);
    for (int i = 0; i < n; ++i) P.rank[P.sigma[i]] = i;
    P.dep.assign(n, {});
    P.max_dep = 0;
    for (int i = 0; i < n; ++i) {
        std::vector<int32_t> dd = dn[i];
        std::sort(dd.begin(), dd.end(), [&](int a, int b) { return P.rank[a] < P.rank[b]; });
        for (int u : dd)
            if (P.rank[u] <= i) { err = "internal: dependent set member precedes its vertex"; return PASE_ERR_STATE; }
        P.dep[i] = dd;
        P.max_dep = std::max<int>(P.max_dep, (int)dd.size());
    }
    if (P.max_dep > kMaxDep) {
        err = fmt("M = max |D(i)| = %lld exceeds %lld (K = %lld): DP tables too wide", P.max_dep, kMaxDep, P.max_k);
        return PASE_ERR_RESOURCE;
    }

    const auto tc = clk::now();
    // a4: elimination tree, E>(sigma_i), levels
    P.parent.assign(n, -1);
    P.children.assign(n, {});
    for (int i = 0; i < n; ++i) {
        if (P.dep[i].empty()) {
            if (i != n - 1) { err = "internal: empty dependent set before the root"; return PASE_ERR_STATE; }
            continue;
        }
        P.parent[i] = P.rank[P.dep[i][0]];                  // lowest-rank member (ascending order)
        P.children[P.parent[i]].push_back(i);               // i ascending -> children sorted
    }
    for (int i = 0; i < n; ++i)                             // lemma: D(j) ⊆ D(i) ∪ {sigma_i}
        for (int j : P.children[i])
            for (int u : P.dep[j])
                if (u != P.sigma[i] && std::find(P.dep[i].begin(), P.dep[i].end(), u) == P.dep[i].end()) {
                    err = "internal: elimination-tree lemma violated";
                    return PASE_ERR_STATE;
                }
    P.egt.assign(n, {});
    for (int e = 0; e < m; ++e) {
        int a = P.rank[P.edges[e].src], b = P.rank[P.edges[e].dst];
        P.egt[std::min(a, b)].push_back(e);
    }
    for (int i = 0; i < n; ++i) {
        auto& L = P.egt[i];
        std::sort(L.begin(), L.end(), [&](int x, int y) {
            int ox = P.rank[P.edges[x].src] == i ? P.rank[P.edges[x].dst] : P.rank[P.edges[x].src];
            int oy = P.rank[P.edges[y].src] == i ? P.rank[P.edges[y].dst] : P.rank[P.edges[y].src];
            return ox != oy ? ox < oy : x < y;
        });
    }
    P.level.assign(n, 0);
    P.levels = 0;
    for (int i = 0; i < n; ++i) {
        int lv = 0;
        for (int j : P.children[i]) lv = std::max(lv, P.level[j] + 1);
        P.level[i] = lv;
        P.levels = std::max(P.levels, lv + 1);
    }

    const auto td = clk::now();
    // layouts
    P.tsize.assign(n, 1);
    P.toff.assign(n + 1, 0);
    P.candidates = 0;
    for (int i = 0; i < n; ++i) {
        long double sz = 1;
        int64_t s = 1;
        for (int u : P.dep[i]) { sz *= P.K[u]; s *= P.K[u]; if (sz > 4e18L) break; }
        if (sz > (long double)(1ll << 40)) {
            err = fmt("T(%lld) has more than 2^40 entries (M = %lld, K = %lld)", i, P.max_dep, P.max_k);
            return PASE_ERR_RESOURCE;
        }
        P.tsize[i] = s;
        P.toff[i + 1] = P.toff[i] + (s + 15) / 16 * 16;   // 128-B aligned tables (no shared L1 lines)
        P.candidates += (uint64_t)s * (uint64_t)P.K[P.sigma[i]];
    }
    P.entries = 0;
    for (int i = 0; i < n; ++i) P.entries += (uint64_t)P.tsize[i];
    // size guard (Table 1 "OOM"): DP + argmin tables
    const uint64_t budget = mach->table_budget_bytes ? mach->table_budget_bytes : (64ull << 30);
    if ((uint64_t)P.toff[n] * 10ull > budget) {
        char buf[200];
        std::snprintf(buf, sizeof buf, "size guard: DP tables need %.3f GB > budget %.3f GB (M = %d, K = %d)",
                      (double)P.toff[n] * 10.0 / 1e9, (double)budget / 1e9, P.max_dep, P.max_k);
        err = buf;
        return PASE_ERR_RESOURCE;
    }
    P.loff.assign(n + 1, 0);
    for (int v = 0; v < n; ++v) P.loff[v + 1] = P.loff[v] + P.K[v];
    P.woff.assign(m + 1, 0);
    for (int e = 0; e < m; ++e)
        P.woff[e + 1] = P.woff[e] + (int64_t)P.K[P.edges[e].src] * P.K[P.edges[e].dst];
    if (const char* tv = std::getenv("PASE_TIMING"); tv && tv[0] == '1') {
        auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "[pase] plan: ingest %.3f ms, C(v) %.3f ms, SortNodes %.3f ms, tree %.3f ms, layout %.3f ms\n",
                     ms(t0, ta), ms(ta, tb), ms(tb, tc), ms(tc, td), ms(td, clk::now()));
    }
    return PASE_OK;
}

}  // namespace pase
