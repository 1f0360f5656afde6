/*
 * oracle.c -- PLAIN, SLOW, OBVIOUSLY-CORRECT CPU ORACLE for PaSE (arXiv 2407.04001).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Never linked into the product.
 * Build: gcc -O2 -std=c99 -ffp-contract=off -fopenmp -shared -fPIC oracle.c -o liboracle.so
 * (-ffp-contract=off: every fp64 operation below is one IEEE round-to-nearest op.)
 *
 * Pins (tests/test_oracle*.py): brute force (Theorem 1), definitional
 * dependent sets (Theorem 2), the Fig. 3 worked example,
 * hand-computed closed forms (tests/golden/closed_forms.json: GEMM data-parallel and
 * column-split t_l / t_x, the conv halo term over the input-tensor axes, t_x with an
 * axis the consumer does not split, the MLP / AlexNet candidate counts), path-graph
 * Viterbi, tree message passing, r=0 separability, the Appendix-A telescoping identity
 * (P:1206-1214).  Every branch of t_l (compute, reduction AR, gradient AR, halo) and of
 * t_x (mapped, unmapped axis) has a hand-derived value.  What stays a READING, not a
 * paper number: the paper does not publish its t_l / t_x formulas
 * (P:268-270), so these closed forms pin the oracle to our reading of Eq. 1, not to the
 * paper's unpublished code.
 */
#include "oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- node access */
#define NREC(nodes, v) ((nodes) + (int64_t)(v) * OR_NODE_REC)
#define EREC(edges, e) ((edges) + (int64_t)(e) * OR_EDGE_REC)

static int nd_dims(const int64_t* r) { return (int)r[0]; }
static int64_t nd_size(const int64_t* r, int k) { return r[1 + k]; }
static int nd_split(const int64_t* r, int k) { return (int)((r[9] >> k) & 1); }
static int nd_nout(const int64_t* r) { return (int)r[10]; }
static int nd_out(const int64_t* r, int a) { return (int)r[11 + a]; }
static int nd_nw(const int64_t* r) { return (int)r[19]; }
static int nd_w(const int64_t* r, int a) { return (int)r[20 + a]; }
static int64_t nd_flopmask(const int64_t* r) { return r[28]; }
static int64_t nd_fpp(const int64_t* r) { return r[29]; }
static int nd_nhalo(const int64_t* r) { return (int)r[30]; }
static int nd_halo_h(const int64_t* r, int q) { return (int)r[31 + q]; }
static int nd_halo_r(const int64_t* r, int q) { return (int)r[35 + q]; }
static int64_t nd_elem(const int64_t* r) { return r[39]; }
static int nd_nin(const int64_t* r) { return (int)r[40]; }
static int nd_in(const int64_t* r, int a) { return (int)r[41 + a]; }

/* ---------------------------------------------------------------- validation */
int or_validate(int n, const int64_t* nodes, int m, const int64_t* edges)
{
    if (n < 1) return 1;
    for (int v = 0; v < n; ++v) {
        const int64_t* r = NREC(nodes, v);
        int d = nd_dims(r);
        if (d < 1 || d > OR_MAXD) return 1;
        for (int k = 0; k < d; ++k) if (nd_size(r, k) < 1) return 1;
        if (nd_nout(r) < 1 || nd_nout(r) > d) return 1;
        for (int a = 0; a < nd_nout(r); ++a) {
            if (nd_out(r, a) < 0 || nd_out(r, a) >= d) return 1;
            for (int b = 0; b < a; ++b) if (nd_out(r, a) == nd_out(r, b)) return 1;
        }
        if (nd_nw(r) < 0 || nd_nw(r) > d) return 1;
        for (int a = 0; a < nd_nw(r); ++a) {
            if (nd_w(r, a) < 0 || nd_w(r, a) >= d) return 1;
            for (int b = 0; b < a; ++b) if (nd_w(r, a) == nd_w(r, b)) return 1;
        }
        if (nd_nin(r) < 0 || nd_nin(r) > d) return 1;
        for (int a = 0; a < nd_nin(r); ++a) {
            if (nd_in(r, a) < 0 || nd_in(r, a) >= d) return 1;
            for (int b = 0; b < a; ++b) if (nd_in(r, a) == nd_in(r, b)) return 1;
        }
        if (nd_nhalo(r) < 0 || nd_nhalo(r) > 4) return 1;
        for (int q = 0; q < nd_nhalo(r); ++q) {
            if (nd_halo_h(r, q) < 0 || nd_halo_h(r, q) >= d) return 1;
            if (nd_halo_r(r, q) < 0 || nd_halo_r(r, q) >= d) return 1;
            /* the halo runs along an axis of the input tensor (reading L) */
            int found = 0;
            for (int a = 0; a < nd_nin(r); ++a) if (nd_in(r, a) == nd_halo_h(r, q)) found = 1;
            if (!found) return 1;
        }
        if (nd_elem(r) < 1 || nd_fpp(r) < 0) return 1;
    }
    for (int e = 0; e < m; ++e) {
        const int64_t* r = EREC(edges, e);
        int s = (int)r[0], t = (int)r[1];
        if (s < 0 || s >= n || t < 0 || t >= n || s == t) return 1;
        int nout = nd_nout(NREC(nodes, s));
        for (int a = 0; a < nout; ++a) {
            if (r[2 + a] < -1 || r[2 + a] >= nd_dims(NREC(nodes, t))) return 1;
        }
    }
    /* weakly connected: plain repeated relaxation */
    uint8_t* seen = (uint8_t*)calloc((size_t)n, 1);
    seen[0] = 1;
    int changed = 1;
    while (changed) {
        changed = 0;
        for (int e = 0; e < m; ++e) {
            int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
            if (seen[s] != seen[t]) { seen[s] = seen[t] = 1; changed = 1; }
        }
    }
    int ok = 1;
    for (int v = 0; v < n; ++v) if (!seen[v]) ok = 0;
    free(seen);
    return ok ? 0 : 1;
}

/* ---------------------------------------------------------------- C(v) */
/* Allowed split values of dim k: divisors of size_k that also divide p (equal parts,
 * P:192-196), or {1} if the dim is not splittable.  Ascending. */
static int split_options(const int64_t* r, int k, int p, int* opt)
{
    int cnt = 0;
    if (!nd_split(r, k)) { opt[0] = 1; return 1; }
    for (int c = 1; c <= p; ++c)
        if (p % c == 0 && nd_size(r, k) % c == 0) opt[cnt++] = c;
    return cnt;
}

/* Enumerate all tuples in lexicographic order (dim 0 most significant) and keep those
 * whose product satisfies the policy.  Returns the count; writes tuples if out != NULL. */
static int enumerate_node(const int64_t* r, int p, int policy, int32_t* out)
{
    int d = nd_dims(r);
    int opts[OR_MAXD][64], nopt[OR_MAXD];
    for (int k = 0; k < d; ++k) nopt[k] = split_options(r, k, p, opts[k]);
    /* target product: p (EXACT_P) or, if no tuple reaches p, the largest product <= p */
    int64_t target = -1;
    if (policy == 0) {
        int64_t best = 0;
        int idx[OR_MAXD] = {0};
        for (;;) {
            int64_t prod = 1;
            for (int k = 0; k < d; ++k) prod *= opts[k][idx[k]];
            if (prod <= p && prod > best) best = prod;
            int k = d - 1;
            while (k >= 0 && ++idx[k] == nopt[k]) { idx[k] = 0; --k; }
            if (k < 0) break;
        }
        target = best;
    }
    int cnt = 0;
    int idx[OR_MAXD] = {0};
    for (;;) {
        int64_t prod = 1;
        for (int k = 0; k < d; ++k) prod *= opts[k][idx[k]];
        int keep = (policy == 0) ? (prod == target) : (prod <= p);
        if (keep) {
            if (out) {
                for (int k = 0; k < OR_MAXD; ++k) out[(int64_t)cnt * OR_MAXD + k] = (k < d) ? opts[k][idx[k]] : 1;
            }
            ++cnt;
        }
        int k = d - 1;
        while (k >= 0 && ++idx[k] == nopt[k]) { idx[k] = 0; --k; }
        if (k < 0) break;
    }
    return cnt;
}

int or_configs(int n, const int64_t* nodes, int p, int policy, int32_t* counts, int32_t* tuples)
{
    if (p < 1 || p > 4096 || (policy != 0 && policy != 1)) return 1;
    int64_t off = 0;
    for (int v = 0; v < n; ++v) {
        counts[v] = enumerate_node(NREC(nodes, v), p, policy, NULL);
        if (tuples) enumerate_node(NREC(nodes, v), p, policy, tuples + off * OR_MAXD);
        off += counts[v];
    }
    return 0;
}

/* ---------------------------------------------------------------- cost model */
/* Ring all-reduce volume over g participants (reading J): 2(g-1)B/g. */
static double allreduce_bytes(int64_t g, int64_t bytes)
{
    if (g <= 1) return 0.0;
    return (double)(uint64_t)(2 * (g - 1) * bytes) / (double)g;
}

/* t_l(v, C, r) (Eq. 1; reading I):
 *   compute (FLOP) + r * (reduction all-reduce + gradient all-reduce + conv halo) bytes */
static double layer_cost(const int64_t* r, const int32_t* c, double ratio)
{
    int d = nd_dims(r);
    int64_t s[OR_MAXD];
    for (int k = 0; k < d; ++k) s[k] = nd_size(r, k) / c[k];
    int64_t compute = nd_fpp(r);
    for (int k = 0; k < d; ++k)
        if (nd_flopmask(r) == 0 || ((nd_flopmask(r) >> k) & 1)) compute *= s[k];
    int in_out[OR_MAXD] = {0}, in_w[OR_MAXD] = {0};
    int64_t out_elems = 1;
    for (int a = 0; a < nd_nout(r); ++a) { in_out[nd_out(r, a)] = 1; out_elems *= s[nd_out(r, a)]; }
    int64_t w_elems = 1;
    for (int a = 0; a < nd_nw(r); ++a) { in_w[nd_w(r, a)] = 1; w_elems *= s[nd_w(r, a)]; }
    int64_t g_red = 1, g_grad = 1;
    for (int k = 0; k < d; ++k) {
        if (!in_out[k]) g_red *= c[k];
        if (!in_w[k]) g_grad *= c[k];
    }
    int64_t out_bytes = nd_elem(r) * out_elems;
    int64_t w_bytes = (nd_nw(r) > 0) ? nd_elem(r) * w_elems : 0;
    if (nd_nw(r) == 0) g_grad = 1;
    /* conv halo (reading L): a split spatial dim h paired with filter dim f exchanges
     * (size_f - 1) input rows per shard; a row is the face of the INPUT-tensor shard across h,
     * i.e. the product of the input-tensor axes other than h; x2 for fwd + bwd */
    int64_t halo = 0;
    for (int q = 0; q < nd_nhalo(r); ++q) {
        int h = nd_halo_h(r, q), f = nd_halo_r(r, q);
        if (c[h] > 1 && nd_size(r, f) > 1) {
            int64_t face = 1;
            for (int a = 0; a < nd_nin(r); ++a)
                if (nd_in(r, a) != h) face *= s[nd_in(r, a)];
            halo += 2 * nd_elem(r) * (nd_size(r, f) - 1) * face;
        }
    }
    double comm = allreduce_bytes(g_red, out_bytes);
    comm = comm + allreduce_bytes(g_grad, w_bytes);
    comm = comm + (double)(uint64_t)halo;
    return (double)(uint64_t)compute + ratio * comm;
}

/* t_x(u, v) bytes (reading K, aligned nested layouts):
 * per output axis a of u: held = ext/c_u, need = ceil(ext/c_v[map]) (ext if unmapped),
 * overlap = min(need, held);  t_x = 2 * elem_u * (prod need - prod overlap). */
static int64_t transfer_bytes(const int64_t* ru, const int32_t* cu, const int64_t* rv,
                              const int32_t* cv, const int64_t* emap)
{
    (void)rv;
    int64_t need = 1, ov = 1;
    for (int a = 0; a < nd_nout(ru); ++a) {
        int du = nd_out(ru, a);
        int64_t ext = nd_size(ru, du);
        int64_t held = ext / cu[du];
        int64_t nd = (emap[a] < 0) ? ext : (ext + cv[emap[a]] - 1) / cv[emap[a]];
        need *= nd;
        ov *= (nd < held) ? nd : held;
    }
    return 2 * nd_elem(ru) * (need - ov);
}

int or_cost_tables(int n, const int64_t* nodes, int m, const int64_t* edges, int p, int policy,
                   double flops, double bandwidth, double* L, double* W)
{
    if (or_validate(n, nodes, m, edges)) return 1;
    const double ratio = flops / bandwidth; /* r = F/B */
    int32_t* K = (int32_t*)malloc(sizeof(int32_t) * n);
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    or_configs(n, nodes, p, policy, K, NULL);
    off[0] = 0;
    for (int v = 0; v < n; ++v) off[v + 1] = off[v] + K[v];
    int32_t* tup = (int32_t*)malloc(sizeof(int32_t) * OR_MAXD * (size_t)off[n]);
    or_configs(n, nodes, p, policy, K, tup);
    int64_t lo = 0;
    for (int v = 0; v < n; ++v)
        for (int c = 0; c < K[v]; ++c)
            L[lo++] = layer_cost(NREC(nodes, v), tup + (off[v] + c) * OR_MAXD, ratio);
    int64_t wo = 0;
    for (int e = 0; e < m; ++e) {
        int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
        for (int cs = 0; cs < K[s]; ++cs)
            for (int ct = 0; ct < K[t]; ++ct) {
                int64_t b = transfer_bytes(NREC(nodes, s), tup + (off[s] + cs) * OR_MAXD,
                                           NREC(nodes, t), tup + (off[t] + ct) * OR_MAXD,
                                           EREC(edges, e) + 2);
                W[wo++] = ratio * (double)(uint64_t)b;
            }
    }
    free(tup); free(off); free(K);
    return 0;
}

/* ---------------------------------------------------------------- graph helpers */
/* adjacency matrix of N(v) (direction agnostic) */
static uint8_t* neighbours(int n, int m, const int64_t* edges)
{
    uint8_t* A = (uint8_t*)calloc((size_t)n * n, 1);
    for (int e = 0; e < m; ++e) {
        int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
        A[(size_t)s * n + t] = A[(size_t)t * n + s] = 1;
    }
    return A;
}

/* dfs(G, U, v): vertices reachable from v through U (v itself included). */
static void dfs(int n, const uint8_t* A, const uint8_t* U, int v, uint8_t* out)
{
    int* stack = (int*)malloc(sizeof(int) * n);
    int sp = 0;
    memset(out, 0, (size_t)n);
    out[v] = 1;
    stack[sp++] = v;
    while (sp) {
        int x = stack[--sp];
        for (int y = 0; y < n; ++y)
            if (A[(size_t)x * n + y] && U[y] && !out[y]) { out[y] = 1; stack[sp++] = y; }
    }
    free(stack);
}

/* ---------------------------------------------------------------- SortNodes (Fig. 4) */
int or_sortnodes(int n, int m, const int64_t* edges, int32_t* sigma, int32_t* dep_off, int32_t* dep_ids)
{
    uint8_t* d = neighbours(n, m, edges);     /* line 1: v.d <- N(v) */
    uint8_t* U = (uint8_t*)malloc((size_t)n); /* line 2: U <- V     */
    uint8_t* Dmask = (uint8_t*)calloc((size_t)n * n, 1);
    memset(U, 1, (size_t)n);
    for (int i = 0; i < n; ++i) {             /* line 4 */
        int best = -1, bestsz = 0;
        for (int u = 0; u < n; ++u) {         /* line 5: argmin |u.d|, ties -> smallest id (reading D) */
            if (!U[u]) continue;
            int sz = 0;
            for (int x = 0; x < n; ++x) sz += d[(size_t)u * n + x];
            if (best < 0 || sz < bestsz) { best = u; bestsz = sz; }
        }
        sigma[i] = best;
        U[best] = 0;                          /* line 6 */
        memcpy(Dmask + (size_t)i * n, d + (size_t)best * n, (size_t)n);
        for (int v = 0; v < n; ++v) {         /* line 7: for v in sigma_i.d */
            if (!Dmask[(size_t)i * n + v]) continue;
            for (int x = 0; x < n; ++x)       /* line 8: v.d <- v.d ∪ sigma_i.d - {sigma_i} (reading C: - {v}) */
                if (Dmask[(size_t)i * n + x]) d[(size_t)v * n + x] = 1;
            d[(size_t)v * n + best] = 0;
            d[(size_t)v * n + v] = 0;
        }
    }
    /* emit D(i) sorted by ascending rank */
    int* rank = (int*)malloc(sizeof(int) * n);
    for (int i = 0; i < n; ++i) rank[sigma[i]] = i;
    int pos = 0;
    for (int i = 0; i < n; ++i) {
        dep_off[i] = pos;
        for (int j = i + 1; j < n; ++j)
            if (Dmask[(size_t)i * n + sigma[j]]) dep_ids[pos++] = sigma[j];
        /* members of sigma_i.d are unsequenced at pick time, hence all of rank > i */
        for (int x = 0; x < n; ++x)
            if (Dmask[(size_t)i * n + x] && rank[x] <= i) { pos = -1; break; }
        if (pos < 0) break;
    }
    if (pos >= 0) dep_off[n] = pos;
    free(rank); free(Dmask); free(U); free(d);
    return pos < 0 ? 1 : 0;
}

/* ---------------------------------------------------------------- BFS order */
int or_bfs_order(int n, int m, const int64_t* edges, int32_t* sigma)
{
    uint8_t* A = neighbours(n, m, edges);
    uint8_t* seen = (uint8_t*)calloc((size_t)n, 1);
    int head = 0, tail = 0;
    sigma[tail++] = 0;
    seen[0] = 1;
    while (head < tail) {
        int x = sigma[head++];
        for (int y = 0; y < n; ++y)
            if (A[(size_t)x * n + y] && !seen[y]) { seen[y] = 1; sigma[tail++] = y; }
    }
    free(seen); free(A);
    return tail == n ? 0 : 1;
}

/* ---------------------------------------------------------------- §3.2 definitions */
int or_sets(int n, int m, const int64_t* edges, const int32_t* sigma, int i,
            uint8_t* X, uint8_t* D, uint8_t* Dbar, int32_t* comp, int32_t* ncomp)
{
    uint8_t* A = neighbours(n, m, edges);
    uint8_t* le = (uint8_t*)calloc((size_t)n, 1);  /* sigma_<=i */
    uint8_t* lt = (uint8_t*)calloc((size_t)n, 1);  /* sigma_<i  */
    uint8_t* gt = (uint8_t*)calloc((size_t)n, 1);  /* sigma_>i  */
    for (int k = 0; k < n; ++k) {
        if (k <= i) le[sigma[k]] = 1;
        if (k < i) lt[sigma[k]] = 1;
        if (k > i) gt[sigma[k]] = 1;
    }
    dfs(n, A, le, sigma[i], X);                    /* X(i) = dfs(G, sigma_<=i, sigma_i) */
    for (int y = 0; y < n; ++y) {                  /* D(i) = N(X(i)) ∩ sigma_>i */
        D[y] = 0;
        Dbar[y] = 0;
        for (int x = 0; x < n; ++x) {
            if (X[x] && A[(size_t)x * n + y] && gt[y]) D[y] = 1;
            if (le[x] && A[(size_t)x * n + y] && gt[y]) Dbar[y] = 1; /* Dbar(i) = N(sigma_<=i) ∩ sigma_>i */
        }
    }
    /* S(i): union over v in X-{sigma_i} of dfs(G, sigma_<i, v) (Fig. 5 line 7) */
    uint8_t* tmp = (uint8_t*)malloc((size_t)n);
    for (int y = 0; y < n; ++y) comp[y] = -1;
    int nc = 0;
    for (int v = 0; v < n; ++v) {
        if (!X[v] || v == sigma[i] || comp[v] >= 0) continue;
        dfs(n, A, lt, v, tmp);
        for (int y = 0; y < n; ++y) if (tmp[y]) comp[y] = nc;
        ++nc;
    }
    *ncomp = nc;
    free(tmp); free(gt); free(lt); free(le); free(A);
    return 0;
}

/* ---------------------------------------------------------------- DP-Alg (Fig. 5) */
typedef struct {
    int n;
    int32_t* sigma;     /* rank -> node */
    int32_t* rank;      /* node -> rank */
    int32_t* doff;      /* D(i) of rank i: dids[doff[i] .. doff[i+1]) ascending rank */
    int32_t* dids;
    int32_t* soff;      /* S(i) lookups: ranks j (ascending) of the connected subsets */
    int32_t* sj;
    int32_t* eoff;      /* edges incident to sigma_i with later other end, sorted (rank, id) */
    int32_t* eids;
    int64_t* toff;      /* table offsets (entries) per rank */
} plan_t;

static void plan_free(plan_t* P)
{
    free(P->sigma); free(P->rank); free(P->doff); free(P->dids); free(P->soff); free(P->sj);
    free(P->eoff); free(P->eids); free(P->toff);
}

static int cmp_i64(const void* a, const void* b)
{
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : x > y;
}

/* Build sigma, D(i), S(i) (as max-rank j per subset), E>(sigma_i), table offsets. */
static int build_plan(int n, int m, const int64_t* edges, const int32_t* K, int order, plan_t* P)
{
    memset(P, 0, sizeof(*P));
    P->n = n;
    P->sigma = (int32_t*)malloc(sizeof(int32_t) * n);
    P->rank = (int32_t*)malloc(sizeof(int32_t) * n);
    P->doff = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    P->dids = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n * n + 1));
    P->soff = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    P->sj = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n * n + 1));
    P->eoff = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    P->eids = (int32_t*)malloc(sizeof(int32_t) * (m + 1));
    P->toff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    if (order == 0) {
        if (or_sortnodes(n, m, edges, P->sigma, P->doff, P->dids)) return 1;   /* Fig. 5 line 1 */
    } else {
        if (or_bfs_order(n, m, edges, P->sigma)) return 1;
    }
    for (int i = 0; i < n; ++i) P->rank[P->sigma[i]] = i;
    uint8_t* X = (uint8_t*)malloc((size_t)n);
    uint8_t* D = (uint8_t*)malloc((size_t)n);
    uint8_t* Db = (uint8_t*)malloc((size_t)n);
    int32_t* comp = (int32_t*)malloc(sizeof(int32_t) * n);
    int spos = 0, dpos = 0;
    for (int i = 0; i < n; ++i) {
        int nc = 0;
        or_sets(n, m, edges, P->sigma, i, X, D, Db, comp, &nc);   /* lines 6-7 */
        if (order != 0) {          /* BFS ordering: definitional D(i) */
            P->doff[i] = dpos;
            for (int k = i + 1; k < n; ++k) if (D[P->sigma[k]]) P->dids[dpos++] = P->sigma[k];
        }
        /* j = max rank of each connected subset X' (line 13), ascending */
        P->soff[i] = spos;
        for (int c = 0; c < nc; ++c) {
            int j = -1;
            for (int y = 0; y < n; ++y) if (comp[y] == c && P->rank[y] > j) j = P->rank[y];
            P->sj[spos++] = j;
        }
        for (int a = P->soff[i] + 1; a < spos; ++a)       /* insertion sort ascending */
            for (int b = a; b > P->soff[i] && P->sj[b - 1] > P->sj[b]; --b) {
                int t = P->sj[b]; P->sj[b] = P->sj[b - 1]; P->sj[b - 1] = t;
            }
    }
    if (order != 0) P->doff[n] = dpos;
    P->soff[n] = spos;
    /* E>(sigma_i): edges whose other endpoint has higher rank, by (rank(other), edge id) */
    int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    int epos = 0;
    for (int i = 0; i < n; ++i) {
        P->eoff[i] = epos;
        int v = P->sigma[i], cnt = 0;
        for (int e = 0; e < m; ++e) {
            int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
            int other = (s == v) ? t : (t == v) ? s : -1;
            if (other >= 0 && P->rank[other] > i) key[cnt++] = (int64_t)P->rank[other] * (m + 1) + e;
        }
        qsort(key, (size_t)cnt, sizeof(int64_t), cmp_i64);
        for (int c = 0; c < cnt; ++c) P->eids[epos++] = (int32_t)(key[c] % (m + 1));
    }
    P->eoff[n] = epos;
    /* Fig. 5 line 14 needs phi'(u) for every u in sigma_j.d: check D(j) ⊆ D(i) ∪ {sigma_i} */
    for (int i = 0; i < n; ++i)
        for (int a = P->soff[i]; a < P->soff[i + 1]; ++a) {
            int j = P->sj[a];
            for (int b = P->doff[j]; b < P->doff[j + 1]; ++b) {
                int u = P->dids[b], found = (u == P->sigma[i]);
                for (int c = P->doff[i]; c < P->doff[i + 1]; ++c) if (P->dids[c] == u) found = 1;
                if (!found) { free(key); free(comp); free(Db); free(D); free(X); return 1; }
            }
        }
    P->toff[0] = 0;
    for (int i = 0; i < n; ++i) {
        int64_t sz = 1;
        for (int a = P->doff[i]; a < P->doff[i + 1]; ++a) {
            sz *= K[P->dids[a]];
            if (sz > ((int64_t)1 << 50)) { sz = (int64_t)1 << 50; }
        }
        P->toff[i + 1] = P->toff[i] + sz;
    }
    free(key); free(comp); free(Db); free(D); free(X);
    return 0;
}

int or_table_sizes(int n, int m, const int64_t* edges, const int32_t* K, int order,
                   int64_t* tbl_off, int64_t* candidates)
{
    plan_t P;
    if (build_plan(n, m, edges, K, order, &P)) { plan_free(&P); return 1; }
    int64_t cand = 0;
    for (int i = 0; i <= n; ++i) tbl_off[i] = P.toff[i];
    for (int i = 0; i < n; ++i) cand += (P.toff[i + 1] - P.toff[i]) * K[P.sigma[i]];
    *candidates = cand;
    plan_free(&P);
    return 0;
}

/* index of phi|D(j) in T(j): mixed radix over D(j) ascending rank, lowest fastest */
static int64_t table_index(const plan_t* P, int j, const int32_t* K, const int32_t* assign)
{
    int64_t idx = 0, stride = 1;
    for (int a = P->doff[j]; a < P->doff[j + 1]; ++a) {
        int u = P->dids[a];
        idx += (int64_t)assign[u] * stride;
        stride *= K[u];
    }
    return idx;
}

static double w_lookup(const int64_t* edges, const int32_t* K, const double* W, const int64_t* woff,
                       int e, const int32_t* assign)
{
    int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
    return W[woff[e] + (int64_t)assign[s] * K[t] + assign[t]];
}

/* Fig. 5 run to completion; *tbl_p / *cfg_p / *plan_p stay owned by the caller. */
static int dp_run(int n, int m, const int64_t* edges, const int32_t* K, const double* L, const double* W,
                  int order, int threads, int64_t table_limit, int32_t* strategy, double* total,
                  double** tbl_p, int32_t** cfg_p, plan_t* plan_p)
{
    plan_t P;
    if (build_plan(n, m, edges, K, order, &P)) { plan_free(&P); return 1; }
    if (table_limit > 0 && P.toff[n] > table_limit) { plan_free(&P); return 2; }
    int64_t* loff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    loff[0] = 0;
    for (int v = 0; v < n; ++v) loff[v + 1] = loff[v] + K[v];
    woff[0] = 0;
    for (int e = 0; e < m; ++e)
        woff[e + 1] = woff[e] + (int64_t)K[EREC(edges, e)[0]] * K[EREC(edges, e)[1]];
    double* tbl = (double*)malloc(sizeof(double) * (size_t)P.toff[n]);   /* v.tbl (line 2) */
    int32_t* cfg = (int32_t*)malloc(sizeof(int32_t) * (size_t)P.toff[n]); /* v.cfg (line 3) */
    if (!tbl || !cfg) { free(tbl); free(cfg); free(loff); free(woff); plan_free(&P); return 2; }
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    for (int i = 0; i < n; ++i) {                               /* line 4 */
        const int v = P.sigma[i];
        const int64_t nphi = P.toff[i + 1] - P.toff[i];         /* |Phi| (1 if D(i) = ∅, line 8) */
#pragma omp parallel
        {
            int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * n);
#pragma omp for schedule(static)
            for (int64_t phi = 0; phi < nphi; ++phi) {          /* line 8 */
                int64_t rem = phi;                              /* decode phi over D(i) */
                for (int a = P.doff[i]; a < P.doff[i + 1]; ++a) {
                    int u = P.dids[a];
                    assign[u] = (int32_t)(rem % K[u]);
                    rem /= K[u];
                }
                double mincost = INFINITY;                      /* line 9 */
                int32_t best = -1;
                for (int C = 0; C < K[v]; ++C) {                /* line 10 */
                    assign[v] = C;                              /* line 11: phi' */
                    double cost = L[loff[v] + C];               /* line 12: h(i, phi') (Eq. 3) */
                    for (int a = P.eoff[i]; a < P.eoff[i + 1]; ++a)
                        cost = cost + w_lookup(edges, K, W, woff, P.eids[a], assign);
                    for (int a = P.soff[i]; a < P.soff[i + 1]; ++a) {   /* lines 13-16 */
                        int j = P.sj[a];
                        cost = cost + tbl[P.toff[j] + table_index(&P, j, K, assign)];
                    }
                    if (cost < mincost) {                       /* lines 17-19 (strict <) */
                        mincost = cost;
                        best = C;
                    }
                }
                tbl[P.toff[i] + phi] = mincost;
                cfg[P.toff[i] + phi] = best;
            }
            free(assign);
        }
    }
    *total = tbl[P.toff[n - 1]];                                /* line 22: sigma_|V|.tbl(∅) */
    /* back-substitution from sigma_|V|.cfg */
    int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * n);
    for (int i = n - 1; i >= 0; --i) {
        int v = P.sigma[i];
        assign[v] = cfg[P.toff[i] + table_index(&P, i, K, assign)];
    }
    for (int v = 0; v < n; ++v) strategy[v] = assign[v];
    free(assign); free(woff); free(loff);
    *tbl_p = tbl;
    *cfg_p = cfg;
    *plan_p = P;
    return 0;
}

int or_dp(int n, int m, const int64_t* edges, const int32_t* K, const double* L, const double* W,
          int order, int threads, int64_t table_limit, int32_t* strategy, double* total,
          double* tbl_out, int32_t* arg_out)
{
    double* tbl;
    int32_t* cfg;
    plan_t P;
    int rc = dp_run(n, m, edges, K, L, W, order, threads, table_limit, strategy, total, &tbl, &cfg, &P);
    if (rc) return rc;
    if (tbl_out) memcpy(tbl_out, tbl, sizeof(double) * (size_t)P.toff[n]);
    if (arg_out) memcpy(arg_out, cfg, sizeof(int32_t) * (size_t)P.toff[n]);
    free(cfg); free(tbl);
    plan_free(&P);
    return 0;
}

int or_dp_select(int n, int m, const int64_t* edges, const int32_t* K, const double* L, const double* W,
                 int order, int threads, int32_t* strategy, double* total,
                 int nsel, const int32_t* sel, double* tbl_out, int32_t* arg_out)
{
    double* tbl;
    int32_t* cfg;
    plan_t P;
    int rc = dp_run(n, m, edges, K, L, W, order, threads, 0, strategy, total, &tbl, &cfg, &P);
    if (rc) return rc;
    int64_t o = 0;
    for (int k = 0; k < nsel; ++k) {
        const int i = sel[k];
        const int64_t sz = P.toff[i + 1] - P.toff[i];
        memcpy(tbl_out + o, tbl + P.toff[i], sizeof(double) * (size_t)sz);
        memcpy(arg_out + o, cfg + P.toff[i], sizeof(int32_t) * (size_t)sz);
        o += sz;
    }
    free(cfg); free(tbl);
    plan_free(&P);
    return 0;
}

/* ---------------------------------------------------------------- Eq. 2 (BFS recurrence) */
int or_dp_bfs_eq2(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
                  const double* W, int64_t table_limit, int32_t* strategy, double* total)
{
    int32_t* sigma = (int32_t*)malloc(sizeof(int32_t) * n);
    if (or_bfs_order(n, m, edges, sigma)) { free(sigma); return 1; }
    int32_t* rank = (int32_t*)malloc(sizeof(int32_t) * n);
    for (int i = 0; i < n; ++i) rank[sigma[i]] = i;
    uint8_t* A = neighbours(n, m, edges);
    /* Dbar(i) = N(sigma_<=i) ∩ sigma_>i, ascending rank */
    int32_t* doff = (int32_t*)malloc(sizeof(int32_t) * (n + 1));
    int32_t* dids = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n * n + 1));
    int64_t* toff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    int pos = 0;
    toff[0] = 0;
    for (int i = 0; i < n; ++i) {
        doff[i] = pos;
        int64_t sz = 1;
        for (int k = i + 1; k < n; ++k) {
            int y = sigma[k], adj = 0;
            for (int q = 0; q <= i; ++q) if (A[(size_t)sigma[q] * n + y]) adj = 1;
            if (adj) { dids[pos++] = y; sz *= K[y]; if (sz > ((int64_t)1 << 50)) sz = (int64_t)1 << 50; }
        }
        toff[i + 1] = toff[i] + sz;
    }
    doff[n] = pos;
    int rc = 0;
    if (table_limit > 0 && toff[n] > table_limit) rc = 2;
    double* tbl = NULL;
    int32_t* cfg = NULL;
    if (!rc) {
        tbl = (double*)malloc(sizeof(double) * (size_t)toff[n]);
        cfg = (int32_t*)malloc(sizeof(int32_t) * (size_t)toff[n]);
        if (!tbl || !cfg) rc = 2;
    }
    int64_t* loff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    loff[0] = 0;
    for (int v = 0; v < n; ++v) loff[v + 1] = loff[v] + K[v];
    woff[0] = 0;
    for (int e = 0; e < m; ++e) woff[e + 1] = woff[e] + (int64_t)K[EREC(edges, e)[0]] * K[EREC(edges, e)[1]];
    int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * n);
    for (int i = 0; i < n && !rc; ++i) {
        int v = sigma[i];
        for (int64_t phi = 0; phi < toff[i + 1] - toff[i]; ++phi) {
            int64_t rem = phi;
            for (int a = doff[i]; a < doff[i + 1]; ++a) { assign[dids[a]] = (int32_t)(rem % K[dids[a]]); rem /= K[dids[a]]; }
            double mincost = INFINITY;
            int32_t best = -1;
            for (int C = 0; C < K[v]; ++C) {
                assign[v] = C;
                double cost = L[loff[v] + C];                                /* h(i, phi') */
                for (int k = i + 1; k < n; ++k)                              /* later neighbours by (rank, id) */
                    for (int e = 0; e < m; ++e) {
                        int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
                        if ((s == v && t == sigma[k]) || (t == v && s == sigma[k]))
                            cost = cost + W[woff[e] + (int64_t)assign[s] * K[t] + assign[t]];
                    }
                if (i > 0) {                                                 /* + fbar(i-1, phi'') */
                    int64_t idx = 0, stride = 1;
                    for (int a = doff[i - 1]; a < doff[i]; ++a) { idx += (int64_t)assign[dids[a]] * stride; stride *= K[dids[a]]; }
                    cost = cost + tbl[toff[i - 1] + idx];
                }
                if (cost < mincost) { mincost = cost; best = C; }
            }
            tbl[toff[i] + phi] = mincost;
            cfg[toff[i] + phi] = best;
        }
    }
    if (!rc) {
        *total = tbl[toff[n - 1]];
        for (int i = n - 1; i >= 0; --i) {
            int64_t idx = 0, stride = 1;
            for (int a = doff[i]; a < doff[i + 1]; ++a) { idx += (int64_t)assign[dids[a]] * stride; stride *= K[dids[a]]; }
            assign[sigma[i]] = cfg[toff[i] + idx];
        }
        for (int v = 0; v < n; ++v) strategy[v] = assign[v];
    }
    (void)rank;
    free(assign); free(woff); free(loff); free(cfg); free(tbl); free(toff); free(dids); free(doff);
    free(A); free(rank); free(sigma);
    return rc;
}

/* ---------------------------------------------------------------- Eq. 1 / brute force */
double or_eval(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
               const double* W, const int32_t* strategy)
{
    double acc = 0.0;
    int64_t off = 0;
    for (int v = 0; v < n; ++v) { acc = acc + L[off + strategy[v]]; off += K[v]; }
    off = 0;
    for (int e = 0; e < m; ++e) {
        int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
        acc = acc + W[off + (int64_t)strategy[s] * K[t] + strategy[t]];
        off += (int64_t)K[s] * K[t];
    }
    return acc;
}

int or_brute(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
             const double* W, int64_t limit, int32_t* strategy, double* total)
{
    double space = 1.0;
    for (int v = 0; v < n; ++v) space *= K[v];
    if (limit > 0 && space > (double)limit) return 2;
    int32_t* phi = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    double best = INFINITY;
    for (;;) {
        double c = or_eval(n, m, edges, K, L, W, phi);
        if (c < best) { best = c; memcpy(strategy, phi, sizeof(int32_t) * n); }
        int v = 0;                                   /* node 0 fastest */
        while (v < n && ++phi[v] == K[v]) { phi[v] = 0; ++v; }
        if (v == n) break;
    }
    *total = best;
    free(phi);
    return 0;
}

double or_sum_h(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
                const double* W, const int32_t* sigma, const int32_t* strategy)
{
    int32_t* rank = (int32_t*)malloc(sizeof(int32_t) * n);
    for (int i = 0; i < n; ++i) rank[sigma[i]] = i;
    int64_t* loff = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
    int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (m + 1));
    loff[0] = 0;
    for (int v = 0; v < n; ++v) loff[v + 1] = loff[v] + K[v];
    woff[0] = 0;
    for (int e = 0; e < m; ++e) woff[e + 1] = woff[e] + (int64_t)K[EREC(edges, e)[0]] * K[EREC(edges, e)[1]];
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {                     /* sum_i h(i, phi) */
        int v = sigma[i];
        double h = L[loff[v] + strategy[v]];          /* t_l(sigma_i) */
        for (int e = 0; e < m; ++e) {                 /* + r t_x to later neighbours (Eq. 3) */
            int s = (int)EREC(edges, e)[0], t = (int)EREC(edges, e)[1];
            int other = (s == v) ? t : (t == v) ? s : -1;
            if (other >= 0 && rank[other] > i)
                h = h + W[woff[e] + (int64_t)strategy[s] * K[t] + strategy[t]];
        }
        acc = acc + h;
    }
    free(woff); free(loff); free(rank);
    return acc;
}

/* ---------------------------------------------------------------- f3: device assignment */
/* Greedy device assignment ("a simple greedy assignment that maximizes data
 * locality, i.e. maximizes |A(v,d,phi) ∩ A(u,d,phi)|"), DESIGN reading U:
 *   shard s of v under config c = digits of s in the radix c, dim 0 most significant;
 *   vertices in node-id order, shards in index order; each shard takes the free device with
 *   the largest sum, over the edges to already-assigned neighbours, of the overlap (elements)
 *   between what the consumer shard on that device needs of the producer's output tensor and
 *   what the producer shard on that device holds; ties -> lowest device id.
 * Realized t_x of an edge = 2 elem max over devices d holding a consumer shard of
 * (|needed on d| - |needed on d ∩ held on d|), bytes. */
static void digits_of(const int32_t* c, int d, int s, int* out)
{
    for (int k = d - 1; k >= 0; --k) { out[k] = s % c[k]; s /= c[k]; }
}

/* producer u (config cu, shard digits iu): held interval of output axis a */
static void held_interval(const int64_t* ru, const int32_t* cu, const int* iu, int a,
                          int64_t* lo, int64_t* hi)
{
    int k = nd_out(ru, a);
    int64_t h = nd_size(ru, k) / cu[k];
    *lo = (int64_t)iu[k] * h;
    *hi = *lo + h;
}

/* consumer v (config cv, shard digits jv) of edge e: needed interval of u's output axis a */
static void need_interval(const int64_t* ru, const int64_t* erec, const int32_t* cv, const int* jv,
                          int a, int64_t* lo, int64_t* hi)
{
    int64_t ext = nd_size(ru, nd_out(ru, a));
    int64_t mp = erec[2 + a];
    if (mp < 0) { *lo = 0; *hi = ext; return; }
    int64_t nd = (ext + cv[mp] - 1) / cv[mp];
    *lo = (int64_t)jv[mp] * nd;
    *hi = *lo + nd < ext ? *lo + nd : ext;
    if (*lo > *hi) *lo = *hi;               /* shard past the tensor's end: needs nothing */
}

/* |needed by consumer shard jv| and |needed ∩ held by producer shard iu| (elements) */
static void edge_overlap(const int64_t* ru, const int32_t* cu, const int* iu, const int64_t* erec,
                         const int32_t* cv, const int* jv, int64_t* need, int64_t* ov)
{
    *need = 1;
    *ov = 1;
    for (int a = 0; a < nd_nout(ru); ++a) {
        int64_t nl, nh, hl, hh;
        need_interval(ru, erec, cv, jv, a, &nl, &nh);
        *need *= nh - nl;
        if (!iu) continue;
        held_interval(ru, cu, iu, a, &hl, &hh);
        int64_t lo = nl > hl ? nl : hl, hi = nh < hh ? nh : hh;
        *ov *= hi > lo ? hi - lo : 0;
    }
    if (!iu) *ov = 0;
}

int or_assign(int n, const int64_t* nodes, int m, const int64_t* edges, int p, const int32_t* cfg,
              int32_t* dev, double* tx)
{
    if (or_validate(n, nodes, m, edges)) return 1;
    int32_t* inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)n * p);   /* shard of v on device d */
    uint8_t* assigned = (uint8_t*)calloc((size_t)n, 1);
    for (int64_t k = 0; k < (int64_t)n * p; ++k) { inv[k] = -1; dev[k] = -1; }
    int iu[OR_MAXD], jv[OR_MAXD];
    for (int v = 0; v < n; ++v) {
        const int64_t* rv = NREC(nodes, v);
        const int32_t* cv = cfg + (size_t)v * OR_MAXD;
        int shards = 1;
        for (int k = 0; k < nd_dims(rv); ++k) shards *= cv[k];
        if (shards > p) { free(inv); free(assigned); return 1; }
        for (int s = 0; s < shards; ++s) {
            int64_t best = -1;
            int bestd = -1;
            for (int d = 0; d < p; ++d) {
                if (inv[(size_t)v * p + d] >= 0) continue;           /* device taken */
                int64_t score = 0;
                for (int e = 0; e < m; ++e) {
                    const int64_t* er = EREC(edges, e);
                    int a = (int)er[0], b = (int)er[1];
                    int64_t need, ov;
                    if (a == v && assigned[b]) {                     /* v produces for b */
                        int t = inv[(size_t)b * p + d];
                        if (t < 0) continue;
                        digits_of(cv, nd_dims(rv), s, iu);
                        digits_of(cfg + (size_t)b * OR_MAXD, nd_dims(NREC(nodes, b)), t, jv);
                        edge_overlap(rv, cv, iu, er, cfg + (size_t)b * OR_MAXD, jv, &need, &ov);
                        score += ov;
                    } else if (b == v && assigned[a]) {              /* v consumes from a */
                        int t = inv[(size_t)a * p + d];
                        if (t < 0) continue;
                        digits_of(cfg + (size_t)a * OR_MAXD, nd_dims(NREC(nodes, a)), t, iu);
                        digits_of(cv, nd_dims(rv), s, jv);
                        edge_overlap(NREC(nodes, a), cfg + (size_t)a * OR_MAXD, iu, er, cv, jv, &need, &ov);
                        score += ov;
                    }
                }
                if (score > best) { best = score; bestd = d; }
            }
            dev[(size_t)v * p + s] = bestd;
            inv[(size_t)v * p + bestd] = s;
        }
        assigned[v] = 1;
    }
    for (int e = 0; e < m; ++e) {
        const int64_t* er = EREC(edges, e);
        int a = (int)er[0], b = (int)er[1];
        const int64_t* ra = NREC(nodes, a);
        int64_t worst = 0;
        for (int d = 0; d < p; ++d) {
            int t = inv[(size_t)b * p + d];
            if (t < 0) continue;                                     /* d needs nothing */
            int u = inv[(size_t)a * p + d];
            digits_of(cfg + (size_t)b * OR_MAXD, nd_dims(NREC(nodes, b)), t, jv);
            if (u >= 0) digits_of(cfg + (size_t)a * OR_MAXD, nd_dims(ra), u, iu);
            int64_t need, ov;
            edge_overlap(ra, cfg + (size_t)a * OR_MAXD, u >= 0 ? iu : NULL, er, cfg + (size_t)b * OR_MAXD, jv,
                         &need, &ov);
            if (need - ov > worst) worst = need - ov;
        }
        tx[e] = (double)(uint64_t)(2 * nd_elem(ra) * worst);
    }
    free(inv); free(assigned);
    return 0;
}
