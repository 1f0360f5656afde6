/*
 * oracle.h -- PLAIN, SLOW, OBVIOUSLY-CORRECT CPU ORACLE for PaSE (arXiv 2407.04001).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product path
 * (paper_2407_04001_b200/, include/pase.h) never includes, links or calls this.
 * It shares no code, header, table or constant with the CUDA path.
 *
 * Each function cites the PAPER.md passage it follows ("P:<line>").
 * Readings of ambiguous passages are the DESIGN.md §2 readings (A..T).
 *
 * Graph encoding (flat int64 records, filled by oracle/oracle.py):
 *   node record, OR_NODE_REC int64 fields:
 *     [0] n_dims  [1..8] size[k]  [9] splittable bitmask
 *     [10] n_out  [11..18] out_axes  [19] n_w  [20..27] w_axes
 *     [28] flop_dims bitmask (0 = all dims)  [29] flops_per_point
 *     [30] n_halo [31..34] halo spatial dims [35..38] halo filter dims
 *     [39] elem_bytes  [40] n_in  [41..48] in_axes (iteration dims of the input-tensor axes;
 *     the conv halo face runs over them, DESIGN reading L)
 *   edge record, OR_EDGE_REC int64 fields: [0] src [1] dst [2..9] axis_map (-1 = none)
 *
 * Cost tables (memoised t_l / t_x, SURVEY §8.c.1 "Implementation notes"):
 *   L: per node v (node-id order) K_v doubles;  L_v[C] = t_l(v, C, r)
 *   W: per edge e (edge-id order) K_src*K_dst doubles, W_e[c_src*K_dst + c_dst] = r*t_x
 */
#ifndef PASE_ORACLE_H
#define PASE_ORACLE_H
#include <stdint.h>

#define OR_MAXD 8
#define OR_NODE_REC 49
#define OR_EDGE_REC 10

#ifdef __cplusplus
extern "C" {
#endif

/* 0 ok, 1 invalid input, 2 resource (size guard) */
int or_validate(int n, const int64_t* nodes, int m, const int64_t* edges);

/* C(v) (DESIGN reading B/G).  policy 0 = EXACT_P, 1 = LE_P.
 * counts[n]; if tuples != NULL it receives, per node in order, counts[v]*OR_MAXD int32. */
int or_configs(int n, const int64_t* nodes, int p, int policy, int32_t* counts, int32_t* tuples);

/* t_l (Eq. 1; reading I/J/L) and r*t_x (reading K/R). */
int or_cost_tables(int n, const int64_t* nodes, int m, const int64_t* edges, int p, int policy,
                   double flops, double bandwidth, double* L, double* W);

/* SortNodes (Fig. 4; readings C, D).  sigma[n]; dep_off[n+1]; dep_ids (<= n*n)
 * lists sigma_i.d at pick time, sorted by ascending rank. */
int or_sortnodes(int n, int m, const int64_t* edges, int32_t* sigma, int32_t* dep_off, int32_t* dep_ids);

/* Breadth-first ordering, source = smallest node id, neighbours by id. */
int or_bfs_order(int n, int m, const int64_t* edges, int32_t* sigma);

/* Definitions of §3.2 for an arbitrary ordering sigma:
 * X(i) = dfs(G, sigma_<=i, sigma_i); D(i) = N(X(i)) ∩ sigma_>i; S(i) components of X(i)-{sigma_i};
 * Dbar(i) = N(sigma_<=i) ∩ sigma_>i.  i is 0-based rank.
 * Outputs are node-id membership masks (uint8[n]); comp[n] gets the component index
 * (0..ncomp-1, -1 if not in X(i)-{sigma_i}) and *ncomp. */
int or_sets(int n, int m, const int64_t* edges, const int32_t* sigma, int i,
            uint8_t* X, uint8_t* D, uint8_t* Dbar, int32_t* comp, int32_t* ncomp);

/* DP-Alg (Fig. 5) over recurrence Eq. 4 with h of Eq. 3.
 * K[n] config counts, L/W as above.  order: 0 = SortNodes (the paper's DP-Alg),
 * 1 = BFS ordering with the same Eq. 4 (then D(i) = Dbar(i) reduced by X).
 * Outputs: strategy[n] (config index per node), *total = f(|V|, ∅).
 * If tbl_out != NULL: per rank i (sigma order) the table T(i) and argmin A(i) are
 * written at tbl_off[i] (caller sizes them with or_table_sizes) in the canonical layout:
 * coordinates D(i) in ascending rank, lowest rank fastest (mixed radix).
 * threads > 1 splits the phi loop (entries are independent). table_limit guards (P:753 OOM). */
int or_table_sizes(int n, int m, const int64_t* edges, const int32_t* K, int order,
                   int64_t* tbl_off /* n+1 */, int64_t* candidates);
int or_dp(int n, int m, const int64_t* edges, const int32_t* K, const double* L, const double* W,
          int order, int threads, int64_t table_limit, int32_t* strategy, double* total,
          double* tbl_out, int32_t* arg_out);

/* or_dp, copying out only the tables of the nsel ranks sel[] (concatenated in that order) --
 * full-size parity checks of configs whose complete tables do not fit twice in host memory. */
int or_dp_select(int n, int m, const int64_t* edges, const int32_t* K, const double* L, const double* W,
                 int order, int threads, int32_t* strategy, double* total,
                 int nsel, const int32_t* sel, double* tbl_out, int32_t* arg_out);

/* Eq. 2 recurrence with the BFS ordering and single predecessor table. */
int or_dp_bfs_eq2(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
                  const double* W, int64_t table_limit, int32_t* strategy, double* total);

/* Brute force: all prod K_v strategies, node 0 fastest, strict '<' keeps first. */
int or_brute(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
             const double* W, int64_t limit, int32_t* strategy, double* total);

/* Eq. 1: sum_v L_v[phi(v)] (node-id order) + sum_e W_e (edge-id order). */
double or_eval(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
               const double* W, const int32_t* strategy);

/* h(i, phi) of Eq. 3 for a total strategy, summed over ranks (App. A). */
double or_sum_h(int n, int m, const int64_t* edges, const int32_t* K, const double* L,
                const double* W, const int32_t* sigma, const int32_t* strategy);

/* f3: greedy device assignment (DESIGN reading U).  cfg = the chosen config tuple
 * of every node (n * OR_MAXD int32).  dev[n * p]: device of shard s of v at dev[v*p + s]
 * (-1 for s >= prod c(v)); tx[m]: realized t_x bytes of each edge under the assignment. */
int or_assign(int n, const int64_t* nodes, int m, const int64_t* edges, int p, const int32_t* cfg,
              int32_t* dev, double* tx);

#ifdef __cplusplus
}
#endif
#endif
