"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each test names the passage it pins.  None of these compares the oracle with itself:
brute force, closed forms, independent textbook recursions (Viterbi, tree message
passing), definitional sets and the paper's worked example.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_04001_b200 import zoo
from tests.helpers import degrees, random_costs, relabel

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel_eq(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


# --------------------------------------------------------------------------- C(v)
def test_config_counts_closed_form():
    """P:204-205 with reading B: power-of-two splits, prod = p -> C(k+d-1, d-1); prod <= p -> C(k+d, d)."""
    for p, k in ((4, 2), (8, 3), (64, 6)):
        for d in range(1, 6):
            g = zoo.GraphBuilder()
            g.node("x", "t", [(f"d{i}", 1 << 12) for i in range(d)], out=["d0"])
            gr = g.graph()
            assert len(O.configs(gr, p, O.EXACT_P)[0]) == math.comb(k + d - 1, d - 1)
            assert len(O.configs(gr, p, O.LE_P)[0]) == math.comb(k + d, d)


def test_config_examples():
    g = zoo.GraphBuilder()
    g.node("x", "t", [("a", 64), ("b", 64)], out=["a"])
    gr = g.graph()
    # SPEC's d=2, p=4 example -> EXACT_P (1,4),(2,2),(4,1); LE_P adds (1,1),(1,2),(2,1)
    assert [tuple(c) for c in O.configs(gr, 4, O.EXACT_P)[0]] == [(1, 4), (2, 2), (4, 1)]
    assert [tuple(c) for c in O.configs(gr, 4, O.LE_P)[0]] == [(1, 1), (1, 2), (1, 4), (2, 1), (2, 2), (4, 1)]
    # p = 1: only the all-ones tuple
    assert [tuple(c) for c in O.configs(gr, 1, O.EXACT_P)[0]] == [(1, 1)]
    # Fig. 1: GEMM configuration (1,4,2) is in C(v) for p = 8
    gm = zoo.gemm_single()
    assert (1, 4, 2) in [tuple(c) for c in O.configs(gm, 8, O.EXACT_P)[0]]
    # odd / unsplittable dims stay 1; no exact-p tuple -> maximal achievable product
    g = zoo.GraphBuilder()
    g.node("x", "t", [("a", 6), ("b", 3)], out=["a"])
    assert [tuple(c) for c in O.configs(g.graph(), 8, O.EXACT_P)[0]] == [(2, 1)]


# --------------------------------------------------------------------------- cost model closed forms
def test_cost_closed_forms_mlp():
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    g = zoo.mlp()
    cfgs = [tuple(c) for c in O.configs(g, 4)[0]]
    K, Ls, Ws = O.cost_tables(g, 4)
    L = Ls[0]
    assert L[cfgs.index((4, 1, 1))] == gold["data_parallel_411"]["t_l"]
    assert L[cfgs.index((1, 4, 1))] == gold["column_split_141"]["t_l"]
    assert L[cfgs.index((1, 2, 2))] == gold["split_122"]["t_l"]
    i141 = cfgs.index((1, 4, 1))
    assert Ws[0][i141, i141] == gold["column_split_141"]["W"]
    i122 = cfgs.index((1, 2, 2))
    assert Ws[0][i122, i122] == 0.0
    i411 = cfgs.index((4, 1, 1))
    assert Ws[0][i411, i411] == 0.0          # aligned batch split: no transfer
    P = O.Problem(g, K, Ls, Ws)
    assert P.eval([i411] * 4) == gold["pure_data_parallel_total"]
    # the optimum is at most the pure data-parallel cost
    assert P.dp()["cost"] <= gold["pure_data_parallel_total"]


def test_cost_gemm_all_ones_and_p1():
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    g = zoo.gemm_single()
    K, Ls, _ = O.cost_tables(g, 1)
    assert list(K) == [1] and Ls[0][0] == gold["gemm_all_ones_1024"]["t_l"]
    # p = 1 on a whole network: all-ones strategy, W == 0, cost = serial FLOPs
    g = zoo.alexnet()
    K, Ls, Ws = O.cost_tables(g, 1)
    assert all(k == 1 for k in K) and all((w == 0).all() for w in Ws)
    serial = 0
    for nd in g["nodes"]:
        sz = [d["size"] for d in nd["dims"]]
        fd = nd["flop_dims"] if nd["flop_dims"] is not None else range(len(sz))
        serial += nd["flops_per_point"] * math.prod(sz[k] for k in fd)
    r = O.Problem(g, K, Ls, Ws).dp()
    assert r["cost"] == float(serial) and list(r["strategy"]) == [0] * len(K)


def test_alexnet_fc_alternation_zero_transfer():
    """FC (1,4,8) -> FC (1,8,4) 'eliminates any inter-layer communication'."""
    g = zoo.alexnet()
    names = [n["name"] for n in g["nodes"]]
    cf = O.configs(g, 32)
    K, Ls, Ws = O.cost_tables(g, 32)
    f1, f2 = names.index("fc1"), names.index("fc2")
    e = [i for i, ed in enumerate(g["edges"]) if ed["src"] == f1 and ed["dst"] == f2][0]
    a = [tuple(c) for c in cf[f1]].index((1, 4, 8))
    b = [tuple(c) for c in cf[f2]].index((1, 8, 4))
    assert Ws[e][a, b] == 0.0
    # batch-split producer -> column-split consumer: every device needs the whole batch
    a2 = [tuple(c) for c in cf[f1]].index((32, 1, 1))
    b2 = [tuple(c) for c in cf[f2]].index((1, 32, 1))
    assert Ws[e][a2, b2] == 1000.0 * 2 * 4 * (128 * 4096 - 4 * 4096)


def test_transfer_symmetric_in_cost_and_reduction_allreduce():
    """t_x >= 0; a reduction split pays an all-reduce of the output."""
    g = zoo.gemm_single(64, 64, 64)
    cf = [tuple(c) for c in O.configs(g, 8)[0]]
    K, Ls, _ = O.cost_tables(g, 8)
    # (1,4,2): compute 6*64*16*32, reduction all-reduce 2*(2-1)*(4*64*16)/2 bytes * r
    expect = 6 * 64 * 16 * 32 + 1000.0 * (2 * 1 * (4 * 64 * 16)) / 2
    assert Ls[0][cf.index((1, 4, 2))] == expect


# --------------------------------------------------------------------------- Theorem 1
@pytest.mark.parametrize("kind", ["int", "real"])
def test_theorem1_dp_equals_bruteforce(kind):
    """f(|V|, ∅) = min_phi cost(G, phi) for any ordering (SortNodes and BFS),
    on 250 random weakly connected graphs per cost kind (500 total)."""
    checked = 0
    seed = 0
    while checked < 250:
        seed += 1
        n = 2 + seed % 7
        g, p = zoo.random_chain_graph(n, seed, kmax=12 if n <= 5 else 6, extra_p=0.35,
                                      multi_p=0.15 if seed % 5 == 0 else 0.0)
        K = np.array([len(c) for c in O.configs(g, p, O.LE_P)], np.int32)
        if np.prod(K.astype(float)) > 3e5:
            continue
        Ls, Ws = random_costs(g, K, seed, kind)
        P = O.Problem(g, K, Ls, Ws)
        bf = P.brute()
        for order in (0, 1):
            dp = P.dp(order=order)
            if kind == "int":
                assert dp["cost"] == bf["cost"], (seed, order)
                assert P.eval(dp["strategy"]) == bf["cost"]
            else:
                assert rel_eq(dp["cost"], bf["cost"]), (seed, order)
                assert rel_eq(P.eval(dp["strategy"]), bf["cost"])
        eq2 = P.dp_bfs_eq2()
        assert rel_eq(eq2["cost"], bf["cost"]), seed
        checked += 1


def test_theorem1_model_costs_random_graphs():
    """Theorem 1 on random graphs with the cost MODEL (random dims, maps, halos)."""
    done = 0
    for seed in range(200):
        g = zoo.random_model_graph(2 + seed % 5, seed, max_log=3)
        K, Ls, Ws = O.cost_tables(g, 4, O.EXACT_P)
        if np.prod(K.astype(float)) > 2e5:
            continue
        P = O.Problem(g, K, Ls, Ws)
        bf, dp = P.brute(), P.dp()
        assert rel_eq(dp["cost"], bf["cost"]), seed
        assert rel_eq(P.eval(dp["strategy"]), bf["cost"]), seed
        done += 1
    assert done >= 100


# --------------------------------------------------------------------------- Theorem 2 + Fig. 3
def test_theorem2_sortnodes_sets_are_dependent_sets():
    """SortNodes' incremental v.d equals D(i) = N(X(i)) ∩ sigma_>i at every rank,
    on 1000 random graphs with |V| <= 12."""
    for seed in range(1000):
        n = 1 + seed % 12
        g, p = zoo.random_chain_graph(n, seed, kmax=3, extra_p=0.1 + 0.4 * (seed % 3) / 2,
                                      multi_p=0.1 if seed % 7 == 0 else 0.0)
        K = np.ones(n, np.int32)
        P = O.Problem(g, K, [np.zeros(1)] * n, [np.zeros((1, 1))] * len(g["edges"]))
        sigma, dsets = P.sortnodes()
        assert sorted(sigma.tolist()) == list(range(n))
        rank = {v: i for i, v in enumerate(sigma)}
        for i in range(n):
            s = P.sets(sigma, i)
            assert set(dsets[i]) == s["D"], (seed, i)
            assert all(rank[u] > i for u in dsets[i])
            assert s["D"] <= s["Dbar"]
            # connected subsets partition X(i) - {sigma_i} (App. A)
            union = set().union(*s["S"]) if s["S"] else set()
            assert union == s["X"] - {int(sigma[i])}
            assert sum(len(x) for x in s["S"]) == len(union)
        assert dsets[-1] == []                                       # D(|V|) = ∅ (connected)


def test_fig3_worked_example():
    gold = json.load(open(os.path.join(GOLD, "fig3_toy.json")))
    g = zoo.toy_fig3()
    assert [(e["src"] + 1, e["dst"] + 1) for e in g["edges"]] == [tuple(x) for x in gold["edges_1based"]]
    n = len(g["nodes"])
    P = O.Problem(g, np.ones(n, np.int32), [np.zeros(1)] * n, [np.zeros((1, 1))] * len(g["edges"]))
    sigma = np.array(gold["sigma_1based"]) - 1
    s = P.sets(sigma, gold["rank_1based"] - 1)
    one = lambda xs: {x - 1 for x in xs}
    assert s["X"] == one(gold["X"])
    assert sorted(map(sorted, s["S"])) == sorted(sorted(one(x)) for x in gold["S"])
    assert s["D"] == one(gold["D"])
    assert s["Dbar"] == one(gold["Dbar"])
    # Fig. 3 costs: DP = brute force on the toy graph at p=4 (3^9 strategies)
    Pm = O.Problem.from_model(g, 4)
    assert rel_eq(Pm.dp()["cost"], Pm.brute()["cost"])


# --------------------------------------------------------------------------- special cases
def _viterbi_path(order, graph, Ls, Ws):
    """Independent min-plus chain recursion (textbook Viterbi) on a path graph."""
    eidx = {}
    for i, e in enumerate(graph["edges"]):
        eidx[(e["src"], e["dst"])] = (i, False)
        eidx[(e["dst"], e["src"])] = (i, True)
    f = Ls[order[0]].copy()
    for a, b in zip(order, order[1:]):
        i, flip = eidx[(a, b)]
        W = Ws[i].T if flip else Ws[i]               # W[c_a, c_b]
        f = Ls[b] + np.min(f[:, None] + W, axis=0)
    return f.min()


def test_path_graphs_viterbi():
    """path graphs (AlexNet, MLP) -> the DP is a min-plus chain."""
    for seed in range(60):
        n = 2 + seed % 9
        g = zoo.GraphBuilder()
        for i in range(n):
            g.node(f"p{i}", "t", [("x", 1 << (seed * 7 + i) % 5)], out=["x"])
        for i in range(n - 1):
            if (seed + i) % 2:
                g.edge(i, i + 1)
            else:
                g.edge(i + 1, i)
        gr = g.graph()
        K = np.array([len(c) for c in O.configs(gr, 16, O.LE_P)], np.int32)
        Ls, Ws = random_costs(gr, K, seed, "int")
        P = O.Problem(gr, K, Ls, Ws)
        assert P.dp()["cost"] == _viterbi_path(list(range(n)), gr, Ls, Ws)
    # AlexNet with the model costs (M = 1)
    g = zoo.alexnet()
    P = O.Problem.from_model(g, 8)
    assert rel_eq(P.dp()["cost"], _viterbi_path(list(range(len(g["nodes"]))), g, P.Ls, P.Ws))
    sigma, ds = P.sortnodes()
    assert max(len(d) for d in ds) == 1


def _tree_dp(graph, Ls, Ws, root=0):
    """Independent recursive min-sum message passing on a tree."""
    n = len(graph["nodes"])
    adj = [[] for _ in range(n)]
    for i, e in enumerate(graph["edges"]):
        adj[e["src"]].append((e["dst"], i, False))
        adj[e["dst"]].append((e["src"], i, True))

    def g(v, parent):
        acc = Ls[v].copy()
        for (u, i, flip) in adj[v]:
            if u == parent:
                continue
            W = Ws[i].T if flip else Ws[i]           # W[c_v, c_u]
            acc = acc + np.min(W + g(u, v)[None, :], axis=1)
        return acc
    return g(root, -1).min()


def test_trees_message_passing():
    """P:398-401 sparse graphs: on trees SortNodes eliminates leaves (M = 1)."""
    for seed in range(80):
        n = 2 + seed % 10
        g, p = zoo.random_chain_graph(n, seed, kmax=6, extra_p=0.0)
        K = np.array([len(c) for c in O.configs(g, p, O.LE_P)], np.int32)
        Ls, Ws = random_costs(g, K, seed, "int")
        P = O.Problem(g, K, Ls, Ws)
        assert P.dp()["cost"] == _tree_dp(g, Ls, Ws)
        _, ds = P.sortnodes()
        assert max(len(d) for d in ds) <= 1


@pytest.mark.parametrize("name", ["alexnet", "inception_v3", "rnnlm"])
def test_separable_r0(name):
    """Eq. 1 with r = 0 (B -> inf): W == 0, optimum = sum_v min L_v and the DP's
    strict-< tie rule picks the lowest-index argmin of L_v at every vertex."""
    g, p = zoo.bench_graph(name)
    K, Ls, Ws = O.cost_tables(g, p, O.EXACT_P, {"flops": 1e13, "bandwidth": math.inf})
    assert all((w == 0).all() for w in Ws)
    P = O.Problem(g, K, Ls, Ws)
    r = P.dp()
    assert list(r["strategy"]) == [int(np.argmin(l)) for l in Ls]
    assert rel_eq(r["cost"], sum(float(np.min(l)) for l in Ls))


def test_telescoping_identity():
    """App. A: sum_i h(i, phi) = cost(G, phi) for any phi, any ordering."""
    rng = np.random.default_rng(5)
    for seed in range(100):
        g, p = zoo.random_chain_graph(3 + seed % 9, seed, kmax=5, multi_p=0.2 if seed % 3 == 0 else 0)
        K = np.array([len(c) for c in O.configs(g, p, O.LE_P)], np.int32)
        Ls, Ws = random_costs(g, K, seed, "int")
        P = O.Problem(g, K, Ls, Ws)
        phi = np.array([rng.integers(0, k) for k in K], np.int32)
        sigma, _ = P.sortnodes()
        assert P.sum_h(sigma, phi) == P.eval(phi)
        assert P.sum_h(P.bfs_order(), phi) == P.eval(phi)


# --------------------------------------------------------------------------- zoo statistics
def test_inception_statistics():
    """P:680-683 (218 nodes, 12 of degree >= 5), P:703-704 (171, 193 high degree),
    P:692-693 (SortNodes |D(i) ∪ {sigma_i}| <= 3), P:687-688 (BF dependent sets large)."""
    g = zoo.inception_v3()
    assert len(g["nodes"]) == 218
    deg = degrees(g)
    assert sum(d >= 5 for d in deg) == 12 and sum(d < 5 for d in deg) == 206
    assert g["nodes"][171]["name"] == "Mixed_7a/concat" and deg[171] >= 5
    assert g["nodes"][193]["name"] == "Mixed_7b/concat" and deg[193] >= 5
    n = len(g["nodes"])
    P = O.Problem(g, np.ones(n, np.int32), [np.zeros(1)] * n, [np.zeros((1, 1))] * len(g["edges"]))
    _, ds = P.sortnodes()
    assert max(len(d) for d in ds) + 1 <= 3
    sb = P.bfs_order()
    dbar = max(len(P.sets(sb, i)["Dbar"]) for i in range(0, n, 3))
    assert dbar >= 6


def test_ordering_invariance_full_scale():
    """Theorem 1 holds for ANY sigma: relabelling vertex ids changes SortNodes'
    ties, sigma and every table, but not the optimum."""
    g, p = zoo.bench_graph("inception_v3")
    base = O.Problem.from_model(g, p).dp()
    for seed in (1, 2):
        g2, perm = relabel(g, seed)
        r = O.Problem.from_model(g2, p).dp()
        assert rel_eq(r["cost"], base["cost"])


@pytest.mark.parametrize("name", ["mlp", "alexnet", "inception_v3", "rnnlm"])
def test_reevaluation_and_data_parallel_bound(name):
    """cost(G, phi*) reproduces f(|V|, ∅); optimum <= pure data parallel."""
    g, p = zoo.bench_graph(name)
    P = O.Problem.from_model(g, p)
    r = P.dp()
    assert rel_eq(P.eval(r["strategy"]), r["cost"])
    cf = O.configs(g, p)
    dp_strat = []
    for v, nd in enumerate(g["nodes"]):
        best = max(range(len(cf[v])), key=lambda c: (cf[v][c][0], -c))   # largest batch split
        dp_strat.append(best)
    assert r["cost"] <= P.eval(dp_strat)


def test_bfs_guard_trips_on_inception():
    """Table 1 'OOM': the BF-ordered DP exceeds a 1e8-entry table limit."""
    g, p = zoo.inception_v3(), 8
    P = O.Problem.from_model(g, p)
    with pytest.raises(O.OracleError) as ei:
        P.dp(order=1, table_limit=10 ** 8)
    assert ei.value.code == 2
    off, _ = P.table_sizes(order=0)
    assert off[-1] < 10 ** 8


# --------------------------------------------------------------------------- reading L / K / counts
def _node(g, name):
    return [n["name"] for n in g["nodes"]].index(name)


def test_conv_halo_closed_form():
    """P:228 'halo communication for convolutions', reading L: the face of a split spatial dim
    runs over the INPUT-tensor axes (b, c, w for h).  Hand-derived values (golden); the second
    config splits c and n, so a face over the output axes (s_n instead of s_c) fails it."""
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))["conv_halo_inception_mixed_7b_b2_3x3"]
    g = zoo.inception_v3()
    v = _node(g, gold["node"])
    cf = [tuple(c) for c in O.configs(g, gold["p"])[v]]
    K, Ls, _ = O.cost_tables(g, gold["p"])
    for key, tup in (("config_16_1_2_1_1_1_1", (16, 1, 2, 1, 1, 1, 1)), ("config_4_2_2_1_2_1_1", (4, 2, 2, 1, 2, 1, 1))):
        assert Ls[v][cf.index(tup)] == gold[key]["t_l"], key
    # no halo when the spatial dims are unsplit, whatever else is split
    c0 = cf.index((32, 1, 1, 1, 1, 1, 1))
    w_bytes = 4 * 448 * 384 * 9
    assert Ls[v][c0] == 2378170368 + 1000.0 * (2 * 31 * w_bytes // 32)


def test_tx_unmapped_axis_closed_form():
    """P:271-276, reading K: an axis the consumer does not split (axis_map -1) is needed whole."""
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))["tx_unmapped_axis_alexnet_pool3_fc1"]
    g = zoo.alexnet()
    a, b = _node(g, "pool3"), _node(g, "fc1")
    e = [i for i, ed in enumerate(g["edges"]) if ed["src"] == a and ed["dst"] == b][0]
    assert g["edges"][e]["axis_map"][2:] == [-1, -1]
    cf = O.configs(g, gold["p"])
    K, Ls, Ws = O.cost_tables(g, gold["p"])
    ia = [tuple(c) for c in cf[a]].index((1, 4, 2, 1, 1, 1))
    ib = [tuple(c) for c in cf[b]].index((1, 1, 8))
    assert Ws[e][ia, ib] == gold["W"]
    # producer with unsplit h, w holds everything the flatten needs along them: only c matters
    ia2 = [tuple(c) for c in cf[a]].index((1, 8, 1, 1, 1, 1))
    assert Ws[e][ia2, ib] == 0.0


def test_candidate_counts_closed_form():
    """Sum_i K(sigma_i)|T(i)| of the two brute-force-sized BASELINE configs (hand-derived)."""
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))["candidate_counts"]
    for name, key in (("mlp", "mlp_p4"), ("alexnet", "alexnet_p8")):
        g, p = zoo.bench_graph(name)
        K = np.array([len(c) for c in O.configs(g, p)], np.int32)
        assert list(K) == gold[key]["K"], name
        P = O.Problem(g, K, [np.zeros(k) for k in K], [np.zeros((K[e["src"]], K[e["dst"]])) for e in g["edges"]])
        assert P.table_sizes()[1] == gold[key]["candidates"], name


def test_halo_requires_input_axes():
    """Reading L: a halo pair must name a spatial dim of the input tensor."""
    g = zoo.GraphBuilder()
    g.node("c", "conv2d", [("b", 8), ("h", 8), ("r", 3)], out=["b", "h"], halo=[("h", "r")], inp=["b"])
    assert O.validate(g.graph()) == 1
    g = zoo.GraphBuilder()
    g.node("c", "conv2d", [("b", 8), ("h", 8), ("r", 3)], out=["b", "h"], halo=[("h", "r")], inp=["b", "h"])
    assert O.validate(g.graph()) == 0
