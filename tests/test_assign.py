"""Row f3: greedy device assignment (DESIGN reading U).

Pins of the oracle (or_assign) against the definition of t_x ("max_d |A(v,d,phi)|
- |A(v,d,phi) ∩ A(u,d,phi)|"), evaluated here on explicit element sets of tiny tensors:
  * the realized t_x the oracle reports equals the element-set count for its assignment;
  * over ALL device permutations of a single edge, the best realized t_x equals the cost
    model's aligned t_x (reading K: aligned = the locality-maximising assignment), and the
    greedy assignment reaches it;
  * realized >= aligned on every edge of every zoo strategy (lower bound), with equality on
    chains; AlexNet's alternating FC splits need no transfer at all.
Then the library's host implementation (pase_assign_devices) must equal the oracle exactly.
Host-side only: no GPU."""
import itertools
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_04001_b200 import pase, zoo

R = 1000.0   # F / B of the zoo machine (DESIGN reading R)


def shard_box(node, tup, s, axes_dims, mapping=None, ext=None):
    """Per output axis, the [lo, hi) interval of shard s.  Producer: axis a is iteration dim
    axes_dims[a]; consumer: mapping[a] (None = whole axis)."""
    d = len(node["dims"])
    digits = []
    x = s
    for k in range(d - 1, -1, -1):
        digits.append(x % tup[k])
        x //= tup[k]
    digits = digits[::-1]
    box = []
    for a in range(len(axes_dims)):
        if mapping is None:
            k = axes_dims[a]
            h = node["dims"][k]["size"] // tup[k]
            box.append((digits[k] * h, digits[k] * h + h))
        elif mapping[a] < 0:
            box.append((0, ext[a]))
        else:
            k = mapping[a]
            part = -(-ext[a] // tup[k])
            box.append((digits[k] * part, min(ext[a], digits[k] * part + part)))
    return box


def mask(shape, box):
    m = np.zeros(shape, bool)
    m[tuple(slice(lo, hi) for lo, hi in box)] = True
    return m


def missing_matrix(graph, e, tu, tw):
    """M[i, j] = elements consumer shard j needs that producer shard i does not hold
    (explicit element sets), plus |need_j|."""
    ed = graph["edges"][e]
    u, w = graph["nodes"][ed["src"]], graph["nodes"][ed["dst"]]
    ext = [u["dims"][k]["size"] for k in u["out_axes"]]
    su, sw = math.prod(tu[:len(u["dims"])]), math.prod(tw[:len(w["dims"])])
    held = [mask(ext, shard_box(u, tu, i, u["out_axes"])) for i in range(su)]
    need = [mask(ext, shard_box(w, tw, j, u["out_axes"], ed["axis_map"], ext)) for j in range(sw)]
    M = np.array([[int((need[j] & ~held[i]).sum()) for j in range(sw)] for i in range(su)])
    return M, np.array([int(x.sum()) for x in need])


def realized_elements(graph, e, tu, tw, dev_u, dev_w):
    """max over devices holding a consumer shard of (needed - needed ∩ held), elements."""
    M, need = missing_matrix(graph, e, tu, tw)
    worst = 0
    for j, d in enumerate(dev_w):
        if d < 0:
            continue
        hits = np.nonzero(dev_u == d)[0]
        worst = max(worst, int(M[hits[0], j]) if len(hits) else int(need[j]))
    return worst


def tuples_of(graph, p, strategy, policy=O.EXACT_P):
    cf = O.configs(graph, p, policy)
    return [tuple(int(x) for x in cf[v][strategy[v]]) for v in range(len(graph["nodes"]))]


def two_node_graph(seed):
    rng = np.random.default_rng(seed)
    g = zoo.GraphBuilder()
    dims_u = [("b", int(2 ** rng.integers(1, 4))), ("n", int(2 ** rng.integers(1, 4))),
              ("c", int(2 ** rng.integers(0, 3)))]
    dims_w = [("b", dims_u[0][1]), ("m", int(2 ** rng.integers(1, 3))), ("n", dims_u[1][1])]
    g.node("u", "gemm", dims_u, out=["b", "n"], w=["n", "c"], fpp=6)
    g.node("w", "gemm", dims_w, out=["b", "m"], w=["m", "n"], fpp=6)
    ren = {"b": "b" if rng.random() < 0.8 else None, "n": "n" if rng.random() < 0.8 else None}
    g.edge(0, 1, ren)
    return g.graph()


@pytest.mark.parametrize("p", [4, 8])
def test_single_edge_aligned_is_best_assignment(p):
    """Reading K: for one edge whose endpoints both use all p devices, the aligned t_x of the
    cost model is the minimum over every device permutation of the definition's max_d |A(v,d)| - |A(v,d) ∩ A(u,d)|; the greedy
    placement attains it, and the oracle's realized t_x equals the element-set count."""
    checked = 0
    for seed in range(12 if p == 8 else 20):
        g = two_node_graph(seed)
        K, Ls, Ws = O.cost_tables(g, p, O.EXACT_P)
        cf = O.configs(g, p, O.EXACT_P)
        rng = np.random.default_rng(100 + seed)
        for _ in range(3):
            a, b = int(rng.integers(K[0])), int(rng.integers(K[1]))
            tu, tw = tuple(int(x) for x in cf[0][a]), tuple(int(x) for x in cf[1][b])
            su, sw = math.prod(tu), math.prod(tw)
            if su != p or sw != p:       # every device holds a producer shard (see reading U)
                continue
            aligned = Ws[0][a, b] / R / (2 * 4)             # elements
            M, need = missing_matrix(g, 0, tu, tw)
            best = None
            dev_u = np.arange(su)
            for perm in itertools.permutations(range(p), sw):  # consumer shard j on device perm[j]
                worst = 0
                for j, d in enumerate(perm):
                    worst = max(worst, int(M[d, j]) if d < su else int(need[j]))
                best = worst if best is None else min(best, worst)
            assert best == aligned, (seed, tu, tw, best, aligned)
            dev, tx = O.assign_devices(g, p, [tu, tw])
            got = realized_elements(g, 0, tu, tw, dev[0][:su], dev[1][:sw])
            assert tx[0] == 2 * 4 * got
            assert got == aligned, (seed, tu, tw)
            checked += 1
    assert checked >= 20


def test_realized_matches_element_sets_on_small_graphs():
    for seed in range(25):
        g = zoo.random_model_graph(2 + seed % 5, 700 + seed, max_log=3)
        p = 4 << (seed % 2)
        K = [len(c) for c in O.configs(g, p, O.LE_P)]
        rng = np.random.default_rng(seed)
        strat = [int(rng.integers(k)) for k in K]
        tups = tuples_of(g, p, strat, O.LE_P)
        dev, tx = O.assign_devices(g, p, tups)
        for v, t in enumerate(tups):                       # a valid placement
            s = math.prod(t[:len(g["nodes"][v]["dims"])])
            assert sorted(dev[v][:s]) == sorted(set(dev[v][:s])) and (dev[v][:s] >= 0).all()
            assert (dev[v][:s] < p).all() and (dev[v][s:] == -1).all()
        for e, ed in enumerate(g["edges"]):
            u, w = ed["src"], ed["dst"]
            su = math.prod(tups[u][:len(g["nodes"][u]["dims"])])
            sw = math.prod(tups[w][:len(g["nodes"][w]["dims"])])
            elem = g["nodes"][u]["elem_bytes"]
            assert tx[e] == 2 * elem * realized_elements(g, e, tups[u], tups[w], dev[u][:su], dev[w][:sw])


@pytest.mark.parametrize("name", ["mlp", "alexnet", "inception_v3", "rnnlm", "gnmt", "transformer"])
def test_lower_bound_and_library_parity(name):
    g, p = zoo.bench_graph(name)
    P = O.Problem.from_model(g, p)
    strategies = [P.dp(threads=4)["strategy"]]
    rng = np.random.default_rng(5)
    strategies.append([int(rng.integers(k)) for k in P.K])
    with pase.Context(g, p, device=-1) as ctx:
        for k, strat in enumerate(strategies):
            dev, tx = O.assign_devices(g, p, tuples_of(g, p, strat))
            aligned = np.array([P.Ws[e][strat[ed["src"]], strat[ed["dst"]]] / R
                                for e, ed in enumerate(g["edges"])])
            assert (tx >= aligned).all(), name                  # lower bound (reading K)
            if name in ("mlp", "alexnet") and k == 0:          # chains reach it
                assert np.array_equal(tx, aligned)
            d2, t2 = ctx.assign_devices(strat)
            assert np.array_equal(dev, d2) and np.array_equal(tx, t2), name


def test_alexnet_fc_alternation_needs_no_transfer():
    """P:988-992 at p = 32 (Table 2): FC1 (1,4,8) -> FC2 (1,8,4) -> FC3 (1,4,8) placed greedily
    moves nothing between the FC layers."""
    g = zoo.alexnet()
    p = 32
    cf = O.configs(g, p)
    names = [n["name"] for n in g["nodes"]]
    P = O.Problem.from_model(g, p)
    strat = list(P.dp(threads=4)["strategy"])
    want = {"fc1": (1, 4, 8), "fc2": (1, 8, 4), "fc3": (1, 4, 8)}
    for nm, t in want.items():
        v = names.index(nm)
        strat[v] = [tuple(int(x) for x in c) for c in cf[v]].index(t)
    with pase.Context(g, p, device=-1) as ctx:
        dev, tx = ctx.assign_devices(strat)
    for e, ed in enumerate(g["edges"]):
        if names[ed["src"]] in ("fc1", "fc2") and names[ed["dst"]] in ("fc2", "fc3"):
            assert tx[e] == 0.0


def test_assign_rejects_bad_index():
    g, p = zoo.bench_graph("mlp")
    with pase.Context(g, p, device=-1) as ctx:
        with pytest.raises(pase.PaseError) as ei:
            ctx.assign_devices([0, 0, 99, 0])
        assert ei.value.status == 1 and "node 2" in str(ei.value)
