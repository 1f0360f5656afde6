"""C-ABI library checks that need no GPU: every symbol of include/pase.h is exported,
the ctypes mirror matches the C struct layout, and the host core (rows a1-a4:
ingest, C(v), SortNodes, elimination tree) agrees with the oracle on every graph.
Uses host-only planning contexts (machine.cuda_device < 0): no device work."""
import os
import re
import subprocess

import ctypes as C
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_04001_b200 import build as B
from paper_2407_04001_b200 import pase, zoo
from tests.helpers import relabel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "pase.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return pase.load()


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:pase_status|const char\*|void|int64_t)\s+(pase_\w+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 13
    out = subprocess.run(["nm", "-D", "--defined-only", B.SO], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (pase_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(pase.EXPORTS) == set(syms)
    for s in syms:
        getattr(lib, s)


def test_struct_layout_matches_header(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text("""
#include <stdio.h>
#include <stddef.h>
#include "pase.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\\n", sizeof(pase_node), sizeof(pase_edge), sizeof(pase_graph),
         sizeof(pase_machine), sizeof(pase_stats));
  printf("%zu %zu %zu %zu\\n", offsetof(pase_node, flops_per_point), offsetof(pase_node, elem_bytes),
         offsetof(pase_machine, reserved), offsetof(pase_stats, ms_create));
  return 0;
}
""")
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    lines = subprocess.check_output([str(exe)], text=True).split("\n")
    sizes = [int(x) for x in lines[0].split()]
    assert sizes == [C.sizeof(pase.pase_node), C.sizeof(pase.pase_edge), C.sizeof(pase.pase_graph),
                     C.sizeof(pase.pase_machine), C.sizeof(pase.pase_stats)]
    offs = [int(x) for x in lines[1].split()]
    assert offs == [pase.pase_node.flops_per_point.offset, pase.pase_node.elem_bytes.offset,
                    pase.pase_machine.reserved.offset, pase.pase_stats.ms_create.offset]


def check_plan_against_oracle(graph, p, policy):
    ctx = pase.Context(graph, p, policy=policy, device=-1)
    pol = pase.POLICIES[policy]
    # a2: C(v) identical tuples, identical order
    oc = O.configs(graph, p, pol)
    gc = ctx.configs()
    assert len(oc) == len(gc)
    for a, b in zip(oc, gc):
        assert np.array_equal(a, b)
    # a3: sigma and D(i) identical (SortNodes readings C, D)
    K = np.array([len(c) for c in oc], np.int32)
    n = len(K)
    P = O.Problem(graph, K, [np.zeros(k) for k in K],
                  [np.zeros((K[e["src"]], K[e["dst"]])) for e in graph["edges"]])
    osig, odeps = P.sortnodes()
    sigma, deps, parent = ctx.order()
    assert list(sigma) == list(osig)
    assert deps == [list(map(int, d)) for d in odeps]
    # a4: elimination tree == Fig. 5's connected subsets: S(i) lookups j are exactly children(i)
    rank = {int(v): i for i, v in enumerate(sigma)}
    for i in range(n):
        s = P.sets(sigma, i)
        js = sorted(max(rank[v] for v in comp) for comp in s["S"])
        kids = [j for j in range(n) if parent[j] == i]
        assert js == kids, (i, js, kids)
    st = ctx.stats()
    off, cand = P.table_sizes()
    assert st["candidates"] == cand and st["table_entries"] == off[-1]
    assert st["max_dep"] == max(len(d) for d in deps)
    ctx.close()


@pytest.mark.parametrize("name", ["mlp", "alexnet", "inception_v3", "rnnlm", "gnmt", "transformer"])
def test_host_plan_matches_oracle_zoo(lib, name):
    g, p = zoo.bench_graph(name)
    check_plan_against_oracle(g, p, "exact_p")
    if name in ("mlp", "alexnet", "transformer"):
        check_plan_against_oracle(g, p, "le_p")


def test_host_plan_matches_oracle_random(lib):
    for seed in range(150):
        g = zoo.random_model_graph(1 + seed % 11, seed, multi_p=0.2 if seed % 4 == 0 else 0.0)
        check_plan_against_oracle(g, 4 << (seed % 3), "exact_p" if seed % 2 else "le_p")


def test_host_plan_relabelled(lib):
    g, p = zoo.bench_graph("inception_v3")
    g2, _ = relabel(g, 3)
    check_plan_against_oracle(g2, p, "exact_p")


def test_invalid_inputs_fail_loudly(lib):
    g = zoo.mlp()
    g["edges"].append({"src": 0, "dst": 0, "axis_map": [0, 1]})
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g, 4, device=-1)
    assert ei.value.status == 1 and "self-loop" in str(ei.value)
    g = zoo.mlp()
    g["edges"] = g["edges"][:1]                      # disconnected
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g, 4, device=-1)
    assert ei.value.status == 1 and "connected" in str(ei.value)
    g = zoo.mlp()
    g["edges"][0]["axis_map"] = [0, 7]
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g, 4, device=-1)
    assert ei.value.status == 1 and "edge 0" in str(ei.value)
    # reading L: a halo along a dim that is not an input-tensor axis
    g = zoo.alexnet()
    g["nodes"][0]["in_axes"] = [0, 1]                 # conv1 without h, w
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g, 8, device=-1)
    assert ei.value.status == 1 and "node 0" in str(ei.value) and "input-tensor axis" in str(ei.value)
    assert O.validate(g) == 1                         # the oracle rejects it too
    # r = F/B must be finite (F = inf would make 0 * inf = NaN costs)
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(zoo.mlp(), 4, device=-1, flops=float("inf"))
    assert ei.value.status == 1


def test_solve_needs_device(lib):
    ctx = pase.Context(zoo.mlp(), 4, device=-1)
    with pytest.raises(pase.PaseError) as ei:
        ctx.solve()
    assert ei.value.status == 5


def test_bfs_ordering_plan_matches_oracle(lib):
    """f1: the BFS ordering's dependent sets from the incremental update equal
    the oracle's definitional D(i) for that ordering; the tree rule still gives S(i)."""
    for name in ("mlp", "alexnet", "rnnlm"):
        g, p = zoo.bench_graph(name)
        ctx = pase.Context(g, p, device=-1, ordering="bfs")
        K = ctx.K()
        n = len(K)
        P = O.Problem(g, K, [np.zeros(k) for k in K], [np.zeros((K[e["src"]], K[e["dst"]])) for e in g["edges"]])
        sb = P.bfs_order()
        sigma, deps, parent = ctx.order()
        assert list(sigma) == list(sb)
        rank = {int(v): i for i, v in enumerate(sigma)}
        for i in range(n):
            s = P.sets(sigma, i)
            assert set(deps[i]) == s["D"]
            kids = [j for j in range(n) if parent[j] == i]
            assert sorted(max(rank[v] for v in comp) for comp in s["S"]) == kids
    for seed in range(40):
        g = zoo.random_model_graph(2 + seed % 10, seed)
        ctx = pase.Context(g, 4, device=-1, ordering="bfs")
        P = O.Problem(g, ctx.K(), [np.zeros(k) for k in ctx.K()],
                      [np.zeros((ctx.K()[e["src"]], ctx.K()[e["dst"]])) for e in g["edges"]])
        sigma, deps, _ = ctx.order()
        assert list(sigma) == list(P.bfs_order())
        for i in range(len(sigma)):
            assert set(deps[i]) == P.sets(sigma, i)["D"]


def test_bfs_ordering_oom_on_inception(lib):
    """Table 1: BF ordering runs out of memory on InceptionV3 -- here the size
    guard reports PASE_ERR_RESOURCE with M and K; SortNodes plans it in a few MB."""
    g = zoo.inception_v3()
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g, 8, device=-1, ordering="bfs")
    assert ei.value.status == 2 and "K =" in str(ei.value)
    ctx = pase.Context(g, 8, device=-1)
    assert ctx.stats()["table_entries"] * 10 < 1e9


def test_premarshalled_graph_same_plan(lib):
    """pase.Graph (the C ABI input layout, marshalled once) plans exactly like the dict."""
    g, p = zoo.bench_graph("transformer")
    G = pase.Graph(g)
    a = pase.Context(g, p, device=-1)
    for _ in range(2):
        b = pase.Context(G, p, device=-1)
        sa, da, pa = a.order()
        sb, db, pb = b.order()
        assert list(sa) == list(sb) and list(pa) == list(pb)
        assert np.array_equal(a.K(), b.K())
        b.close()
    a.close()


def test_gnmt_depth_guard(lib):
    """SURVEY §8.d.1 row 4b / sizing rule iii: GNMT 4+4 plans (M = 5, the same candidate count
    as the oracle's Fig. 5 plan); the real 8+8 depth trips the width guard (M = 15 > 12,
    PASE_ERR_RESOURCE naming M and K) -- the BF-'OOM' analogue of Table 1."""
    g, p = zoo.bench_graph("gnmt4")
    ctx = pase.Context(g, p, device=-1)
    st = ctx.stats()
    assert st["max_dep"] == 5 and st["max_configs"] == 28
    K = ctx.K()
    P = O.Problem(g, K, [np.zeros(k) for k in K], [np.zeros((K[e["src"]], K[e["dst"]])) for e in g["edges"]])
    assert P.table_sizes()[1] == st["candidates"]
    g8, p8 = zoo.bench_graph("gnmt8")
    with pytest.raises(pase.PaseError) as ei:
        pase.Context(g8, p8, device=-1)
    assert ei.value.status == 2 and "M = max |D(i)| = 15" in str(ei.value) and "K = 28" in str(ei.value)


def test_streaming_clique_plan(lib):
    """The synthetic streaming benchmark's structure: vertex 0 (K = 1) first with D = the rest,
    vertex 1 next with D(1) = D(0) - {1}: T(0) spans (sigma_1, D(1)) -- 205^4 entries."""
    g, p = zoo.bench_graph("stream205")
    ctx = pase.Context(g, p, device=-1)
    sigma, deps, parent = ctx.order()
    K = ctx.K()
    assert list(sigma[:2]) == [0, 1] and K[0] == 1 and all(k == 205 for k in K[1:])
    assert deps[0] == [1, 2, 3, 4] and deps[1] == [2, 3, 4] and parent[0] == 1
    assert ctx.stats()["table_entries"] > 205 ** 4
