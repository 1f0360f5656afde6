"""Row f2: Eq. 1 on the GPU -- pase_evaluate and pase_brute_force.

Pins: (i) the GPU brute force equals the oracle's CPU brute force bit for bit
(same definition, same summation order, same lowest-index tie rule) on random graphs with
tie-heavy integer and rounding-heavy real costs; (ii) by Theorem 1 its minimum
equals the DP total (1e-12 relative: the DP associates the sum differently), which the GPU
brute force checks at sizes no CPU brute force reaches -- the whole AlexNet p=8 benchmark
config (BASELINE configs[1], 3.1e10 strategies); (iii) pase_evaluate equals the oracle's
Eq. 1 evaluation bit for bit on random strategies of every zoo graph.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_04001_b200 import pase, zoo
from tests.helpers import random_costs

pytestmark = pytest.mark.gpu


def rel_eq(a, b, tol=1e-12):
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))


def bits(x):
    return int(np.float64(x).view(np.uint64))


@pytest.mark.parametrize("kind", ["int", "real"])
def test_brute_force_matches_cpu_brute_force(kind):
    for seed in range(40):
        n = 1 + seed % 8
        g, p = zoo.random_chain_graph(n, 500 + seed, kmax=10 if n <= 5 else 6, extra_p=0.4,
                                      multi_p=0.2 if seed % 3 == 0 else 0.0)
        K = np.array([len(c) for c in O.configs(g, p, O.LE_P)], np.int32)
        if np.prod(K.astype(float)) > 3e5:
            continue
        Ls, Ws = random_costs(g, K, 2000 + seed, kind)
        P = O.Problem(g, K, Ls, Ws)
        bf = P.brute()
        with pase.Context(g, p, policy="le_p", device=0) as ctx:
            ctx.set_cost_tables(Ls, Ws)
            r = ctx.brute_force()
            dp = ctx.solve()
        assert r["n_strategies"] == int(np.prod(K.astype(np.int64)))
        assert bits(r["cost"]) == bits(bf["cost"]), (seed, r["cost"], bf["cost"])
        assert list(r["config_index"]) == list(bf["strategy"]), seed
        assert rel_eq(dp["cost"], r["cost"]), seed                        # Theorem 1


@pytest.mark.parametrize("name", ["mlp", "alexnet", "inception_v3", "rnnlm", "gnmt", "transformer"])
def test_evaluate_matches_oracle_eval(name):
    g, p = zoo.bench_graph(name)
    P = O.Problem.from_model(g, p)
    rng = np.random.default_rng(7)
    S = np.stack([rng.integers(0, P.K) for _ in range(64)]).astype(np.int32)
    with pase.Context(g, p, device=0) as ctx:
        got = ctx.evaluate(S)
        dp = ctx.solve()
        re = ctx.evaluate(dp["config_index"])[0]
    for s in range(len(S)):
        assert bits(got[s]) == bits(P.eval(S[s])), (name, s)
    # re-evaluation of phi* (SURVEY §8.c.3): Eq. 1 of the DP's strategy = the DP total
    assert bits(re) == bits(P.eval(dp["config_index"]))
    assert rel_eq(re, dp["cost"])


def test_brute_force_full_alexnet_config():
    """Theorem 1 at a benchmark config: exhaustive minimum over all 3.07e10 AlexNet p=8
    strategies = the DP optimum; the DP's strategy attains it."""
    g, p = zoo.bench_graph("alexnet")
    with pase.Context(g, p, device=0) as ctx:
        dp = ctx.solve()
        r = ctx.brute_force(max_strategies=1 << 36)
        e = ctx.evaluate(np.stack([dp["config_index"], r["config_index"]]))
    assert r["n_strategies"] == 30_720_000_000
    assert rel_eq(dp["cost"], r["cost"])
    assert rel_eq(e[0], r["cost"]) and bits(e[1]) == bits(r["cost"])
    # the DP strategy is optimal: no strategy is strictly cheaper beyond rounding
    assert e[0] <= r["cost"] * (1 + 1e-12)


def test_brute_force_model_costs_toy_and_mlp():
    for g, p in ((zoo.toy_fig3(), 4), zoo.bench_graph("mlp")):
        P = O.Problem.from_model(g, p)
        bf = P.brute(limit=10 ** 8)
        with pase.Context(g, p, device=0) as ctx:
            r = ctx.brute_force()
            dp = ctx.solve()
        assert bits(r["cost"]) == bits(bf["cost"])
        assert list(r["config_index"]) == list(bf["strategy"])
        assert rel_eq(dp["cost"], r["cost"])


def test_eq1_errors():
    g, p = zoo.bench_graph("alexnet")
    with pase.Context(g, p, device=0) as ctx:
        with pytest.raises(pase.PaseError) as ei:
            ctx.brute_force(max_strategies=1000)
        assert ei.value.status == 2 and "limit" in str(ei.value)
        bad = np.zeros(ctx.n, np.int32)
        bad[3] = 999
        with pytest.raises(pase.PaseError) as ei:
            ctx.evaluate(bad)
        assert ei.value.status == 1 and "node 3" in str(ei.value)
        assert len(ctx.evaluate(np.zeros((0, ctx.n), np.int32))) == 0
