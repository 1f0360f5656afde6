"""One small search per case for compute-sanitizer (SURVEY §5 race / failure detection):
mlp, alexnet, a random synthetic-cost graph (one-lane and narrow tiles), inception (2-D tiles,
latency mode), and a virtual 2-rank group (peer stores, system-scope counters, group barriers).
Every result is checked against the oracle so a sanitizer-perturbed run that still 'passes'
also has to be right."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402
from tests.helpers import random_costs  # noqa: E402

case = sys.argv[1]
if case in ("mlp", "alexnet", "inception_v3"):
    g, p = zoo.bench_graph(case)
    with pase.Context(g, p) as c:
        r = c.solve()
    o = O.Problem.from_model(g, p).dp(threads=os.cpu_count())
    assert list(r["config_index"]) == list(o["strategy"]) and r["cost"] == o["cost"], case
elif case == "random":
    for seed in range(6):
        g, p = zoo.random_chain_graph(3 + seed, 70 + seed, kmax=9, extra_p=0.4)
        K = np.array([len(x) for x in O.configs(g, p, O.LE_P)], np.int32)
        Ls, Ws = random_costs(g, K, seed, "int")
        with pase.Context(g, p, policy="le_p") as c:
            c.set_cost_tables(Ls, Ws)
            r = c.solve()
        o = O.Problem(g, K, Ls, Ws).dp()
        assert list(r["config_index"]) == list(o["strategy"]) and r["cost"] == o["cost"], seed
elif case == "group2":
    g, p = zoo.bench_graph("inception_v3")
    ctxs = pase.virtual_group(g, p, 2, redundant_below=1 << 12)
    res = pase.solve_group(ctxs)
    o = O.Problem.from_model(g, p).dp(threads=os.cpu_count())
    for r in res:
        assert list(r["config_index"]) == list(o["strategy"]) and r["cost"] == o["cost"]
    for c in ctxs:
        c.close()
print("sanitize case ok:", case)
