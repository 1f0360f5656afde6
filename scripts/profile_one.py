"""One search of a bench workload (for ncu).  `--top` prints the rank of the DP vertex with
the most candidates (with PASE_NO_GRAPH=1 the DP kernels launch in rank order, so that
rank is the --launch-skip of the dominant dp_fill launch)."""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", default="transformer", nargs="?")
ap.add_argument("--top", action="store_true")
ap.add_argument("--solves", type=int, default=1)
a = ap.parse_args()
key, p, policy, _ = WORKLOADS[a.workload]
g = zoo.bench_graph(key)[0]
if a.top:
    ctx = pase.Context(g, p, policy=policy, device=-1)
    K = ctx.K()
    sigma, deps, _ = ctx.order()
    cand = [int(K[sigma[i]]) * math.prod(int(K[u]) for u in deps[i]) for i in range(len(sigma))]
    print(max(range(len(cand)), key=lambda i: cand[i]))
    sys.exit(0)
ctx = pase.Context(g, p, policy=policy, device=0)
for _ in range(a.solves):
    r = ctx.solve()
print(r["cost"], ctx.stats()["ms_solve"])
