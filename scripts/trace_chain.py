"""Critical chain of a saved PASE_TRACE timeline (gpurun_out/trace_<workload>.npy): per chain
vertex, when its children finished, when its tasks started / computed / synced / released."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "transformer"
tr = np.load(f"gpurun_out/trace_{wl}.npy")
key, p, policy, _ = WORKLOADS[wl]
ctx = pase.Context(zoo.bench_graph(key)[0], p, policy=policy, device=-1)
K = ctx.K()
sigma, deps, parent = ctx.order()
n = len(sigma)
t0 = tr[:, 2].min()
kids = [[] for _ in range(n)]
for j in range(n):
    if parent[j] >= 0:
        kids[parent[j]].append(j)
start, end = {}, {}
for i in range(n):
    m = tr[:, 0] == i
    if m.any():
        start[i] = (tr[m, 3].min() - t0) / 1e3
        end[i] = (tr[m, 6].max() - t0) / 1e3
v, chain = n - 1, []
while True:
    chain.append(v)
    ks = [j for j in kids[v] if j in end]
    if not ks:
        break
    v = max(ks, key=lambda j: end[j])
print(f"{wl}: span {(tr[:, 6].max() - t0) / 1e3:.1f} us, critical chain {len(chain)} vertices")
print("vtx K M cand tasks | kids_end start end | gap | per-task us: claim->start start->comp comp->sync sync->end (max task)")
tot = np.zeros(4)
for v in chain:
    m = tr[:, 0] == v
    cand = int(K[sigma[v]]) * math.prod(int(K[u]) for u in deps[v])
    kend = max([end[j] for j in kids[v]], default=0.0)
    rows = tr[m]
    k = np.argmax(rows[:, 6])
    ph = np.diff(rows[k, 2:7]) / 1e3
    tot += ph
    print(f"{v} {K[sigma[v]]} {len(deps[v])} {cand} {int(m.sum())} | {kend:.1f} {start[v]:.1f} {end[v]:.1f} | "
          f"{start[v] - kend:.1f} | " + " ".join(f"{x:.2f}" for x in ph))
print("chain totals (last task of each vertex): claim->start %.1f start->comp %.1f comp->sync %.1f sync->end %.1f us" % tuple(tot))
