"""Persistent-schedule timeline of one search (PASE_TRACE=1) + create/solve/destroy timing.
Writes gpurun_out/trace_<workload>.npy and prints a per-vertex summary."""
import math
import os
import sys
import time

os.environ["PASE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "transformer"
key, p, policy, _ = WORKLOADS[wl]
g = zoo.bench_graph(key)[0]
for it in range(4):
    t0 = time.perf_counter()
    gg, keep = pase.marshal_graph(g)
    t1 = time.perf_counter()
    ctx = pase.Context(g, p, policy=policy, device=0)
    t2 = time.perf_counter()
    ctx.solve()
    t3 = time.perf_counter()
    st = ctx.stats()
    ctx.close()
    t4 = time.perf_counter()
    print(f"e2e iter {it}: marshal {1e3*(t1-t0):.2f} ms, create {1e3*(t2-t1):.2f} ms (lib {st['ms_create']:.2f}), "
          f"solve {1e3*(t3-t2):.2f} ms (dev {st['ms_solve']:.3f}), destroy {1e3*(t4-t3):.2f} ms")
ctx = pase.Context(g, p, policy=policy, device=0)
for _ in range(3):
    ctx.solve()
tr = ctx.trace()
K = ctx.K()
sigma, deps, parent = ctx.order()
st = ctx.stats()
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_{wl}.npy", tr)
t0 = tr[:, 2].min()
print(f"dp phase {st['ms_dp']:.3f} ms, tasks {len(tr)}, span {(tr[:, 6].max() - t0) / 1e3:.1f} us")
n = len(sigma)
rows = []
for i in range(n):
    m = tr[:, 0] == i
    if not m.any():
        continue
    cand = int(K[sigma[i]]) * math.prod(int(K[u]) for u in deps[i])
    s, e = tr[m, 3].min() - t0, tr[m, 6].max() - t0
    busy = (tr[m, 6] - tr[m, 3]).sum()
    waitw = (tr[m, 3] - tr[m, 2]).sum()
    rows.append((i, int(m.sum()), cand, s / 1e3, e / 1e3, (e - s) / 1e3, busy / 1e3, waitw / 1e3))
rows.sort(key=lambda r: -r[5])
print("rank tasks cand start_us end_us span_us busy_us wait_us")
for r in rows[:25]:
    print(" ".join(f"{x:.1f}" if isinstance(x, float) else str(x) for x in r))
# critical chain: follow the vertex finishing last backwards through its last-finishing child
kids = [[] for _ in range(n)]
for j in range(n):
    if parent[j] >= 0:
        kids[parent[j]].append(j)
end = {r[0]: r[4] for r in rows}
start = {r[0]: r[3] for r in rows}
v = n - 1
chain = []
while True:
    chain.append(v)
    ks = [j for j in kids[v] if j in end]
    if not ks:
        break
    v = max(ks, key=lambda j: end[j])
print("critical chain (rank:start-end us):", " ".join(f"{v}:{start[v]:.0f}-{end[v]:.0f}" for v in chain[:60]))
