"""Critical chain of a saved PASE_TRACE timeline with the per-warp gate stamps: for the last
task of every chain vertex, the time from its children's last release to its gate opening
(poll latency), the gate's fence, the tile after the fence, the CTA barrier and the release."""
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
end = {}
for i in range(n):
    m = tr[:, 0] == i
    if m.any():
        end[i] = (tr[m, 6].max() - t0) / 1e3
v, chain = n - 1, []
while True:
    chain.append(v)
    ks = [j for j in kids[v] if j in end]
    if not ks:
        break
    v = max(ks, key=lambda j: end[j])
print(f"{wl}: span {(tr[:, 6].max() - t0) / 1e3:.1f} us, critical chain {len(chain)} vertices")
print("vtx K M cand tasks shape? | kids_end | poll fence tile bar rel (us) | warps gated")
tot = np.zeros(5)
for v in reversed(chain):
    m = tr[:, 0] == v
    rows = tr[m]
    k = np.argmax(rows[:, 6])
    r = rows[k]
    cand = int(K[sigma[v]]) * math.prod(int(K[u]) for u in deps[v])
    kend = max([end[j] for j in kids[v]], default=0.0)
    seen = r[7:23:2]
    fenced = r[8:23:2]
    g = seen > 0
    if g.any():
        s_max = (seen[g].max() - t0) / 1e3
        f_max = (fenced[g].max() - t0) / 1e3
    else:
        s_max = f_max = (r[3] - t0) / 1e3
    comp, sync, e = [(x - t0) / 1e3 for x in r[4:7]]
    ph = np.array([s_max - kend, f_max - s_max, comp - f_max, sync - comp, e - sync])
    tot += ph
    print(f"{v} {K[sigma[v]]} {len(deps[v])} {cand} {int(m.sum())} | {kend:.1f} | " +
          " ".join(f"{x:.2f}" for x in ph) + f" | {int(g.sum())}")
print("chain totals: poll %.1f fence %.1f tile %.1f bar %.1f rel %.1f us" % tuple(tot))
