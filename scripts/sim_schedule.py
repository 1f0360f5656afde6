"""List-schedule simulation with MEASURED task durations from a PASE_TRACE timeline:
what makespan would a static claim order built from true durations give?
usage: python scripts/sim_schedule.py <trace.npy> <workload> [env...]"""
import heapq, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import WORKLOADS
from paper_2407_04001_b200 import pase, zoo
tr = np.load(sys.argv[1]); wl = sys.argv[2]
for kv in sys.argv[3:]:
    a, b = kv.split("="); os.environ[a] = b
key, p, policy, _ = WORKLOADS[wl]
c = pase.Context(zoo.bench_graph(key)[0], p, policy=policy, device=-1)
sigma, deps, parent = c.order(); n = len(sigma)
# trace rows are in local task-id order (vertex-major)
vt = tr[:, 0].astype(int)
dur = (tr[:, 6] - tr[:, 3]) / 1e3          # start -> end (compute + sync + release)
LAT = float(os.environ.get("SIM_LAT", "1.0"))   # dependency latency (release -> consumer sees it)
NB = 296
tasks_of = [[] for _ in range(n)]
for t, v in enumerate(vt): tasks_of[v].append(t)
kids = [[] for _ in range(n)]
for j in range(n):
    if parent[j] >= 0: kids[parent[j]].append(j)
# bottom level with measured durations
bl = [0.0] * n
for i in range(n - 1, -1, -1):
    w = sum(dur[t] for t in tasks_of[i]); lo = max(dur[t] for t in tasks_of[i])
    bl[i] = max(lo, w / NB) + LAT + (bl[parent[i]] if parent[i] >= 0 else 0)
pend = [len(sum((tasks_of[j] for j in kids[i]), [])) for i in range(n)]
ready = []; ev = []; now = 0.0; free = NB; done = 0; cur = {}
for i in range(n):
    if not kids[i]: heapq.heappush(ready, (-bl[i], i, 0.0))
end_t = 0.0
while done < len(dur):
    while free > 0 and ready:
        pr, i, rt = ready[0]
        k = cur.get(i, 0)
        t = tasks_of[i][k]
        st = max(now, rt)
        heapq.heappush(ev, (st + dur[t], i)); free -= 1
        cur[i] = k + 1
        if cur[i] == len(tasks_of[i]): heapq.heappop(ready)
    now, i = heapq.heappop(ev); free += 1; done += 1; end_t = max(end_t, now)
    pa = parent[i]
    if pa >= 0:
        pend[pa] -= 1
        if pend[pa] == 0: heapq.heappush(ready, (-bl[pa], pa, now + LAT))
print(f"{wl}: measured span {(tr[:, 6].max() - tr[:, 2].min()) / 1e3:.1f} us, total busy {dur.sum():.0f} us "
      f"(/{NB} = {dur.sum() / NB:.1f}), critical path {max(bl):.1f} us, simulated list schedule {end_t:.1f} us")
if os.environ.get("SIM_PATH"):
    own = [max(max(dur[t] for t in tasks_of[i]), sum(dur[t] for t in tasks_of[i]) / NB) + LAT for i in range(n)]
    h = [0.0] * n                                       # longest path from a leaf up to i (incl.)
    for i in range(n):                                  # children have lower ranks
        h[i] = own[i] + max((h[j] for j in kids[i]), default=0.0)
    K = c.K(); vi = c.schedule()["vinfo"]
    v = n - 1
    print(f"longest path {h[v]:.1f} us")
    while True:
        w = sum(dur[t] for t in tasks_of[v]); lo = max(dur[t] for t in tasks_of[v])
        cand = int(K[sigma[v]]) * math.prod(int(K[u]) for u in deps[v])
        print(f"  {v:4d} K {int(K[sigma[v]]):4d} cand {cand:10d} tasks {len(tasks_of[v]):4d} shape {vi[v][4]:3d} glog {vi[v][5]} wlog {vi[v][6]}  longest {lo:6.1f}  work/NB {w / NB:6.1f}")
        if not kids[v]: break
        v = max(kids[v], key=lambda j: h[j])
