"""Per-vertex busy time (sum of task durations) of two PASE_TRACE timelines of one workload
(scripts/gpu_ab_trace.sh outputs 0 and 1), with the plan of each variant recomputed here.
usage: python scripts/ab_compare.py <workload> "<env of variant 0>" "<env of variant 1>" """
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

wl = sys.argv[1]
key, p, policy, _ = WORKLOADS[wl]
g = zoo.bench_graph(key)[0]
res = {}
for k, envs in enumerate(sys.argv[2:4]):
    for e in ("PASE_NO_2D", "PASE_C_PER_LANE", "PASE_WIDE_WAVES", "PASE_SPREAD", "PASE_SPREAD_TASKS", "PASE_WAVE_TAIL"):
        os.environ.pop(e, None)
    for kv in envs.split():
        a, b = kv.split("=")
        os.environ[a] = b
    # knobs are read once per process by the library: plan each variant in a subprocess
    import subprocess
    out = subprocess.run([sys.executable, "-c", f"""
import sys; sys.path.insert(0, {os.getcwd()!r})
import numpy as np
from paper_2407_04001_b200 import pase, zoo
from bench import WORKLOADS
key, p, policy, _ = WORKLOADS[{wl!r}]
c = pase.Context(zoo.bench_graph(key)[0], p, policy=policy, device=-1)
np.save('/tmp/vinfo_{k}.npy', c.schedule()['vinfo'])
"""], env=dict(os.environ), capture_output=True, text=True)
    if out.returncode:
        print(out.stderr)
    v = np.load(f"/tmp/vinfo_{k}.npy")
    tr = np.load(f"gpurun_out/trace_{wl}_{k}.npy")
    res[k] = (v, tr)
ctx = pase.Context(g, p, policy=policy, device=-1)
K = ctx.K()
sigma, deps, parent = ctx.order()
rows = []
for i in range(len(sigma)):
    cand = int(K[sigma[i]]) * math.prod(int(K[u]) for u in deps[i])
    b = []
    for k in (0, 1):
        v, tr = res[k]
        m = tr[:, 0] == i
        b.append(((tr[m, 6] - tr[m, 3]).sum() / 1e3, int(v[i, 4]), int(v[i, 5]), int(m.sum())))
    rows.append((b[0][0] - b[1][0], i, cand, b[0], b[1]))
rows.sort()
print("total busy [0] %.0f us  [1] %.0f us" % (sum(r[3][0] for r in rows), sum(r[4][0] for r in rows)))
for r in rows[-10:] + rows[:6]:
    print(r[1], "K", int(K[sigma[r[1]]]), "cand %.3g" % r[2], "| [0] busy %.0f shape %d glog %d tasks %d" % r[3],
          "| [1] busy %.0f shape %d glog %d tasks %d" % r[4],
          "| rate %.0f vs %.0f cand/us" % (r[2] / max(r[3][0], 1e-9), r[2] / max(r[4][0], 1e-9)))
