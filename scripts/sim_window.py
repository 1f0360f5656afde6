"""Simulate the persistent claim order on a PASE_TRACE timeline (measured task durations):
static order (window 1) vs claiming the first READY task within a window of the order.
usage: python scripts/sim_window.py  (reads gpurun_out/trace_transformer.npy)"""
import heapq, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2407_04001_b200 import pase, zoo
tr = np.load("gpurun_out/trace_transformer.npy")
c = pase.Context(zoo.bench_graph("transformer")[0], 64, policy="exact_p", device=-1)
s = c.schedule(); order = s["order"]; tasks = s["tasks"].reshape(-1, 4)
sigma, deps, parent = c.order(); n = len(sigma)
vt = tr[:, 0].astype(int)
dur = (tr[:, 5] - tr[:, 3]) / 1e3      # start -> sync (compute) ... trace columns: vtx,smid,claim,start,comp,sync,end
rel = (tr[:, 6] - tr[:, 5]) / 1e3
LAT = 0.5
pend0 = np.zeros(n, int)
for t in range(len(vt)):
    if parent[vt[t]] >= 0: pend0[parent[vt[t]]] += 1
def run(window, claim_cost):
    pend = pend0.copy(); ready_time = np.full(n, np.inf)
    for i in range(n):
        if pend[i] == 0: ready_time[i] = 0.0
    claimed = np.zeros(len(order), bool); head = 0
    free_at = [0.0] * 296; heapq.heapify(free_at)
    done_events = []   # (time, vertex)
    finish = 0.0; nclaimed = 0
    # event-driven: each CTA becomes free at time f; picks a task
    import bisect
    pending_done = []
    while nclaimed < len(order):
        f = heapq.heappop(free_at)
        # apply completions up to f
        while pending_done and pending_done[0][0] <= f:
            tdone, v = heapq.heappop(pending_done)
            p = parent[v]
            if p >= 0:
                pend[p] -= 1
                if pend[p] == 0: ready_time[p] = tdone + LAT
        while head < len(order) and claimed[head]: head += 1
        pick = -1
        for k in range(head, min(len(order), head + window)):
            if not claimed[k] and ready_time[vt[order[k]]] <= f:
                pick = k; break
        if pick < 0:
            pick = head
        claimed[pick] = True; nclaimed += 1
        t = order[pick]; v = vt[t]
        # wait until ready (may need future completions)
        while ready_time[v] == np.inf:
            tdone, vv = heapq.heappop(pending_done)
            p = parent[vv]
            if p >= 0:
                pend[p] -= 1
                if pend[p] == 0: ready_time[p] = tdone + LAT
        start = max(f + claim_cost, ready_time[v])
        end = start + dur[t] + rel[t]
        heapq.heappush(pending_done, (end, v))
        heapq.heappush(free_at, end)
        finish = max(finish, end)
    return finish
print("measured span", (tr[:, 6].max() - tr[:, 2].min()) / 1e3)
for w, cc in [(1, 1.0), (8, 1.5), (32, 1.5), (32, 2.0), (128, 2.0)]:
    print("window", w, "claim", cc, "-> %.1f us" % run(w, cc))
