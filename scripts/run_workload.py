"""Solve one bench workload a few times and print timings / stats (GPU experiments)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--solves", type=int, default=5)
ap.add_argument("--oracle-threads", type=int, default=0, help="also run the oracle (strategy/cost parity)")
a = ap.parse_args()
key, p, policy, desc = WORKLOADS[a.workload]
g = zoo.bench_graph(key)[0]
t0 = time.perf_counter()
ctx = pase.Context(g, p, policy=policy, device=0)
t1 = time.perf_counter()
ms = []
for _ in range(a.solves):
    r = ctx.solve()
    s = ctx.stats()
    ms.append((s["ms_solve"], s["ms_tables"], s["ms_dp"]))
st = ctx.stats()
out = {"workload": a.workload, "create_s": t1 - t0, "solves_ms": ms, "cost": r["cost"],
       "candidates": st["candidates"], "table_entries": st["table_entries"], "alg_bytes_dp": st["alg_bytes_dp"],
       "M": st["max_dep"], "K": st["max_configs"], "levels": st["tree_levels"]}
best_dp = min(x[2] for x in ms)
out["best_dp_ms"] = best_dp
out["cand_per_s"] = st["candidates"] / (best_dp / 1e3)
out["alg_gbs"] = st["alg_bytes_dp"] / (best_dp / 1e3) / 1e9
if a.oracle_threads:
    from oracle import oracle as O
    t2 = time.perf_counter()
    P = O.Problem.from_model(g, p, O.EXACT_P if policy == "exact_p" else O.LE_P)
    o = P.dp(threads=a.oracle_threads)
    out["oracle_s"] = time.perf_counter() - t2
    out["oracle_threads"] = a.oracle_threads
    out["parity"] = bool(list(o["strategy"]) == list(r["config_index"]) and o["cost"] == r["cost"])
print(json.dumps(out))
