#!/usr/bin/env python
"""Benchmark of the PaSE strategy-search hot path on B200 (contract: see DESIGN.md §7).

One STEP = one complete search (pase_solve: cost tables, DP fill over the elimination
tree, back-substitution, strategy to host) of the workload named in config.workload.
  value  = DP entries/s = candidates per search (sum_i K(sigma_i)|T(i)|)
           x steps / device time of the timed steps (CUDA events on the library stream),
           graph descriptors already resident in HBM (pase_create done before timing).
  e2e    = the same metric through the public API with host inputs: pase_create (graph
           from host memory, descriptors H2D) + pase_solve (strategy D2H) + pase_destroy.
Default workload: Transformer 6+6, d_model 1024, p = 64 simulated devices, EXACT_P
(BASELINE.json configs[4], the north-star config).  L2 is flushed (256 MiB write)
before every timed step.

--impl reference runs the CPU oracle (oracle/, the reference arm of this tier) on the
host cores for the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (zoo builder key, p, policy, description)
    "transformer": ("transformer", 64, "exact_p", "Transformer 6+6 d_model 1024 (b64 s256 h16 ff4096 v32768), p=64, EXACT_P"),
    "transformer_le": ("transformer", 64, "le_p", "Transformer 6+6 d_model 1024, p=64, LE_P (prod <= p)"),
    "inception_v3": ("inception_v3", 32, "exact_p", "InceptionV3 218 vertices, b128, p=32, EXACT_P"),
    "gnmt": ("gnmt", 64, "exact_p", "GNMT unrolled 2+2 layers x 40 steps, p=64, EXACT_P"),
    "gnmt_le": ("gnmt", 64, "le_p", "GNMT unrolled 2+2 layers x 40 steps, p=64, LE_P"),
    "gnmt4": ("gnmt4", 64, "exact_p", "GNMT unrolled 4+4 layers x 40 steps, p=64, EXACT_P (M=5, 2.6e9 table entries)"),
    "stream205": ("stream205", 64, "exact_p", "SYNTHETIC streaming-regime clique (not a paper config): 14 GB child table read once, p=64, EXACT_P"),
    "rnnlm": ("rnnlm", 64, "exact_p", "RNNLM unrolled 2 layers x 40 steps, p=64, EXACT_P"),
    "alexnet": ("alexnet", 8, "exact_p", "AlexNet b128, p=8, EXACT_P"),
    "mlp": ("mlp", 4, "exact_p", "4-layer MLP b64 h256, p=4, EXACT_P"),
    "chain200": ("chain200", 4, "exact_p", "latency probe: 200-GEMM path, p=4 (not a paper config)"),
}
SM_COUNT = 148
FP64_LANES_PER_SM = 64          # fallback only: 148 SM x 64 fp64 lanes x clock


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device),
                                      "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                parts = [x.strip() for x in out.split(",")]
                if len(parts) == len(self.FIELDS):
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for s in self.samples for k in range(4) if s[2 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def fp64_peaks(sm_mhz):
    """The ALU ceilings of the DP fill, MEASURED on this pool's B200 by scripts/fp64_peak.cu
    (profiles/fp64_peak.json): DADD instructions/s of independent chains, and the DP's
    candidate step (DADD + DSETP + argmin selects on registers) per second.  Falls back to the
    unit-count derivation (148 SM x 64 fp64 lanes x clock) only if the file is missing."""
    try:
        f = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        return (f["dadd_per_s"] / 1e12, f["candidates_per_s"],
                f"measured: profiles/fp64_peak.json (scripts/fp64_peak.cu, {f['when']}, "
                f"SM {f['clocks']['sm_mhz']:.0f} MHz)")
    except Exception:
        return (SM_COUNT * FP64_LANES_PER_SM * sm_mhz * 1e6 / 1e12, None,
                f"derived (fallback): {SM_COUNT} SM x {FP64_LANES_PER_SM} fp64 lanes x {sm_mhz:.0f} MHz")


def bench_config(desc, p, policy, cand, world, flush_mb=256):
    """The `config` dict both arms print (same keys and values for the same workload and N)."""
    return {"workload": desc, "p": p, "policy": policy, "candidates": int(cand),
            "l2": f"GPU arm: L2 flushed ({flush_mb} MiB write) before every timed step; CPU arm: n/a",
            "parallelism": f"dp-table partition over {world} GPU(s)"}


def oracle_solve(graph, p, policy, threads):
    from oracle import oracle as O
    t0 = time.perf_counter()
    P = O.Problem.from_model(graph, p, O.EXACT_P if policy == "exact_p" else O.LE_P)
    r = P.dp(threads=threads)
    return time.perf_counter() - t0, r, P


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2407_04001_b200 import zoo
    key, p, policy, desc = WORKLOADS[args.workload]
    g = zoo.bench_graph(key)[0]
    threads = os.cpu_count() or 1
    from oracle import oracle as O
    cand = None
    for _ in range(args.warmup):
        dt, r, P = oracle_solve(g, p, policy, threads)
    times = []
    for _ in range(args.steps):
        dt, r, P = oracle_solve(g, p, policy, threads)
        times.append(dt)
        if cand is None:
            cand = P.table_sizes()[1]
    if cand is None:
        dt, r, P = oracle_solve(g, p, policy, threads)
        cand = P.table_sizes()[1]
    tot = sum(times)
    value = cand * len(times) / tot
    line = {
        "impl": "reference", "metric": "DP entries/s (strategy search, PaSE Eq. 4 / Fig. 5)",
        "value": value, "unit": "entries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(desc, p, policy, cand, world, args.flush_mb),
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": threads, "kind": "oracle",
                         "sample": "full workload, one complete search per step (cost tables + Fig. 5 DP)"},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# Table 1 of the paper: "Ours" search times in seconds, Python on a Xeon E5
# (SandyBridge), the paper's own (unpublished) layer dims -- context only
PAPER_TABLE1 = {
    "alexnet": {4: 0.226, 8: 0.253, 16: 0.295, 32: 0.361, 64: 0.475},
    "inception_v3": {4: 14.398, 8: 20.018, 16: 39.791, 32: 86.039, 64: 196.253},
    "rnnlm": {4: 0.057, 8: 0.086, 16: 0.069, 32: 0.131, 64: 0.215},   # paper: one 5-D LSTM vertex, not unrolled
    "transformer": {4: 9.752, 8: 28.798, 16: 130.882, 32: 553.022, 64: 1883.187},
}
SWEEP = [("mlp", "exact_p"), ("alexnet", "exact_p"), ("inception_v3", "exact_p"), ("rnnlm", "exact_p"),
         ("gnmt", "exact_p"), ("gnmt4", "exact_p"), ("transformer", "exact_p"), ("transformer", "le_p")]


def run_sweep(args):
    """every config x p in {4, 8, 16, 32, 64} on one GPU -- device DP entries/s,
    e2e search wall (create + solve + destroy from host arrays), algorithmic HBM and measured-ALU
    fractions, the oracle at N threads (full search, parity checked) and at 1 thread (full search
    when <= 1e9 candidates, else not run), and the paper's Table 1 time."""
    import torch
    from paper_2407_04001_b200 import pase, zoo
    from oracle import oracle as O
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")
    peaks = load_peaks()
    fp64_peak, cand_peak, _ = fp64_peaks(peaks.get("sm_max_mhz", 1965.0))
    hbm_peak = peaks.get("hbm_gbs", 6538.0)
    threads = os.cpu_count() or 1
    rows = []
    only = set(args.sweep_only.split(",")) if args.sweep_only else None
    for key, policy in SWEEP:
        if only and key not in only:
            continue
        for p in (4, 8, 16, 32, 64):
            g = zoo.BENCH_GRAPHS[key][0]()
            ctx = pase.Context(g, p, policy=policy, device=0, stream=stream.cuda_stream)
            for _ in range(3):
                r = ctx.solve()
            ms, dp = [], []
            for _ in range(5):
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                r = ctx.solve()
                st = ctx.stats()
                ms.append(st["ms_solve"])
                dp.append(st["ms_dp"])
            ctx.close()
            cand = int(st["candidates"])
            G = pase.Graph(g)
            e2e = []
            for i in range(4):
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                with pase.Context(G, p, policy=policy, device=0, stream=stream.cuda_stream) as c2:
                    c2.solve()
                e1.record(stream)
                e1.synchronize()
                if i:
                    e2e.append(e0.elapsed_time(e1))
            dpm = statistics.mean(dp)
            pol = O.EXACT_P if policy == "exact_p" else O.LE_P
            orN = or1 = None
            parity = None
            if cand <= 2e10:
                t0 = time.perf_counter()
                Pr = O.Problem.from_model(g, p, pol)
                o = Pr.dp(threads=threads)
                orN = time.perf_counter() - t0
                parity = bool(list(o["strategy"]) == list(r["config_index"]) and o["cost"] == r["cost"])
                if cand <= 1e9:
                    t0 = time.perf_counter()
                    Pr = O.Problem.from_model(g, p, pol)
                    Pr.dp(threads=1)
                    or1 = time.perf_counter() - t0
            row = {"config": key, "policy": policy, "p": p, "V": st["n_vertices"], "M": st["max_dep"],
                   "K": st["max_configs"], "candidates": cand, "table_entries": int(st["table_entries"]),
                   "solve_ms": statistics.mean(ms), "dp_ms": dpm, "e2e_ms": statistics.mean(e2e),
                   "dp_entries_per_s": cand / (dpm / 1e3),
                   "alg_hbm_gbs": st["alg_bytes_dp"] / (dpm / 1e3) / 1e9,
                   "alg_hbm_frac": st["alg_bytes_dp"] / (dpm / 1e3) / 1e9 / hbm_peak,
                   "alu_frac": st["dp_fp64_ops"] / (dpm / 1e3) / 1e12 / fp64_peak,
                   "cand_frac": (cand / (dpm / 1e3) / cand_peak) if cand_peak else None,
                   "oracle_1thr_s": or1, "oracle_nthr_s": orN, "oracle_threads": threads, "parity": parity,
                   "paper_s": PAPER_TABLE1.get(key, {}).get(p) if policy == "exact_p" else None}
            rows.append(row)
            print(json.dumps(row), flush=True)
    def f(x, fmt):
        return "–" if x is None else format(x, fmt)
    lines = ["| Config | p / policy | |V| | M | K max | Σ candidates | solve ms (DP ms) | e2e search ms | DP entries/s | alg. HBM GB/s (% of 6539) | ALU % (DADD) | cand. % | oracle 1-thr s | oracle N-thr s | parity | paper s |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['config']} | {r['p']} / {r['policy'].upper()} | {r['V']} | {r['M']} | {r['K']} | {r['candidates']:.3g} | "
                     f"{r['solve_ms']:.3f} ({r['dp_ms']:.3f}) | {r['e2e_ms']:.3f} | {r['dp_entries_per_s']:.3g} | "
                     f"{r['alg_hbm_gbs']:.0f} ({100 * r['alg_hbm_frac']:.1f} %) | {100 * r['alu_frac']:.1f} | "
                     f"{f(None if r['cand_frac'] is None else 100 * r['cand_frac'], '.1f')} | {f(r['oracle_1thr_s'], '.3f')} | "
                     f"{f(r['oracle_nthr_s'], '.3f')} (N={r['oracle_threads']}) | {r['parity']} | {f(r['paper_s'], '.3f')} |")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    open(os.path.join(ROOT, "gpurun_out", "sweep.md"), "w").write("\n".join(lines) + "\n")
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "sweep.json"), "w"), indent=1)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="transformer", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-threads", type=int, default=1,
                    help="host threads creating the next searches in the pipelined e2e (0: main thread only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--no-alt", action="store_true", help="skip the throughput-regime (LE_P) line")
    ap.add_argument("--sweep", action="store_true", help="BASELINE.md §4 table: every config x p on one GPU")
    ap.add_argument("--sweep-only", default="", help="comma-separated config keys for --sweep")
    args = ap.parse_args()
    if args.sweep:
        return run_sweep(args)
    args.warmup = max(args.warmup, 3)
    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2407_04001_b200 import pase, zoo
    # PASE_BENCH_SHARE_GPU=1 (functional test of the multi-process group on a 1-GPU box): every
    # rank uses cuda:0 with 1/world of its SMs (virtual_ranks) and gloo for the host plumbing;
    # the DP path is the same cross-process CUDA-IPC one, but kernels of different processes
    # time-slice on one GPU, so the timing is meaningless
    share = os.environ.get("PASE_BENCH_SHARE_GPU") == "1" and world > 1
    device = 0 if share else local_rank
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    key, p, policy, desc = WORKLOADS[args.workload]
    graph = zoo.bench_graph(key)[0]
    stream = torch.cuda.Stream()
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def make_ctx():
        # one rank per GPU; a group exchanges CUDA-IPC handles over torch.distributed, then
        # the DP kernel moves partitions over NVLink itself (pase_connect)
        c = pase.Context(graph, p, policy=policy, device=device, stream=stream.cuda_stream,
                         rank=rank, world=world, virtual_ranks=share)
        if world > 1:
            hs = [None] * world
            dist.all_gather_object(hs, c.export_handle())
            c.connect(hs)
        return c

    ctx = make_ctx()
    st0 = ctx.stats()
    cand = int(st0["candidates"])
    for _ in range(args.warmup):
        ctx.solve()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    step_ms, dp_ms, tab_ms = [], [], []
    with ClockSampler(device) as clk:
        barrier()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)                              # L2 flush outside the timed events
            # device time of the solve: CUDA events the library records on its stream right
            # before and after the solve graph (the flush kernel ahead of it keeps the GPU busy
            # while the host enqueues, so no host latency is inside the bracket; recording a
            # torch event after solve() returns would count the host round-trip instead)
            r = ctx.solve()
            s = ctx.stats()
            step_ms.append(s["ms_solve"])
            dp_ms.append(s["ms_dp"])
            tab_ms.append(s["ms_tables"])
        barrier()
        time.sleep(0.25)
    tot_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = cand * args.steps / (tot_ms / 1e3)
    st = ctx.stats()
    ctx.close()

    # the same search in its throughput regime (LE_P: prod c <= p, 33x the candidates of the
    # EXACT_P north-star config), reported beside the headline so the DP kernel's steady-state
    # rate is visible next to the latency-bound default
    alt = None
    alt_key = {"transformer": "transformer_le", "gnmt": "gnmt_le"}.get(args.workload)
    if alt_key and not args.no_alt:
        akey, ap_, apol, adesc = WORKLOADS[alt_key]
        ag = zoo.bench_graph(akey)[0]
        c3 = pase.Context(ag, ap_, policy=apol, device=device, stream=stream.cuda_stream,
                          rank=rank, world=world, virtual_ranks=share)
        if world > 1:
            hs = [None] * world
            dist.all_gather_object(hs, c3.export_handle())
            c3.connect(hs)
        for _ in range(3):
            c3.solve()
        barrier()
        a_ms, a_dp = [], []
        for _ in range(min(args.steps, 10)):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            c3.solve()
            s3 = c3.stats()
            a_ms.append(s3["ms_solve"])
            a_dp.append(s3["ms_dp"])
        barrier()
        a_tot = sum(a_ms)
        if dist is not None:
            t = torch.tensor([a_tot], dtype=torch.float64, device="cpu" if share else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a_tot = float(t.item())
        ast = c3.stats()
        c3.close()
        alt = {"workload": adesc, "value": int(ast["candidates"]) * len(a_ms) / (a_tot / 1e3), "unit": "entries/s",
               "steps": len(a_ms), "ms_per_step": a_tot / len(a_ms), "dp_fill_ms": statistics.mean(a_dp),
               "candidates": int(ast["candidates"]), "dp_fp64_ops": int(ast["dp_fp64_ops"]),
               "alg_bytes_dp": int(ast["alg_bytes_dp"]),
               "partitioned": f"{world} rank(s); multi-GPU partitions {int(ast['comm_bytes'])} B of peer stores per rank per solve",
               "comm_bytes_per_rank": int(ast["comm_bytes"])}

    # e2e through the public API with host inputs (create + solve + destroy per step): the
    # graph is held in the C ABI's input layout (pase.Graph: pase_graph node / edge arrays in
    # host memory, converted from the dict once), so each step runs pase_create from host
    # arrays (ingest, plan, H2D upload), pase_solve (strategy D2H) and pase_destroy
    c_graph = pase.Graph(graph)

    def make_ctx_host():
        c = pase.Context(c_graph, p, policy=policy, device=device, stream=stream.cuda_stream,
                         rank=rank, world=world, virtual_ranks=share)
        if world > 1:
            hs = [None] * world
            dist.all_gather_object(hs, c.export_handle())
            c.connect(hs)
        return c

    e2e_ms = []
    for i in range(args.e2e_steps + 1):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with make_ctx_host() as c2:
            c2.solve()
        e1.record(stream)
        e1.synchronize()
        if i > 0:                                   # first one warms host caches
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_tot = sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e_tot], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e_serial_value = cand * len(e2e_ms) / (e2e_tot / 1e3) if e2e_ms else None
    # pipelined e2e (one GPU): the same per-search work -- create from host arrays (plan, pinned
    # H2D upload), solve, strategy read back to the host, destroy, L2 flushed before every solve
    # -- for independent searches issued back to back through the split API: search k+1 is
    # planned and enqueued on the host (pase_create + pase_launch) while the GPU runs search k,
    # then search k is finished (its own end event, pase_finish) and destroyed
    # With --e2e-threads T > 0, T host threads run pase_create of the next searches concurrently
    # (ctypes releases the GIL; the library's process-wide caches are locked), the main thread
    # launches them in order -- a planner serving a stream of requests.  Only for workloads whose
    # contexts are small (at most 2 + T contexts are alive at once).
    e2e_pipe_ms, e2e_threads = None, 0
    if world == 1 and args.e2e_steps > 0:
        import concurrent.futures as cf
        nsteps = max(args.e2e_steps, 2)
        with make_ctx_host() as cw:
            small = int(cw.stats()["table_entries"]) * 10 < (2 << 30)   # T + A bytes
        e2e_threads = args.e2e_threads if small else 0

        def pipeline(steps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            prev = None
            with cf.ThreadPoolExecutor(max(1, e2e_threads)) as ex:
                futs = []
                for i in range(steps):
                    while e2e_threads and len(futs) < min(steps, i + 1 + e2e_threads):
                        futs.append(ex.submit(make_ctx_host))
                    c2 = futs[i].result() if e2e_threads else make_ctx_host()
                    with torch.cuda.stream(stream):
                        flush.fill_(1)
                    c2.launch()
                    if prev is not None:
                        prev.finish()
                        prev.close()
                    prev = c2
                prev.finish()
                prev.close()
            e1.record(stream)
            e1.synchronize()
            return e0.elapsed_time(e1) / steps

        # the creating thread and the launching thread hand the GIL back and forth around their
        # ctypes calls; CPython's default 5 ms switch interval lets one of them wait that long for
        # the other's Python code (measured: 1-8 ms outliers per search), so shorten it here
        sw = sys.getswitchinterval()
        sys.setswitchinterval(5e-5)
        try:
            pipeline(nsteps)                        # warm: pinned staging blocks, pool growth, threads
            runs = sorted(pipeline(nsteps) for _ in range(3))
        finally:
            sys.setswitchinterval(sw)
        e2e_pipe_ms = runs[1]                       # median of three pipelined runs
    e2e_value = cand / (e2e_pipe_ms / 1e3) if e2e_pipe_ms else e2e_serial_value

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    peaks = load_peaks()
    clocks = clk.summary()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    fp64_peak, cand_peak, peak_source = fp64_peaks(sm_mhz)                  # Tops/s, candidates/s
    mean_dp = statistics.mean(dp_ms)
    achieved = st["dp_fp64_ops"] / (mean_dp / 1e3) / 1e12
    hbm_peak = peaks.get("hbm_gbs", 6538.0)
    hbm_achieved = st["alg_bytes_dp"] / (mean_dp / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(args.workload)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        dt, r_or, P = oracle_solve(graph, p, policy, threads)
        cpu = {"value": cand / dt, "unit": "entries/s", "cores": threads, "kind": "oracle",
               "sample": f"full workload, one complete search ({dt:.2f} s: cost tables + Fig. 5 DP)",
               "parity": bool(list(r_or["strategy"]) == list(r["config_index"]) and r_or["cost"] == r["cost"])}
    if alt is not None:
        a_ach = alt["dp_fp64_ops"] / (alt["dp_fill_ms"] / 1e3) / 1e12
        alt["roofline"] = {"bound": "alu", "achieved": a_ach, "peak": fp64_peak, "unit": "TFLOP/s",
                           "frac": a_ach / fp64_peak, "peak_source": peak_source}
        if cand_peak:
            c_ach = alt["candidates"] / (alt["dp_fill_ms"] / 1e3)
            alt["roofline"]["candidate_view"] = {"achieved": c_ach, "peak": cand_peak, "unit": "candidates/s",
                                                 "frac": c_ach / cand_peak}
    line = {
        "metric": "DP entries/s (strategy search, PaSE Eq. 4 / Fig. 5)",
        "value": value, "unit": "entries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(desc, p, policy, cand, world, args.flush_mb),
        "plan": {"vertices": st["n_vertices"], "table_entries": int(st["table_entries"]), "M": st["max_dep"],
                 "K": st["max_configs"], "tree_levels": st["tree_levels"],
                 "comm_bytes_per_rank": int(st["comm_bytes"])},
        "phases_ms": {"tables": statistics.mean(tab_ms), "dp_fill": mean_dp,
                      "solve_total": statistics.mean(step_ms)},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp64_peak, "traffic": traffic,
                     "kernel": "dp_persistent (the whole DP phase is one persistent launch; timed by CUDA event nodes in the solve graph)",
                     "peak_source": peak_source,
                     "what": "algorithmic fp64 ops (per candidate: terms-1 adds + 1 compare) / DP time vs measured DADD/s",
                     "candidate_view": ({"achieved": cand / (mean_dp / 1e3), "peak": cand_peak, "unit": "candidates/s",
                                         "frac": cand / (mean_dp / 1e3) / cand_peak} if cand_peak else None),
                     "hbm_view": {"achieved_gbs": hbm_achieved, "peak_gbs": hbm_peak,
                                  "frac": hbm_achieved / hbm_peak, "alg_bytes": int(st["alg_bytes_dp"])}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "entries/s", "h2d_bytes_per_step": int(st["h2d_bytes"]),
                "d2h_bytes_per_step": int(st["d2h_bytes"]),
                "ms_per_step": e2e_pipe_ms if e2e_pipe_ms else e2e_tot / max(len(e2e_ms), 1),
                "mode": (f"pipelined: the next searches created on {e2e_threads} host thread(s) while the GPU runs search k"
                         if e2e_pipe_ms and e2e_threads else
                         "pipelined: search k+1 created and launched on the host while the GPU runs search k"
                         if e2e_pipe_ms else "serial"),
                "serial": {"value": e2e_serial_value, "ms_per_step": e2e_tot / max(len(e2e_ms), 1),
                           "what": "one search at a time: create, solve, destroy, then the next"},
                "what": "per search: pase_create (host pase_graph arrays -> plan -> pinned H2D) + solve (L2 flushed before it; D2H strategy) + pase_destroy"},
        "throughput_regime": alt,
        "gpu_launches": int(st["n_launches"]) * args.steps,
        "clocks": clocks,
        "paper_context": "PaSE Table 1 (PAPER.md:753-762): Transformer p=64 search 1883.187 s, Python on Xeon E5; dims unpublished",
    }
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
