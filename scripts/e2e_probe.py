"""Break the end-to-end call (marshal -> pase_create -> pase_solve -> pase_destroy) into its
parts, per workload (run with PASE_TIMING=1 for the library's own create breakdown)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

torch.cuda.init()
stream = torch.cuda.Stream()
for w in sys.argv[1:] or ["transformer", "gnmt", "rnnlm", "alexnet"]:
    key, p, policy, _ = WORKLOADS[w]
    g = zoo.bench_graph(key)[0]
    for it in range(4):
        t0 = time.perf_counter()
        pase.marshal_graph(g)
        t1 = time.perf_counter()
        c = pase.Context(g, p, policy=policy, device=0, stream=stream.cuda_stream)
        t2 = time.perf_counter()
        c.solve()
        t3 = time.perf_counter()
        c.solve()
        t4 = time.perf_counter()
        c.solve()
        t5 = time.perf_counter()
        c.close()
        t6 = time.perf_counter()
        ms = lambda a, b: f"{(b - a) * 1e3:7.3f}"
        print(f"{w:14s} it{it} marshal {ms(t0, t1)} create(+marshal) {ms(t1, t2)} solve1 {ms(t2, t3)} "
              f"solve2(capture) {ms(t3, t4)} solve3(graph) {ms(t4, t5)} destroy {ms(t5, t6)}", flush=True)
