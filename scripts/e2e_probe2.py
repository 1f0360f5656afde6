"""Host-side anatomy of the pipelined e2e loop (bench.py): per step, python wall of create /
launch / finish / close, with 0 or T host threads creating ahead."""
import concurrent.futures as cf
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2407_04001_b200 import pase, zoo  # noqa: E402

torch.cuda.init()
stream = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
w = sys.argv[1] if len(sys.argv) > 1 else "transformer"
key, p, policy, _ = WORKLOADS[w]
G = pase.Graph(zoo.bench_graph(key)[0])
mk = lambda: pase.Context(G, p, policy=policy, device=0, stream=stream.cuda_stream)
for c in [mk() for _ in range(3)]:
    c.solve(); c.close()
for threads in (0, 1, 2, 3):
    for rep in range(2):
        n = 40
        tc, tl, tf, tx = [], [], [], []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prev = None
        with cf.ThreadPoolExecutor(max(1, threads)) as ex:
            futs = []
            for i in range(n):
                a = time.perf_counter()
                while threads and len(futs) < min(n, i + 1 + threads):
                    futs.append(ex.submit(mk))
                c = futs[i].result() if threads else mk()
                b = time.perf_counter()
                with torch.cuda.stream(stream):
                    flush.fill_(1)
                c.launch()
                d = time.perf_counter()
                if prev is not None:
                    prev.finish()
                    e = time.perf_counter()
                    prev.close()
                    f = time.perf_counter()
                    tf.append(e - d); tx.append(f - e)
                prev = c
                tc.append(b - a); tl.append(d - b)
            prev.finish(); prev.close()
        torch.cuda.synchronize()
        tot = time.perf_counter() - t0
        ms = lambda v: f"{1e3 * statistics.median(v):.3f}"
        print(f"{w} threads {threads}: {1e3 * tot / n:.3f} ms/step | create(wait) {ms(tc)} launch {ms(tl)} "
              f"finish {ms(tf)} close {ms(tx)}", flush=True)
