"""Build and run scripts/fp64_peak.cu on the GPU box with nvidia-smi clocks sampled during
the run; writes gpurun_out/fp64_peak.json (commit it as profiles/fp64_peak.json)."""
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402

exe = "/tmp/fp64_peak"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                       "--fmad=false", os.path.join(HERE, "fp64_peak.cu"), "-o", exe])
with ClockSampler(0) as clk:
    time.sleep(0.3)
    out = subprocess.check_output([exe], text=True)
    time.sleep(0.3)
r = json.loads(out)
r["clocks"] = clk.summary()
r["what"] = ("k_dadd: 8 independent __dadd_rn chains per thread, 148x8 CTAs x 256 threads; "
             "k_cand: the DP candidate step (DADD + DSETP + argmin selects) on registers, 16 "
             "candidates per C; best of 6 timed runs (CUDA events)")
r["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(r, open(os.path.join(ROOT, "gpurun_out", "fp64_peak.json"), "w"), indent=1)
print(json.dumps(r))
