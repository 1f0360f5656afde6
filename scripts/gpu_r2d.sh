set -x
cd $GRAFT_REPO_ROOT
bash scripts/gpu_sanitize.sh
PASE_TIMING=1 timeout 300 python scripts/e2e_probe.py transformer 2>&1 | tail -24
timeout 600 python bench.py --steps 50 --warmup 5 --no-alt > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
