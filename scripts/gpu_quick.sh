set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
PASE_TIMING=1 timeout 300 python scripts/trace_run.py transformer 2>&1 | tail -60
timeout 300 python scripts/trace_run.py chain200 2>&1 | grep -E 'dp phase|iter 3'
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
