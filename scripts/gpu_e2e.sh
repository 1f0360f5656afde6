set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
PASE_TIMING=1 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -40
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 10 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('EXACT', d['ms_per_step'], d['phases_ms'], d['e2e'])"
timeout 600 python bench.py --workload rnnlm --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 10 2>> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RNNLM', d['ms_per_step'], d['phases_ms'], d['e2e'])"
