set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "zoo_exact_p or random_synthetic" 2>&1 | tail -2
timeout 300 python scripts/trace_run.py transformer 2>&1 | grep -E "dp phase"
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 3 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('EXACT', d['ms_per_step'], d['phases_ms'], d['value'])"
timeout 600 python bench.py --workload transformer_le --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LE', d['ms_per_step'], d['phases_ms'], d['value'])"
timeout 600 python bench.py --workload gnmt_le --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('GNMT_LE', d['ms_per_step'], d['phases_ms'], d['value'])"
