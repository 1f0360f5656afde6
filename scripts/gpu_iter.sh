# one build->measure iteration: GPU parity, transformer trace, short benches
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1; grep "dp phase" gpurun_out/trace_transformer.log
for w in transformer chain200 gnmt; do
timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 3 2>> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"
done
for w in ${EXTRA:-}; do
timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 2>> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, 'frac', round(d['roofline']['frac'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],2))"
done
