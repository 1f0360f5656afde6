# round 2, call T: round-based back-substitution -- parity, bench (pipelined e2e), launch list
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 --e2e-steps 30 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('solve', d['ms_per_step'], d['phases_ms'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['mode'], 'serial', d['e2e']['serial']['ms_per_step'])"
for w in inception_v3 gnmt rnnlm; do timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 10 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],3), d['phases_ms'], 'e2e', round(d['e2e']['ms_per_step'],3))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-alt > gpurun_out/ncu_launches.log 2>&1; python scripts/launches.py gpurun_out/launches.csv 2>&1 | head -12
