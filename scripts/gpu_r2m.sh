# round 2, call M: cost-table chunk size A/B (build variants), trace with the early gate
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt; do
  for lib in base rows128 rows256 base; do
    envs=""; [ "$lib" != "base" ] && envs="PASE_LIB=paper_2407_04001_b200/libpase_$lib.so"
    env $envs timeout 600 python bench.py --workload $w --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$lib]', round(d['ms_per_step'],3), 'tables', round(d['phases_ms']['tables'],4), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1
timeout 300 python scripts/trace_chain.py transformer > gpurun_out/trace_chain_transformer.log 2>&1; head -2 gpurun_out/trace_chain_transformer.log; tail -1 gpurun_out/trace_chain_transformer.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-alt > gpurun_out/ncu_launches.log 2>&1; tail -1 gpurun_out/ncu_launches.log
