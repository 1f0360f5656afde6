# round 2, call I: critical-chain trace of the north-star search (static order) + knob sweep
set -x
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1; tail -3 gpurun_out/trace_transformer.log
timeout 300 python scripts/trace_chain.py transformer > gpurun_out/trace_chain_transformer.log 2>&1; head -70 gpurun_out/trace_chain_transformer.log
for v in "base" "PASE_C_PER_LANE=16" "PASE_C_PER_LANE=64" "PASE_LATENCY_CAND=1048576" "PASE_LATENCY_CAND=65536" "PASE_MIN_2S=1048576" "PASE_WIDEN=0"; do
  envs=""; [ "$v" != "base" ] && envs="$v"
  env $envs timeout 600 python bench.py --workload transformer --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('transformer', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
done
