# round 2, call K: knobs around the new tile threshold; trace of the new critical chain
set -x
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1
timeout 300 python scripts/trace_chain.py transformer > gpurun_out/trace_chain_transformer.log 2>&1; head -3 gpurun_out/trace_chain_transformer.log; tail -1 gpurun_out/trace_chain_transformer.log
for w in transformer inception_v3 transformer_le; do
  steps=30; case $w in *_le) steps=6;; esac
  for v in "base" "PASE_C_PER_LANE=24" "PASE_C_PER_LANE=48" "PASE_2S_WIDE=0" "PASE_2S_MAXG=4" "PASE_WAVE_TAIL=0" "PASE_WIDEN=0" "PASE_LATENCY_CAND=196608" "base"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
