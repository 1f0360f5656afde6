# round 2 (re-entry), call F: critical-chain task-shaping knobs (interleaved, DP ms)
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm; do
  for v in base PASE_WIDEN_MINC=4 PASE_WIDEN_MINC=2 PASE_LATENCY_CAND=2097152 PASE_WARM=0 PASE_TASKS_PER_BLOCK=8 base PASE_WIDEN_MINC=4 PASE_WIDEN_MINC=2 PASE_LATENCY_CAND=2097152 PASE_WARM=0 PASE_TASKS_PER_BLOCK=8; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/f.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
