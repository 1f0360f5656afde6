# round 2 (re-entry), call J: task-length cap (PASE_MAX_LANE_CAND) A/B, interleaved, DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for v in base PASE_MAX_LANE_CAND=256 PASE_MAX_LANE_CAND=160 PASE_MAX_LANE_CAND=96 base PASE_MAX_LANE_CAND=256 PASE_MAX_LANE_CAND=160 PASE_MAX_LANE_CAND=96; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/j.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
PASE_MAX_LANE_CAND=160 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_cap.log 2>&1; python scripts/trace_gate.py transformer | tail -1
