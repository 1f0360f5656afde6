# round 2 (re-entry), call X: gate-related runtime knobs under the new defaults (same binary), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer gnmt rnnlm inception_v3; do
  for rep in 1 2; do for v in base PASE_WARM=0 PASE_GATE_ELECT=1 "PASE_GATE_ELECT=1 PASE_WARM=0" PASE_TASKS_PER_BLOCK=2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/x.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]'.replace(' ','_'), round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
