# round 2 (re-entry), call O: MORE pessimistic big-task durations in the list schedule (PASE_DUR), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for v in base PASE_DUR=4:3:2000 PASE_DUR=4:3:1500 PASE_DUR=4:3:1000 PASE_DUR=2:3:2000,4:3:2000 PASE_DUR=2:3:2000,3:3:2000,4:3:2000; do
  for rep in 1 2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/o.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
