# round 2 (re-entry), call Y: tasks per CTA of big vertices (PASE_TASKS_PER_BLOCK 4 default vs 2 / 3), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer transformer_le gnmt4 alexnet; do
  steps=40; case $w in *_le) steps=8;; gnmt4) steps=4;; esac
  for rep in 1 2; do for v in base PASE_TASKS_PER_BLOCK=2 PASE_TASKS_PER_BLOCK=3; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/y.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
