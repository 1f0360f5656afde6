# round 2 (re-entry), call 4g: lane-group sizing on the throughput configs (host-only knobs), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer_le gnmt_le gnmt4; do
  steps=8; case $w in gnmt4) steps=4;; esac
  for rep in 1 2; do for v in base PASE_C_PER_LANE=16 PASE_C_PER_LANE=64 PASE_2S_MAXG=4 PASE_2S_MAXG=3 PASE_MIN_2S=1048576; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/4g.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
