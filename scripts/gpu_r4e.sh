# round 2 (re-entry), call 4e: criticality threshold of the widening, 2-D tile gain threshold, wave tail (host-only), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm; do
  for rep in 1 2; do for v in base PASE_CRIT_FRAC=0.7 PASE_CRIT_FRAC=0.95 PASE_2D_GAIN=0.9 PASE_2D_GAIN=0.7 PASE_WAVE_TAIL=0; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/4e.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
