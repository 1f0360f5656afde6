# round 2 (re-entry), call H: list-schedule duration model fitted to the PASE_TRACE timelines
# (PASE_DUR family:a_us:rate) vs the single-constant model; interleaved, DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for v in base PASE_DUR=1:3.4:2500,2:4:9000,3:3.3:3500,4:5:8500 PASE_DUR=4:4.5:8000 PASE_DUR=2:4:9000,4:4.5:8000 PASE_DUR=1:3.4:2500,2:4:6000,3:3.3:3500,4:4:6000; do
  for rep in 1 2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/h.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
