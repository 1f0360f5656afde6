# round 2 (re-entry), call 4h: code-placement pads 8 / 16 / 24 / 32, DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for rep in 1 2; do for v in PASE_LIB=paper_2407_04001_b200/libpase_pad16.so PASE_LIB=paper_2407_04001_b200/libpase_pad8.so PASE_LIB=paper_2407_04001_b200/libpase_pad32.so; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/4i.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
