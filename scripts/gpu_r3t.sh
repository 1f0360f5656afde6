# round 2 (re-entry), call T: ld.acquire gate (libpase_ldacq.so) vs fence, second box, 4 interleaved reps
cd $GRAFT_REPO_ROOT
for w in transformer gnmt rnnlm inception_v3 transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for rep in 1 2 3 4; do for v in base PASE_LIB=paper_2407_04001_b200/libpase_ldacq.so; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/t.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
