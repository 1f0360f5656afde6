# round 2, call AA: small-K widening (PASE_SMALLK_MINC) A/B
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le gnmt4; do
  steps=30; case $w in *_le|gnmt4) steps=6;; esac
  for v in base PASE_SMALLK_MINC=2 PASE_SMALLK_MINC=4 base PASE_SMALLK_MINC=2 PASE_SMALLK_MINC=4; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
PASE_SMALLK_MINC=2 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
