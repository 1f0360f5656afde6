# round 2, call X: CTA-tiled min-plus (PASE_CTA=1) -- parity, A/B
set -x
cd $GRAFT_REPO_ROOT
PASE_CTA=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for w in transformer transformer_le gnmt4 stream205; do
  steps=30; case $w in *_le|gnmt4|stream205) steps=6;; esac
  for v in base PASE_CTA=1 base PASE_CTA=1; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
PASE_CTA=1 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_cta.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_cta.npy; tail -1 gpurun_out/trace_cta.log
