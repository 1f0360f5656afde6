# round 2, call F: ready-queue vs static claim order (interleaved A/B), traces, parity
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q 2>&1 | tail -4
for rep in 1 2; do
  for w in transformer transformer_le gnmt gnmt4 inception_v3 rnnlm stream205; do
    steps=30; case $w in *_le|gnmt4|stream205) steps=8;; esac
    for q in 1 0; do
      PASE_QUEUE=$q timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', 'queue=$q', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
    done
  done
done
PASE_TIMING=1 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1; tail -30 gpurun_out/trace_transformer.log
