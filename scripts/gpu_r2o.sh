# round 2, call O: bounded warm pass, elected gate poller, tasks per block; per-warp gate stamps
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=30; case $w in *_le) steps=6;; esac
  for v in base PASE_WARM=0 PASE_GATE_ELECT=1 PASE_TASKS_PER_BLOCK=2 base PASE_WARM=0 PASE_GATE_ELECT=1 PASE_TASKS_PER_BLOCK=2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_base.npy
PASE_GATE_ELECT=1 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_elect.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_elect.npy
PASE_WARM=0 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_nowarm.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_nowarm.npy
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
PASE_GATE_ELECT=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
