# round 2, call P: dynamic vertices (PASE_DYN), claim-ahead (PASE_CLAIM_AHEAD) -- A/B and parity
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le gnmt4; do
  steps=30; case $w in *_le|gnmt4) steps=6;; esac
  for v in base PASE_DYN=1 "PASE_DYN=1 PASE_DYN_MIN=0.2" PASE_CLAIM_AHEAD=1 base PASE_DYN=1 "PASE_DYN=1 PASE_DYN_MIN=0.2" PASE_CLAIM_AHEAD=1; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
PASE_DYN=1 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_dyn.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_dyn.npy
PASE_DYN=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -3
PASE_DYN=1 PASE_DYN_MIN=0.01 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
PASE_CLAIM_AHEAD=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
