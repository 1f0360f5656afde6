# round 2, call V: back-substitution v4 -- parity + solve phases on every workload
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=30; case $w in *_le) steps=6;; esac
  timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; print('$w', round(d['ms_per_step'],4), 'dp', round(p['dp_fill'],4), 'tables', round(p['tables'],4), 'rest', round(d['ms_per_step']-p['dp_fill']-p['tables'],4))"
done
