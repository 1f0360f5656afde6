# round 2, call U: back-substitution rounds (warp per slice), inlined cost tables, item order A/B
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-alt > gpurun_out/ncu_launches.log 2>&1; python scripts/launches.py gpurun_out/launches.csv 2>&1 | head -6
for w in transformer inception_v3 gnmt rnnlm transformer_le gnmt4; do
  steps=30; case $w in *_le|gnmt4) steps=6;; esac
  for v in base PASE_TILE_FAST=1 PASE_TILE_FAST=2 base PASE_TILE_FAST=1 PASE_TILE_FAST=2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3), 'tables', round(d['phases_ms']['tables'],4))"
  done
done
PASE_TILE_FAST=2 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 100 --warmup 5 --e2e-steps 30 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('solve', d['ms_per_step'], d['phases_ms'], 'e2e', d['e2e']['ms_per_step'], 'serial', d['e2e']['serial']['ms_per_step'])"
