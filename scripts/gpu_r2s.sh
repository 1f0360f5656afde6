# round 2, call S: critical-path dynamic vertices with widened lane groups (PASE_DYN=2); e2e anatomy
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le gnmt4; do
  steps=30; case $w in *_le|gnmt4) steps=6;; esac
  for v in base PASE_DYN=2 "PASE_DYN=2 PASE_DYN_MIN=0.1" "PASE_DYN=2 PASE_DYN_MINC=2" "PASE_DYN=2 PASE_DYN_MINC=8" base PASE_DYN=2 "PASE_DYN=2 PASE_DYN_MIN=0.1" "PASE_DYN=2 PASE_DYN_MINC=2" "PASE_DYN=2 PASE_DYN_MINC=8"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
PASE_DYN=2 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_dyn2.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_dyn2.npy
PASE_DYN=2 PASE_DYN_MIN=0.01 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 600 python scripts/e2e_probe2.py transformer 2>&1 | tail -8
timeout 600 python bench.py --steps 50 --warmup 5 --e2e-steps 30 --no-cpu-baseline --no-alt > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print('solve', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], d['e2e']['mode'], 'serial', d['e2e']['serial']['ms_per_step'])"
