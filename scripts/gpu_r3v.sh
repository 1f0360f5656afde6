# round 2 (re-entry), call V: new default (ld.acquire gates) vs the fence (PASE_GATE_LDACQ=0) and
# red.release releases (PASE_REL_RED=1), same binary, DP ms; parity suite; default bench line
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for w in transformer gnmt rnnlm inception_v3 transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for rep in 1 2 3; do for v in base PASE_GATE_LDACQ=0 PASE_REL_RED=1; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/v.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
PASE_REL_RED=1 PYTHONPATH=$GRAFT_REPO_ROOT timeout 900 python tests/parity_variant_main.py mlp,alexnet,inception_v3,transformer 8 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('BENCH', d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['e2e']['serial']['ms_per_step'], d['throughput_regime']['dp_fill_ms'], d['cpu_baseline']['parity'])"
