# round 2 (re-entry), call U: per-shape gate acquire (PASE_GATE_LDACQ=1: ld.acquire at the gates of
# 1-D tiles, fence elsewhere; =2: ld.acquire everywhere) vs fence (default), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer gnmt rnnlm inception_v3 transformer_le alexnet; do
  steps=40; case $w in *_le) steps=8;; esac
  for rep in 1 2 3; do for v in base PASE_GATE_LDACQ=1 PASE_GATE_LDACQ=2; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/u.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
PASE_GATE_LDACQ=1 PYTHONPATH=$GRAFT_REPO_ROOT timeout 900 python tests/parity_variant_main.py mlp,alexnet,inception_v3,transformer,gnmt,rnnlm 12 2>&1 | tail -1
