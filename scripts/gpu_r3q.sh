# round 2 (re-entry), call Q: escape claims v2 (peek overlapped with the order claim) (PASE_ESCAPE=1): parity, A/B, gate-stamped chain
cd $GRAFT_REPO_ROOT
PASE_ESCAPE=1 PYTHONPATH=$GRAFT_REPO_ROOT timeout 900 python tests/parity_variant_main.py mlp,alexnet,inception_v3,transformer,gnmt,rnnlm 12 2>&1 | tail -3
for w in transformer inception_v3 gnmt rnnlm transformer_le; do
  steps=40; case $w in *_le) steps=8;; esac
  for v in base "PASE_ESCAPE=1 PASE_ESC_MAXT=2" "PASE_ESCAPE=1 PASE_ESC_MAXT=4" "PASE_ESCAPE=1 PASE_ESC_MAXT=32" base "PASE_ESCAPE=1 PASE_ESC_MAXT=2" "PASE_ESCAPE=1 PASE_ESC_MAXT=4" "PASE_ESCAPE=1 PASE_ESC_MAXT=32"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/p.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
PASE_ESCAPE=1 PASE_ESC_MAXT=4 timeout 300 python scripts/trace_run.py transformer > /dev/null 2>&1; python scripts/trace_gate.py transformer > gpurun_out/trace_gate_escape.txt; tail -1 gpurun_out/trace_gate_escape.txt
