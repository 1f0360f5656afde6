# round 2 (re-entry), call 4b: latency-mode values of C per lane (PASE_LAT_CPL; host-only, same kernel binary), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm; do
  for rep in 1 2; do for v in base PASE_LAT_CPL=1 PASE_LAT_CPL=4 PASE_LAT_CPL=8; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/4b.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
PASE_LAT_CPL=4 PYTHONPATH=$GRAFT_REPO_ROOT timeout 900 python tests/parity_variant_main.py mlp,alexnet,inception_v3,transformer 8 2>&1 | tail -1
