# round 2 (re-entry), call M: speculative back-substitution (default) vs one lookup per level
# (libpase_nospec.so); "rest" = solve - tables - DP (back-substitution + graph gaps), ms
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_report.py -x -q 2>&1 | tail -2
for w in transformer gnmt rnnlm inception_v3 gnmt4; do
  steps=40; case $w in gnmt4) steps=5;; esac
  for v in base PASE_LIB=paper_2407_04001_b200/libpase_nospec.so base PASE_LIB=paper_2407_04001_b200/libpase_nospec.so; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/m.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['phases_ms']; print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(p['dp_fill'],4), 'rest', round(p['solve_total']-p['tables']-p['dp_fill'],4))"
  done
done
