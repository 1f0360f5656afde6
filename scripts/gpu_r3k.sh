# round 2 (re-entry), call K: pipelined e2e with 1 / 2 / 3 creating host threads (median of 3 runs each)
cd $GRAFT_REPO_ROOT
nproc
for rep in 1 2; do for t in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 20 --e2e-threads $t --no-alt 2>>gpurun_out/k.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('threads=$t', round(d['ms_per_step'],3), 'pipe', round(e['ms_per_step'],3), 'serial', round(e['serial']['ms_per_step'],3))"
done; done
