# round 2 (re-entry), call C: (1) L2 flush vs none on the latency-bound configs (cold code /
# descriptor misses?), (2) e2e pipelined vs serial with host threads 0/1 and PASE_TIMING
set -x
cd $GRAFT_REPO_ROOT
for w in mlp alexnet transformer; do
  for f in 256 0 256 0; do
    timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-alt --flush-mb $f 2>>gpurun_out/c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w flush=$f', round(d['ms_per_step'],4), 'tables', round(d['phases_ms']['tables'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
for t in 0 1 0 1; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 10 --e2e-threads $t --no-alt 2>>gpurun_out/c.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('e2e threads=$t', round(d['ms_per_step'],3), 'pipe', round(e['ms_per_step'],3), 'serial', round(e['serial']['ms_per_step'],3))"
done
PASE_TIMING=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 4 --e2e-threads 1 --no-alt > /dev/null 2> gpurun_out/c_timing.err; tail -40 gpurun_out/c_timing.err
