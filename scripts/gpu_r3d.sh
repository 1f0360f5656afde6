# round 2 (re-entry), call D: L2 flush vs none on the latency-bound configs; e2e in the default
# bench command (with the LE_P line ahead of it) twice, create timings of the second
set -x
cd $GRAFT_REPO_ROOT
for w in mlp alexnet transformer; do
  for f in 256 0 256 0; do
    timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-alt --flush-mb $f 2>>gpurun_out/d.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w flush=$f', round(d['ms_per_step'],4), 'tables', round(d['phases_ms']['tables'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
for k in 1 2; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>>gpurun_out/d.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('default', round(d['ms_per_step'],3), 'pipe', round(e['ms_per_step'],3), 'serial', round(e['serial']['ms_per_step'],3))"
done
PASE_TIMING=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/d_timing.json 2> gpurun_out/d_timing.err; python -c "import json; d=json.load(open('gpurun_out/d_timing.json')); e=d['e2e']; print('timed', e['ms_per_step'], e['serial']['ms_per_step'])"
