# round 2 (re-entry): shipped build check (define on the command line, as the measured pad-16 build)
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 rnnlm; do
  timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/4k.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
done
