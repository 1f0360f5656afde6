# round 2 (re-entry), call N: list schedule from MEASURED per-task durations (PASE_DUR_FILE, from a
# PASE_TRACE timeline of the same plan; two refinement passes) vs the model, DP ms
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm; do
  timeout 300 python scripts/trace_run.py $w > /dev/null 2>&1; python scripts/trace_durations.py $w /tmp/dur1_$w.bin
  PASE_DUR_FILE=/tmp/dur1_$w.bin timeout 300 python scripts/trace_run.py $w > /dev/null 2>&1; python scripts/trace_durations.py $w /tmp/dur2_$w.bin
  for v in base PASE_DUR_FILE=/tmp/dur1_$w.bin PASE_DUR_FILE=/tmp/dur2_$w.bin base PASE_DUR_FILE=/tmp/dur1_$w.bin PASE_DUR_FILE=/tmp/dur2_$w.bin; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/n.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
