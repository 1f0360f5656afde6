# round 2, call H: stream prefetch lookahead A/B; GPU tests
set -x
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for a in 0 1 2 3; do
  PASE_STREAM_PF_AHEAD=$a timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stream205 persistent ahead=$a', round(d['best_dp_ms'],3), 'ms DP')"
done; done
for a in 0 1 2; do
  PASE_STREAM_PF_AHEAD=$a PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_a$a.csv python scripts/run_workload.py stream205 --solves 2 > /dev/null 2>&1
done
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
