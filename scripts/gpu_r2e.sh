# round 2, call E: TMA stream tile A/B + ncu, full GPU tests, BASELINE §4 sweep, bench line
set -x
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -1
  PASE_STREAM_TMA=0 timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -1
done
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_tma.csv python scripts/run_workload.py stream205 --solves 2 > gpurun_out/stream_launches_tma.log 2>&1; tail -1 gpurun_out/stream_launches_tma.log
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip 1 --launch-count 1 -o /tmp/prof_stream_tma -f python scripts/run_workload.py stream205 --solves 1 > gpurun_out/ncu_stream_tma.log 2>&1; tail -1 gpurun_out/ncu_stream_tma.log
python scripts/ncu_summary.py /tmp/prof_stream_tma.ncu-rep > gpurun_out/ncu_stream_tma.txt 2>&1
ncu -i /tmp/prof_stream_tma.ncu-rep --page raw --csv > gpurun_out/ncu_stream_tma_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 1800 python bench.py --sweep > gpurun_out/sweep.log 2>&1; tail -2 gpurun_out/sweep.log
PASE_TIMING=1 timeout 300 python scripts/e2e_probe.py transformer > gpurun_out/e2e_probe.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
