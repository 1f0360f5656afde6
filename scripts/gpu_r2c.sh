# round 2, call C: streaming / one-lane tile forms -- parity and the streaming clique's ncu
set -x
cd $GRAFT_REPO_ROOT
timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -1
PASE_SCHEDULE=launches timeout 600 python scripts/run_workload.py stream205 --solves 3 2>&1 | tail -1
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches.csv python scripts/run_workload.py stream205 --solves 2 > gpurun_out/stream_launches.log 2>&1; tail -1 gpurun_out/stream_launches.log
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip 0 --launch-count 2 -o /tmp/prof_stream -f python scripts/run_workload.py stream205 --solves 1 > gpurun_out/ncu_stream.log 2>&1; tail -1 gpurun_out/ncu_stream.log
python scripts/ncu_summary.py /tmp/prof_stream.ncu-rep > gpurun_out/ncu_stream.txt 2>&1
ncu -i /tmp/prof_stream.ncu-rep --page raw --csv > gpurun_out/ncu_stream_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
