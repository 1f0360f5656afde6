# round 2, call B: the big workloads (GNMT 4+4, streaming clique): timings, per-vertex launch
# list, ncu on the streaming vertices
set -x
cd $GRAFT_REPO_ROOT
free -g | head -2; nproc; lscpu | grep -E "Model name|Socket|Core|Thread" 
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 600 python scripts/run_workload.py gnmt4 --solves 5 2>&1 | tail -2
timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -2
PASE_SCHEDULE=launches timeout 600 python scripts/run_workload.py stream205 --solves 3 2>&1 | tail -2
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches.csv python scripts/run_workload.py stream205 --solves 2 > gpurun_out/stream_launches.log 2>&1; tail -1 gpurun_out/stream_launches.log
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip 0 --launch-count 2 -o /tmp/prof_stream -f python scripts/run_workload.py stream205 --solves 1 > gpurun_out/ncu_stream.log 2>&1; tail -1 gpurun_out/ncu_stream.log
python scripts/ncu_summary.py /tmp/prof_stream.ncu-rep > gpurun_out/ncu_stream.txt 2>&1
ncu -i /tmp/prof_stream.ncu-rep --page raw --csv > gpurun_out/ncu_stream_raw.csv 2>/dev/null
FREE_GB=$(free -g | awk '/Mem:/{print $7}')
if [ "$FREE_GB" -gt 100 ]; then timeout 900 python scripts/run_workload.py gnmt4 --solves 2 --oracle-threads $(nproc) 2>&1 | tail -2; else echo "skip oracle: $FREE_GB GB free"; fi
