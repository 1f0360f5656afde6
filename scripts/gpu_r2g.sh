# round 2, call G: where the throughput-regime DP kernel spends its issue slots (ncu source
# page of dp_persistent on Transformer LE_P and of GNMT 4+4's dominant vertex)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o /tmp/prof_le -f python scripts/profile_one.py transformer_le --solves 3 > gpurun_out/ncu_le.log 2>&1; tail -1 gpurun_out/ncu_le.log
python scripts/ncu_summary.py /tmp/prof_le.ncu-rep > gpurun_out/ncu_le.txt 2>&1
ncu -i /tmp/prof_le.ncu-rep --page source --csv --print-source sass > /tmp/ncu_le_source.csv 2>/dev/null; python scripts/ncu_source_top.py /tmp/ncu_le_source.csv 60 > gpurun_out/ncu_le_source_top.txt 2>&1
TOP=$(python scripts/profile_one.py gnmt4 --top)
echo "gnmt4 top vertex $TOP"
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip $TOP --launch-count 1 -o /tmp/prof_g4 -f python scripts/profile_one.py gnmt4 --solves 1 > gpurun_out/ncu_g4.log 2>&1; tail -1 gpurun_out/ncu_g4.log
python scripts/ncu_summary.py /tmp/prof_g4.ncu-rep > gpurun_out/ncu_g4.txt 2>&1
ncu -i /tmp/prof_g4.ncu-rep --page source --csv --print-source sass > /tmp/ncu_g4_source.csv 2>/dev/null; python scripts/ncu_source_top.py /tmp/ncu_g4_source.csv 60 > gpurun_out/ncu_g4_source_top.txt 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2407_04001_b200 import pase, zoo
g,p=zoo.bench_graph('gnmt4'); c=pase.Context(g,p,device=-1); v=c.schedule()['vinfo']; print('gnmt4 vinfo top', v[$TOP])"

# stream A/B: the three streaming-vertex forms, persistent and per-vertex launches, interleaved
for rep in 1 2; do for m in 2 0 1; do
  PASE_STREAM_TMA=$m timeout 600 python scripts/run_workload.py stream205 --solves 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stream205 persistent mode=$m', round(d['best_dp_ms'],3), 'ms DP')"
done; done
for m in 2 0 1; do
  PASE_STREAM_TMA=$m PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/stream_launches_m$m.csv python scripts/run_workload.py stream205 --solves 2 > /dev/null 2>&1
done
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip 1 --launch-count 1 -o /tmp/prof_stream_pf -f python scripts/run_workload.py stream205 --solves 1 > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_stream_pf.ncu-rep > gpurun_out/ncu_stream_pf.txt 2>&1
