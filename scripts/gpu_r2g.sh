# round 2, call G: where the throughput-regime DP kernel spends its issue slots (ncu source
# page of dp_persistent on Transformer LE_P and of GNMT 4+4's dominant vertex)
set -x
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o /tmp/prof_le -f python scripts/profile_one.py transformer_le --solves 3 > gpurun_out/ncu_le.log 2>&1; tail -1 gpurun_out/ncu_le.log
python scripts/ncu_summary.py /tmp/prof_le.ncu-rep > gpurun_out/ncu_le.txt 2>&1
ncu -i /tmp/prof_le.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_le_source.csv 2>/dev/null; ls -la gpurun_out/ncu_le_source.csv
TOP=$(python scripts/profile_one.py gnmt4 --top)
echo "gnmt4 top vertex $TOP"
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill_vertex --launch-skip $TOP --launch-count 1 -o /tmp/prof_g4 -f python scripts/profile_one.py gnmt4 --solves 1 > gpurun_out/ncu_g4.log 2>&1; tail -1 gpurun_out/ncu_g4.log
python scripts/ncu_summary.py /tmp/prof_g4.ncu-rep > gpurun_out/ncu_g4.txt 2>&1
ncu -i /tmp/prof_g4.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_g4_source.csv 2>/dev/null; ls -la gpurun_out/ncu_g4_source.csv
python -c "
import sys; sys.path.insert(0,'.')
from paper_2407_04001_b200 import pase, zoo
g,p=zoo.bench_graph('gnmt4'); c=pase.Context(g,p,device=-1); v=c.schedule()['vinfo']; print('gnmt4 vinfo top', v[$TOP])"
