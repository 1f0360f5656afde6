set -x
cd $GRAFT_REPO_ROOT
R=$(python scripts/profile_one.py transformer --top)
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill --launch-skip $R --launch-count 1 -o gpurun_out/prof_top -f python scripts/profile_one.py transformer > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
PASE_SCHEDULE=launches PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill --launch-skip 180 --launch-count 1 -o gpurun_out/prof_180 -f python scripts/profile_one.py transformer > gpurun_out/ncu_full2.log 2>&1; tail -3 gpurun_out/ncu_full2.log
