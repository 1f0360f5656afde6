set -x
cd $GRAFT_REPO_ROOT
for w in ${WLS:-transformer transformer_le}; do
  timeout 300 python scripts/trace_run.py $w > gpurun_out/trace_$w.log 2>&1
  grep "dp phase" gpurun_out/trace_$w.log
done
