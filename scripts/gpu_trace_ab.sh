cd $GRAFT_REPO_ROOT
for w in ${WLS:-transformer}; do
  timeout 300 python scripts/trace_run.py $w > gpurun_out/trace_$w.log 2>&1; grep "dp phase" gpurun_out/trace_$w.log
  cp gpurun_out/trace_$w.npy gpurun_out/trace_${w}_0.npy
  env $VAR timeout 300 python scripts/trace_run.py $w > gpurun_out/trace_${w}_1.log 2>&1; grep "dp phase" gpurun_out/trace_${w}_1.log
  cp gpurun_out/trace_$w.npy gpurun_out/trace_${w}_1.npy
done
