# round 2 (re-entry), call G: PASE_TRACE timelines of every zoo workload (duration-model fit)
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm alexnet transformer_le; do
  timeout 300 python scripts/trace_run.py $w > gpurun_out/trace_$w.log 2>&1; grep 'dp phase' gpurun_out/trace_$w.log
done
