# round 2 (re-entry), call E: gate-stamped critical chain of the north-star search
set -x
cd $GRAFT_REPO_ROOT
for w in transformer mlp; do
  timeout 300 python scripts/trace_run.py $w > gpurun_out/trace_$w.log 2>&1; head -3 gpurun_out/trace_$w.log
  python scripts/trace_gate.py $w > gpurun_out/trace_gate_$w.txt 2>&1; cat gpurun_out/trace_gate_$w.txt
done
