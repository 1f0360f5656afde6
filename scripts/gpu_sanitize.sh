# compute-sanitizer over the hot path: memcheck, racecheck (shared-memory hazards),
# synccheck (barrier misuse), initcheck; logs to gpurun_out/sanitize_*.log
cd $GRAFT_REPO_ROOT
export PASE_SPIN_TIMEOUT_MS=60000 PASE_NO_GRAPH=1
for tool in memcheck racecheck synccheck initcheck; do
  for c in mlp alexnet random inception_v3 group2; do
    echo "== $tool $c" >> gpurun_out/sanitize_$tool.log
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_case.py $c >> gpurun_out/sanitize_$tool.log 2>&1
    echo "== exit $?" >> gpurun_out/sanitize_$tool.log
  done
done
grep -h "== \|ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize case ok" gpurun_out/sanitize_*.log
