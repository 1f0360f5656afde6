# Round measurement sweep: every workload (bench.py line each), the chain latency probe,
# the launch list and one full ncu capture of the dominant kernel, clocks.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/bench_all.jsonl
for w in transformer transformer_le gnmt gnmt_le inception_v3 rnnlm alexnet mlp chain200; do
  steps=100; [ $w = transformer_le ] && steps=20; [ $w = gnmt_le ] && steps=20
  timeout 900 python bench.py --workload $w --steps $steps --warmup 5 --e2e-steps 5 >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err
done
wc -l gpurun_out/bench_all.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; tail -2 gpurun_out/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o gpurun_out/prof_dp -f python scripts/profile_one.py transformer --solves 3 > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o gpurun_out/prof_dp_le -f python scripts/profile_one.py transformer_le --solves 3 > gpurun_out/ncu_full_le.log 2>&1; tail -2 gpurun_out/ncu_full_le.log
