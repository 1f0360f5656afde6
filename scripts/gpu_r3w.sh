# Round 2 (re-entry) final evidence + BASELINE §4 sweep: gpu tests, smoke, bench (default line incl. the LE_P throughput regime), the
# reference arm, the ncu launch list of the bench command, full ncu captures of the DP kernel
# (both regimes) and the cost-table kernel, summarised on the box (reports are too big to ship).
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-alt > gpurun_out/ncu_launches.log 2>&1; tail -1 gpurun_out/ncu_launches.log
for w in transformer transformer_le; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o /tmp/prof_dp_$w -f python scripts/profile_one.py $w --solves 3 > gpurun_out/ncu_full_$w.log 2>&1; tail -1 gpurun_out/ncu_full_$w.log
  python scripts/ncu_summary.py /tmp/prof_dp_$w.ncu-rep > gpurun_out/ncu_dp_$w.txt 2>&1
  ncu -i /tmp/prof_dp_$w.ncu-rep --page raw --csv > gpurun_out/ncu_dp_${w}_raw.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cost_tables --launch-skip 2 --launch-count 1 -o /tmp/prof_cost -f python scripts/profile_one.py transformer --solves 3 > gpurun_out/ncu_cost.log 2>&1; tail -1 gpurun_out/ncu_cost.log
python scripts/ncu_summary.py /tmp/prof_cost.ncu-rep > gpurun_out/ncu_cost.txt 2>&1
du -sh gpurun_out
ncu -i /tmp/prof_cost.ncu-rep --page raw --csv > gpurun_out/ncu_cost_raw.csv 2>/dev/null
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; head -20 gpurun_out/launches_summary.txt
timeout 3000 python bench.py --sweep > gpurun_out/sweep.log 2>&1; tail -3 gpurun_out/sweep.log; wc -l gpurun_out/sweep.md
