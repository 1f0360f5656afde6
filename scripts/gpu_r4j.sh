# round 2 (re-entry), FINAL evidence on the shipped build: smoke, GPU suite, bench, reference arm,
# launch list, ncu full of dp_persistent (EXACT_P, LE_P) and cost tables, sweep
set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('BENCH', d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['e2e']['serial']['ms_per_step'], d['throughput_regime']['dp_fill_ms'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-alt > gpurun_out/ncu_launches.log 2>&1
python scripts/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; cat gpurun_out/launches_summary.txt
for w in transformer transformer_le; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 2 --launch-count 1 -o /tmp/prof_dp_$w -f python scripts/profile_one.py $w --solves 3 > gpurun_out/ncu_full_$w.log 2>&1
  python scripts/ncu_summary.py /tmp/prof_dp_$w.ncu-rep > gpurun_out/ncu_dp_$w.txt 2>&1
  ncu -i /tmp/prof_dp_$w.ncu-rep --page raw --csv > gpurun_out/ncu_dp_${w}_raw.csv 2>/dev/null
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cost_tables --launch-skip 2 --launch-count 1 -o /tmp/prof_cost -f python scripts/profile_one.py transformer --solves 3 > gpurun_out/ncu_cost.log 2>&1
python scripts/ncu_summary.py /tmp/prof_cost.ncu-rep > gpurun_out/ncu_cost.txt 2>&1
timeout 3000 python bench.py --sweep > gpurun_out/sweep.log 2>&1; wc -l gpurun_out/sweep.md
