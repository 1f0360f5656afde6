# GPU round: parity tests, smoke, bench, launch list, one full ncu capture of the top dp_fill.
set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
PASE_TIMING=1 timeout 300 python scripts/profile_one.py transformer --solves 3 2>&1 | tail -3
PASE_TIMING=1 timeout 300 python scripts/profile_one.py transformer --solves 3 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --workload transformer_le --steps 20 --warmup 3 --e2e-steps 3 > gpurun_out/bench_le.json 2> gpurun_out/bench_le.err; tail -3 gpurun_out/bench_le.err; cat gpurun_out/bench_le.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_one.py transformer --solves 3 > gpurun_out/ncu_launches.log 2>&1; tail -2 gpurun_out/ncu_launches.log
R=$(python scripts/profile_one.py transformer --top)
PASE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_fill --launch-skip $R --launch-count 1 -o gpurun_out/prof_top -f python scripts/profile_one.py transformer > gpurun_out/ncu_full.log 2>&1; tail -3 gpurun_out/ncu_full.log
