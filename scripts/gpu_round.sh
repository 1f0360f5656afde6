# quick GPU round: parity tests, bench (EXACT_P default + LE_P), per-task trace of the default
set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --workload transformer_le --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_le.json 2> gpurun_out/bench_le.err; tail -3 gpurun_out/bench_le.err; cat gpurun_out/bench_le.json
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_transformer.log 2>&1; tail -5 gpurun_out/trace_transformer.log
