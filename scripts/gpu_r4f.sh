# round 2 (re-entry), final: smoke, full GPU suite, default bench line, reference arm, sweep
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('BENCH', d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'], d['e2e']['serial']['ms_per_step'], d['throughput_regime']['dp_fill_ms'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
timeout 3000 python bench.py --sweep > gpurun_out/sweep.log 2>&1; wc -l gpurun_out/sweep.md
