# round 2, call J: tile-threshold sweep (2-D single-suffix threshold, latency-mode threshold)
set -x
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm transformer_le gnmt_le; do
  steps=30; case $w in *_le) steps=6;; esac
  for v in "base" "PASE_MIN_2S=262144" "PASE_MIN_2S=1048576" "PASE_MIN_2S=4194304" "PASE_MIN_2S=1048576 PASE_LATENCY_CAND=65536" "PASE_MIN_2S=1048576 PASE_LATENCY_CAND=131072" "base"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-alt 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3))"
  done
done
