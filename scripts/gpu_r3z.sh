# round 2 (re-entry), call Z: tile / task-shaping knobs under the final defaults (same binary), DP ms
cd $GRAFT_REPO_ROOT
for w in transformer gnmt rnnlm inception_v3; do
  for rep in 1 2; do for v in base PASE_C_PER_LANE=24 PASE_C_PER_LANE=48 PASE_LATENCY_CAND=524288 PASE_MIN_2S=2097152 PASE_MIN_2S=8388608 PASE_SMALLK_MINC=4 PASE_TAIL_MINC=4 PASE_TAIL_MINC=16; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/z.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done; done
done
