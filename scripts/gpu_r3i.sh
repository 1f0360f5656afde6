# round 2 (re-entry), call I: per-warp gate acquire by ld.acquire (libpase_ldacq.so) vs fence.acq_rel
cd $GRAFT_REPO_ROOT
for w in transformer inception_v3 gnmt rnnlm mlp; do
  for v in base PASE_LIB=paper_2407_04001_b200/libpase_ldacq.so base PASE_LIB=paper_2407_04001_b200/libpase_ldacq.so; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 300 python bench.py --workload $w --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-alt 2>>gpurun_out/i.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],4), 'dp', round(d['phases_ms']['dp_fill'],4))"
  done
done
PASE_LIB=paper_2407_04001_b200/libpase_ldacq.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
