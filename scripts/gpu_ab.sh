# A/B of env knobs on the DP phase: for each workload, each variant in $VARIANTS
# (";"-separated env assignments, "base" = none), prints ms_per_step and phases.
cd $GRAFT_REPO_ROOT
WLS=${WLS:-"transformer transformer_le"}
IFS=';' read -ra VS <<< "${VARIANTS:-base;PASE_NO_2D=1}"
for w in $WLS; do
  steps=30; case $w in *_le) steps=8;; esac
  for v in "${VS[@]}"; do
    envs=""; [ "$v" != "base" ] && envs="$v"
    env $envs timeout 600 python bench.py --workload $w --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 2>>gpurun_out/ab.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '[$v]', round(d['ms_per_step'],3), 'dp', round(d['phases_ms']['dp_fill'],3), 'frac', round(d['roofline']['frac'],3))"
  done
done
