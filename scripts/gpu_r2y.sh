# round 2, call Y: ncu of the CTA-tiled min-plus vs the default tiles (Transformer LE_P DP kernel)
set -x
cd $GRAFT_REPO_ROOT
for v in base cta; do
  envs=""; [ "$v" = "cta" ] && envs="PASE_CTA=1"
  env $envs timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 1 --launch-count 1 -o /tmp/prof_$v -f python scripts/profile_one.py transformer_le --solves 2 > gpurun_out/ncu_$v.log 2>&1; tail -1 gpurun_out/ncu_$v.log
  python scripts/ncu_summary.py /tmp/prof_$v.ncu-rep > gpurun_out/ncu_sum_$v.txt 2>&1
  python scripts/ncu_source_top.py /tmp/prof_$v.ncu-rep > gpurun_out/ncu_src_$v.txt 2>&1
done
cat gpurun_out/ncu_sum_base.txt gpurun_out/ncu_sum_cta.txt
