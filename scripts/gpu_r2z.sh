# round 2, call Z: source-level ncu of the CTA tile (Transformer LE_P)
set -x
cd $GRAFT_REPO_ROOT
PASE_CTA=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dp_persistent --launch-skip 1 --launch-count 1 -o /tmp/prof_cta -f python scripts/profile_one.py transformer_le --solves 2 > gpurun_out/ncu_cta.log 2>&1; tail -1 gpurun_out/ncu_cta.log
ncu -i /tmp/prof_cta.ncu-rep --page source --csv --print-source sass > /tmp/ncu_cta_source.csv 2>/dev/null; python scripts/ncu_source_top.py /tmp/ncu_cta_source.csv 70 > gpurun_out/ncu_cta_source_top.txt 2>&1
head -90 gpurun_out/ncu_cta_source_top.txt
