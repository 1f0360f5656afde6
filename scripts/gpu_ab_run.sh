set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_eq1.py -m gpu -x -q 2>&1 | tail -15
WLS="transformer transformer_le gnmt gnmt_le inception_v3 rnnlm" VARIANTS="base;PASE_SPREAD=0" bash scripts/gpu_ab.sh
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
