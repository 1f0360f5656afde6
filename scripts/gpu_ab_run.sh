set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
WLS="${WLS:-transformer transformer_le gnmt gnmt_le inception_v3 rnnlm}" VARIANTS="${VARIANTS:-base}" bash scripts/gpu_ab.sh
