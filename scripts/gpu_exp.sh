set -x
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_base.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_t_base.npy
PASE_SMALL_MODE=g32 PASE_SMALL_CAND=2000000 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_g32.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_t_g32.npy
PASE_SMALL_MODE=generic PASE_SMALL_CAND=2000000 timeout 300 python scripts/trace_run.py transformer > gpurun_out/trace_gen.log 2>&1; cp gpurun_out/trace_transformer.npy gpurun_out/trace_t_gen.npy
grep "dp phase" gpurun_out/trace_base.log gpurun_out/trace_g32.log gpurun_out/trace_gen.log
