# round 2 (re-entry): bench N = 2 path (two processes sharing the one GPU; functional check only)
cd $GRAFT_REPO_ROOT
PASE_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo rc $?; tail -c 600 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
