"""Multi-PROCESS group check on one GPU (functional test of the cross-process CUDA-IPC path of
pase_connect): run under torchrun with N ranks; every rank uses cuda:0 with 1/N of
the SMs (virtual_ranks) and gloo for the handle exchange.  Each rank's strategy and total must
equal a single-GPU solve bit for bit.  Kernels of different processes time-slice on one GPU,
so no timing is meaningful here."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2407_04001_b200 import pase, zoo  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
ok = True
for name, thr in (("transformer", 1 << 16), ("inception_v3", 1 << 12), ("gnmt", 1 << 16)):
    g, p = zoo.bench_graph(name)
    ref = pase.Context(g, p, device=0).solve() if rank == 0 else None
    ctx = pase.Context(g, p, device=0, rank=rank, world=world, virtual_ranks=True, redundant_below=thr)
    hs = [None] * world
    dist.all_gather_object(hs, ctx.export_handle())
    ctx.connect(hs)
    dist.barrier()
    for rep in range(2):
        r = ctx.solve()
    sch = ctx.schedule()
    parts = int(sch["vinfo"][:, 0].sum())
    res = [None] * world
    dist.all_gather_object(res, (list(map(int, r["config_index"])), float(r["cost"]), parts))
    if rank == 0:
        for q, (ci, cost, np_) in enumerate(res):
            same = ci == list(map(int, ref["config_index"])) and \
                np.float64(cost).view(np.uint64) == np.float64(ref["cost"]).view(np.uint64)
            ok &= same
            print(f"{name}: rank {q} strategy+cost identical to 1-GPU: {same} ({np_} partitioned tables)", flush=True)
    dist.barrier()
    ctx.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
