"""Multi-GPU host logic on CPU: two processes with the gloo backend
each build their rank's schedule (host-only planning contexts, no device) and check, after
exchanging them, that the partition covers every DP entry exactly once, that replicated
tables are computed by every rank, that broadcast flags and pending counters agree with
their definition, and that the claim order is a permutation."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

WORKLOADS = [("transformer", 64, "exact_p", 1 << 16), ("inception_v3", 32, "exact_p", 1 << 12),
             ("gnmt", 64, "exact_p", 1 << 16), ("mlp", 4, "exact_p", 0)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2407_04001_b200 import pase, zoo
        out = {}
        for name, p, pol, thr in WORKLOADS:
            g, _ = zoo.bench_graph(name)
            ctx = pase.Context(g, p, policy=pol, device=-1, rank=rank, world=world, redundant_below=thr)
            sch = ctx.schedule()
            sigma, deps, parent = ctx.order()
            K = ctx.K()
            mine = {"vinfo": sch["vinfo"], "tasks": sch["tasks"], "order": sch["order"],
                    "K": K, "deps": deps, "parent": parent, "sigma": sigma}
            allr = [None] * world
            dist.all_gather_object(allr, mine)
            out[name] = allr
        if rank == 0:
            q.put(("ok", out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e)))


def zoo_graph(name):
    from paper_2407_04001_b200 import zoo
    return zoo.bench_graph(name)


def _units(K, deps_i):
    n = 1
    for u in deps_i:
        n *= int(K[u])
    return n


@pytest.mark.parametrize("world", [2])
def test_two_rank_partition_plan(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    status, res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
    assert status == "ok", res
    any_part = False
    for name, ranks in res.items():
        r0 = ranks[0]
        n = len(r0["sigma"])
        # identical plan on every rank
        for r in ranks[1:]:
            assert np.array_equal(r["sigma"], r0["sigma"])
            assert np.array_equal(r["vinfo"][:, :2], r0["vinfo"][:, :2])       # part, bcast
        for i in range(n):
            part, bcast = int(r0["vinfo"][i, 0]), int(r0["vinfo"][i, 1])
            any_part |= bool(part)
            # coverage of units (items of the tiled kernel, or outputs): per rank intervals
            ivs = []
            for rk, r in enumerate(ranks):
                t = r["tasks"][r["tasks"][:, 0] == i]
                assert int(r["vinfo"][i, 2]) == len(t)
                assert (t[:, 3] >= 0).all()                    # plain or wave-tail tasks
                ivs.append(sorted((int(a), int(b)) for _, a, b, _ in t))
            if not part:
                assert all(iv == ivs[0] for iv in ivs)            # replicated: same full cover
                cover = ivs[0]
                assert cover[0][0] == 0
                for (a, b), (c, d) in zip(cover, cover[1:]):
                    assert b == c                                  # contiguous
            else:
                merged = sorted(x for iv in ivs for x in iv)
                for (a, b), (c, d) in zip(merged, merged[1:]):
                    assert b <= c                                  # disjoint across ranks
                assert merged[0][0] == 0
                assert bcast & 2                                   # argmin always broadcast
            # broadcast-T flag: partitioned and the parent does not share its top coordinate
            par = int(r0["parent"][i])
            if part:
                top = r0["deps"][i][-1]
                aligned = par >= 0 and bool(r0["vinfo"][par, 0]) and r0["deps"][par][-1] in r0["deps"][i]
                assert bool(bcast & 1) == (not aligned)
        # pending counters: children's tasks each rank waits for (plus, with PASE_COST_TASKS=1, the cost-table chunks
        # the vertex reads (its L, and W of the edges it pays: 64-row chunks of the later
        # endpoint's configs), which every rank computes itself
        g, _ = zoo_graph(name)
        rank_of = {int(v): i for i, v in enumerate(r0["sigma"])}
        chunks_of = [1] * n
        for ed in g["edges"]:
            a, b = rank_of[ed["src"]], rank_of[ed["dst"]]
            late = ed["src"] if a > b else ed["dst"]
            chunks_of[min(a, b)] += -(-int(r0["K"][late]) // 64)
        if os.environ.get("PASE_COST_TASKS") != "1":
            chunks_of = [0] * n
        for rk, r in enumerate(ranks):
            assert int((r["tasks"][:, 0] < 0).sum()) == sum(chunks_of)
            for p_ in range(n):
                kids = [j for j in range(n) if int(r0["parent"][j]) == p_]
                want = chunks_of[p_]
                for j in kids:
                    if int(r0["vinfo"][j, 1]) & 1:
                        want += sum(int(x["vinfo"][j, 2]) for x in ranks)
                    else:
                        want += int(r["vinfo"][j, 2])
                assert int(r["vinfo"][p_, 3]) == want, (name, rk, p_)
            assert sorted(r["order"].tolist()) == list(range(len(r["tasks"])))
    assert any_part
