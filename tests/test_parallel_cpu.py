"""Multi-process (gloo, world_size 2) and layout tests of the sharding / TP
logic, on CPU.  The GPU kernels are replaced by exact int64 matmuls; the
sharding, K-alignment and the all-reduce composition are what is tested."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_15443_b200 import parallel


def test_shard_ranges_cover_and_balance():
    rng = np.random.default_rng(0)
    for n, world in ((1, 1), (7, 2), (150, 8), (9600, 4), (3, 8)):
        w = rng.integers(1, 100, n)
        rs = parallel.shard_ranges(w, world)
        assert len(rs) == world and rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        loads = [w[a:b].sum() for a, b in rs]
        if n >= 8 * world:
            assert max(loads) <= w.sum() / world + w.max()


@pytest.mark.parametrize("model,world", [("llama-13b", 8), ("opt-1.3b", 2), ("opt-2.7b", 4)])
def test_tp_layout_partitions_every_linear(model, world):
    per_rank = [parallel.tp_layout(model, world, r, layers=1) for r in range(world)]
    for shards in zip(*per_rank):
        s0 = shards[0]
        if s0.kind == "col":
            assert [s.r0 for s in shards][0] == 0 and shards[-1].r1 == s0.rows
            assert all(a.r1 == b.r0 for a, b in zip(shards, shards[1:]))
        else:
            assert shards[0].c0 == 0 and shards[-1].c1 == s0.cols
            assert all(a.c1 == b.c0 for a, b in zip(shards, shards[1:]))
            assert all(s.c0 % parallel.K_ALIGN == 0 for s in shards)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        model = "llama-13b"
        shards = parallel.tp_layout(model, world, rank, layers=1)
        ok = True
        for s in shards:
            if s.rows * s.cols > 30_000_000:
                continue
            W = torch.randint(-127, 128, (s.rows, s.cols), generator=g, dtype=torch.int8)
            X = torch.randint(-127, 128, (3, s.cols), generator=g, dtype=torch.int8)
            full = X.long() @ W.long().T
            part = X[:, s.c0:s.c1].long() @ W[s.r0:s.r1, s.c0:s.c1].long().T
            acc = part.to(torch.int32).clone()
            if s.kind == "row":
                parallel.allreduce_partials([acc])
                ok &= torch.equal(acc.long(), full)
            else:
                outs = [torch.zeros((3, b - a), dtype=torch.int32)
                        for a, b in (parallel._split(s.rows, world)[r] for r in range(world))]
                dist.all_gather(outs, acc)
                ok &= torch.equal(torch.cat(outs, 1).long(), full)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_tp_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
