"""Chunk-sharded unpack of one container on the GPU engine: world 1 equals
container.unpack; world 2 (two processes, gloo verdict all-reduce; both on
cuda:0 here -- their kernels never wait on each other) reads only each rank's
byte range and split points and decodes it exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _model(dc):
    from paper_2502_15443_b200 import container
    rng = np.random.default_rng(3)
    ts, st = [], {}
    for i, (r, c) in enumerate([(512, 1024), (300, 2048), (1000, 640)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        ts.append(dc.QuantizedTensor(f"w{i}", q, 0.01, dc.ScaleVector.identity(c)))
        st[f"w{i}"] = dc.ActivationStats(f"w{i}", np.ones(c))
    data, index = container.pack_indexed(ts, st, chunk_size=1 << 18, seg_shift=8)
    payload = np.concatenate([t.qvalues.reshape(-1).view(np.uint8) for t in ts])
    return data, index.to_bytes(container.binding_of(data)), payload


def test_shard_world1_equals_unpack(cuda, tmp_path):
    from paper_2502_15443_b200 import sharded
    data, side, payload = _model(cuda)
    for idx in (None, side):
        r = sharded.unpack_shard(data, 0, 1, index=idx)
        assert np.array_equal(r.out.cpu().numpy(), payload)
    p = tmp_path / "m.dcc"
    p.write_bytes(data)
    r = sharded.unpack_shard(str(p), 0, 1, index=side)
    assert np.array_equal(r.out.cpu().numpy(), payload)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, path, side_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2502_15443_b200 import sharded
        r = sharded.unpack_shard(path, rank, world, index=side_path)
        q.put((rank, (r.shard.out0, r.shard.out1, r.out.cpu().numpy().tobytes())))
    finally:
        dist.destroy_process_group()


def test_shard_world2_gpu(cuda, tmp_path):
    data, side, payload = _model(cuda)
    p, s = tmp_path / "m.dcc", tmp_path / "m.dcc.dcidx"
    p.write_bytes(data)
    s.write_bytes(side)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, str(p), str(s))) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    (a0, a1, b0), (c0, c1, d0) = res[0], res[1]
    assert a0 == 0 and a1 == c0 and c1 == payload.size
    assert np.frombuffer(b0, np.uint8).tobytes() == payload[a0:a1].tobytes()
    assert np.frombuffer(d0, np.uint8).tobytes() == payload[c0:c1].tobytes()


def test_quantize_prune_shard_world1_equals_api(cuda, oracle):
    """world 1, the default GPU per-tensor function: the shard is the whole
    model and equals quantize_scaled + prune through the API (and the oracle)."""
    from paper_2502_15443_b200 import sharded, tensors
    from paper_2502_15443_b200.pruning import PruneConfig
    ws, st = [], {}
    for i, (r, c) in enumerate([(64, 96), (128, 64), (40, 200)]):
        w, s = tensors.synth_ensemble(tensors.SynthSpec(rows=r, cols=c, name=f"t{i}"), 300 + i)
        ws.append(w)
        st[w.name] = s
    got = sharded.quantize_prune_shard(ws, st, 0.5, PruneConfig(0.2), 0, 1)
    for g, w in zip(got, ws):
        s = oracle.compute_scale(np.asarray(st[w.name].channel_max), 0.5)
        q, wsc = oracle.quantize(w.values, s)
        q = oracle.prune(q, np.asarray(st[w.name].channel_max), 0.2, False)
        assert np.array_equal(g.qvalues, q) and g.w_scale == wsc


def _pack_model(dc):
    rng = np.random.default_rng(5)
    ts, st = [], {}
    for i, (r, c) in enumerate([(512, 1024), (300, 2048), (1000, 640), (7, 9)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        if i == 1:
            q[:100] = rng.integers(-127, 128, (100, c))  # a chunk that does not compress: stored
        ts.append(dc.QuantizedTensor(f"w{i}", q, 0.01, dc.ScaleVector.identity(c)))
        st[f"w{i}"] = dc.ActivationStats(f"w{i}", np.ones(c))
    return ts, st


def test_pack_shard_world1_equals_pack(cuda):
    from paper_2502_15443_b200 import container, sharded
    ts, st = _pack_model(cuda)
    for cs in (1 << 16, 1 << 18):
        assert sharded.pack_shard(ts, st, cs) == container.pack(ts, st, cs)


def _pack_worker(rank, world, port, q, cs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2502_15443_b200 as dc
        from paper_2502_15443_b200 import sharded
        ts, st = _pack_model(dc)
        q.put((rank, sharded.pack_shard(ts, st, cs, None, rank, world)))
    finally:
        dist.destroy_process_group()


def test_pack_shard_world2_gpu(cuda):
    """Two ranks (gloo; both on cuda:0 here) encode disjoint chunk ranges on
    the GPU; rank 0's assembled file equals single-process container.pack."""
    from paper_2502_15443_b200 import container
    ts, st = _pack_model(cuda)
    cs = 1 << 16
    want = container.pack(ts, st, cs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_pack_worker, args=(r, 2, port, q, cs)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res[1] is None
    assert res[0] == want
