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


# ------------------------------------------------- sharded unpack (C3, N GPUs)
def _oracle_decode(image, loc, body, seg_shift):
    """Test decoder: the oracle restatement decodes this rank's chunks
    (the GPU engine's role); same (out, status, crc) contract."""
    from oracle import oracle as O
    from paper_2502_15443_b200 import native as nv
    outs, status, crcs = [], [], []
    for e in loc:
        blob = image[int(e["file_offset"]):int(e["file_offset"] + e["comp_len"])].tobytes()
        n = int(e["uncomp_len"])
        st, raw = nv.CHUNK_OK, np.zeros(n, np.uint8)
        if e["codec"] == 0:
            raw = np.frombuffer(blob, np.uint8).copy()
        else:
            try:
                raw = np.frombuffer(O.decompress_blob(blob, n), np.uint8).copy()
            except O.OracleError as x:
                st = {"TruncatedError": nv.CHUNK_TRUNC_TABLE}.get(x.kind, nv.CHUNK_CORRUPT)
                if "frequency table" in x.msg:
                    st = nv.CHUNK_BAD_TABLE
                elif "out of range" in x.msg:
                    st = nv.CHUNK_STATE_RANGE
        outs.append(raw)
        status.append(st)
        crcs.append(O.crc32(raw))
    return np.concatenate(outs), np.array(status, np.int32), np.array(crcs, np.uint32)


def _model_bytes(seed=0):
    from oracle import oracle as O
    rng = np.random.default_rng(seed)
    ents = []
    for i, (r, c) in enumerate([(300, 700), (128, 1024), (77, 513), (256, 600)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        ents.append((f"w{i}", q, 0.01, 0.5, np.ones(c), np.ones(c)))
    n = -(-sum(e[1].size for e in ents) // 16384)
    mask = np.array([i % 5 != 3 for i in range(n)])  # a few stored chunks
    data = O.pack(ents, 16384, mask=mask)
    return data, np.concatenate([e[1].reshape(-1).view(np.uint8) for e in ents])


def _outcome(fn):
    try:
        return ("ok", fn())
    except Exception as e:  # noqa: BLE001
        return (type(e).__name__, str(e))


def _sharded_worker(rank, world, port, q, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_15443_b200 import container, sharded
        data, payload = _model_bytes()
        ent = container._parse(data)[2]
        res = {}
        r = sharded.unpack_shard(path, rank, world, decode=_oracle_decode)
        res["exact"] = bool(np.array_equal(r.out, payload[r.shard.out0:r.shard.out1]))
        res["range"] = (r.shard.c0, r.shard.c1)
        # damage: a corrupt ANS stream on the last rank, a prologue error and a
        # stored-chunk bit flip (CRC) on the first: every rank must raise the
        # reference's first error (prologue before corrupt before checksum)
        ans = [i for i in range(len(ent)) if ent["codec"][i] == 1]
        store = [i for i in range(len(ent)) if ent["codec"][i] == 0]
        cases = {}
        b = bytearray(data)
        last = ans[-1]
        b[int(ent["file_offset"][last]) + 400] ^= 0x20
        cases["corrupt_last"] = bytes(b)
        b2 = bytearray(cases["corrupt_last"])
        b2[int(ent["file_offset"][ans[0]]) + 384] = 0  # start state -> out of range (prologue)
        b2[int(ent["file_offset"][ans[0]]) + 387] = 0
        cases["prologue_first_and_corrupt_last"] = bytes(b2)
        b3 = bytearray(data)
        b3[int(ent["file_offset"][store[-1]]) + 10] ^= 1
        cases["crc_store"] = bytes(b3)
        for k, v in cases.items():
            res[k] = _outcome(lambda: sharded.unpack_shard(v, rank, world, decode=_oracle_decode) and None)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_unpack_gloo_world2(tmp_path):
    """One container, two ranks: each reads and decodes only its chunk range;
    the union is the payload; verdicts agree with the single-process unpack
    (oracle) on every rank."""
    from oracle import oracle as O
    from paper_2502_15443_b200 import container, sharded
    data, _ = _model_bytes()
    path = tmp_path / "m.dcc"
    path.write_bytes(data)
    ent = container._parse(data)[2]
    plan = sharded.plan_shards(ent, 2)
    assert plan[0].c0 == 0 and plan[0].c1 == plan[1].c0 and plan[1].c1 == len(ent)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, str(path))) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[0]["exact"] and res[1]["exact"]
    assert res[0]["range"][1] == res[1]["range"][0]
    # expected verdicts: the oracle's single-process unpack of the same bytes
    data2, _ = _model_bytes()
    for k in ("corrupt_last", "prologue_first_and_corrupt_last", "crc_store"):
        assert res[0][k] == res[1][k], k
        assert res[0][k][0] != "ok", k
    ans = [i for i in range(len(ent)) if ent["codec"][i] == 1]
    assert res[0]["corrupt_last"] == ("CorruptStreamError", f"corrupt stream (chunk {ans[-1]})")
    assert res[0]["prologue_first_and_corrupt_last"][0] == "CorruptStreamError"
    assert f"chunk {ans[0]})" in res[0]["prologue_first_and_corrupt_last"][1]
    assert res[0]["crc_store"][0] == "ChecksumError"
    # the oracle agrees on which chunk fails first
    b = bytearray(data2)
    b[int(ent["file_offset"][ans[-1]]) + 400] ^= 0x20
    try:
        O.unpack(bytes(b))
        raise AssertionError("oracle accepted a corrupt stream")
    except O.OracleError as e:
        assert e.chunk == ans[-1] or f"chunk {ans[-1]}" in e.msg


def _oracle_qp(w, st, alpha, cfg):
    from oracle import oracle as O
    from paper_2502_15443_b200.pruning import PruneScope
    from paper_2502_15443_b200.scaling import QuantizedTensor, ScaleVector
    s = O.compute_scale(np.asarray(st.channel_max), alpha)
    q, ws = O.quantize(w.values, s)
    if cfg is not None and cfg.sparsity > 0:
        q = O.prune(q, np.asarray(st.channel_max), cfg.sparsity, cfg.scope is PruneScope.PER_ROW)
    return QuantizedTensor(w.name, q, ws, ScaleVector(alpha, s))


def _qp_model():
    from paper_2502_15443_b200 import tensors
    ws, st = [], {}
    for i, (r, c) in enumerate([(64, 96), (128, 64), (40, 200), (96, 96), (17, 33)]):
        w, s = tensors.synth_ensemble(tensors.SynthSpec(rows=r, cols=c, name=f"t{i}"), 100 + i)
        ws.append(w)
        st[w.name] = s
    return ws, st


def _qp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_15443_b200 import sharded
        from paper_2502_15443_b200.pruning import PruneConfig
        ws, st = _qp_model()
        out = sharded.quantize_prune_shard(ws, st, 0.5, PruneConfig(0.2), rank, world, fn=_oracle_qp)
        q.put((rank, [(t.name, t.qvalues.copy(), t.w_scale, t.scale_vec.s.copy()) for t in out]))
    finally:
        dist.destroy_process_group()


def test_quantize_prune_sharded_by_tensor_gloo_world2():
    """Quantize + prune sharded by tensor over two ranks (no data-path
    collective; one all-gather so every rank holds the whole model): every
    rank's gathered tensors equal the single-process result, in model order."""
    from paper_2502_15443_b200 import sharded
    from paper_2502_15443_b200.pruning import PruneConfig
    ws, st = _qp_model()
    want = [_oracle_qp(w, st[w.name], 0.5, PruneConfig(0.2)) for w in ws]
    plan = sharded.plan_tensor_shards([w.values.size for w in ws], 2)
    assert plan[0][0] == 0 and plan[0][1] == plan[1][0] and plan[1][1] == len(ws)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_qp_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        got = res[r]
        assert [g[0] for g in got] == [t.name for t in want]
        for (name, qv, wsc, s), t in zip(got, want):
            assert np.array_equal(qv, t.qvalues) and wsc == t.w_scale and np.array_equal(s, t.scale_vec.s), name


def _oracle_encode(raw, cs, mask):
    """The reference's per-chunk codec choice (container.py:160-171) with the
    oracle's encoder, in pack_shard's encode() shape."""
    from oracle import oracle as O
    codec, clen, crc, parts = [], [], [], []
    for i in range(-(-raw.size // cs)):
        ch = raw[i * cs:(i + 1) * cs]
        blob = O.compress_blob(ch) if mask[i] else None
        data = blob if blob is not None and len(blob) < ch.size else ch.tobytes()
        codec.append(1 if data is blob else 0)
        clen.append(len(data))
        crc.append(O.crc32(ch))
        parts.append(data)
    return (np.array(codec, np.uint8), np.array(clen, np.uint64), np.array(crc, np.uint32),
            np.frombuffer(b"".join(parts), np.uint8))


def _pack_model():
    from paper_2502_15443_b200.scaling import QuantizedTensor, ScaleVector
    from paper_2502_15443_b200.tensors import ActivationStats
    rng = np.random.default_rng(3)
    ts, st, ents = [], {}, []
    for i, (r, c) in enumerate([(300, 700), (128, 1024), (77, 513), (256, 600)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        s = rng.uniform(0.5, 2.0, c)
        cm = rng.uniform(0.1, 3.0, c).astype(np.float32)
        ts.append(QuantizedTensor(f"w{i}", q, 0.01 * (i + 1), ScaleVector(0.5, s)))
        st[f"w{i}"] = ActivationStats(f"w{i}", cm)
        ents.append((f"w{i}", q, 0.01 * (i + 1), 0.5, s, cm))
    return ts, st, ents


def _pack_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_15443_b200 import sharded
        ts, st, _ = _pack_model()
        n = -(-sum(t.qvalues.size for t in ts) // 16384)
        mask = np.array([i % 5 != 3 for i in range(n)])  # some chunks stored by plan
        out = sharded.pack_shard(ts, st, 16384, mask, rank, world, encode=_oracle_encode)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_pack_sharded_by_chunk_gloo_world2():
    """container.pack with the chunks encoded on two ranks (each only its
    contiguous chunk range), blobs sent to rank 0: byte-identical to the
    single-process pack of the same tensors (the oracle's, which equals the
    reference's); rank 1 returns None."""
    from oracle import oracle as O
    _, _, ents = _pack_model()
    n = -(-sum(e[1].size for e in ents) // 16384)
    mask = np.array([i % 5 != 3 for i in range(n)])
    want = O.pack(ents, 16384, mask=mask)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pack_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[1] is None
    assert res[0] == want
