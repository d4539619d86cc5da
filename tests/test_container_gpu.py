"""GPU parity of DCC1 pack/unpack: bit-exact container bytes against the
reference's golden files / digests, split-point decode == exact decode,
reference error classes and chunk indices on corrupted inputs."""

import hashlib
import struct

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def small_model(dc, seed=0, rows=64, cols=96):
    rng = np.random.default_rng(seed)
    tensors, stats = [], {}
    for i, name in enumerate(("alpha", "beta", "gamma")):
        q = rng.integers(-30, 31, (rows + i, cols)).astype(np.int8)
        sv = dc.ScaleVector(0.5, np.exp(rng.normal(0, 0.2, cols)))
        tensors.append(dc.QuantizedTensor(name, q, float(rng.uniform(0.001, 0.1)), sv))
        stats[name] = dc.ActivationStats(name, np.abs(rng.normal(0, 1, cols)))
    return tensors, stats


@pytest.mark.parametrize("bs", [0, 1, 2, 5])
def test_pack_bit_exact_vs_reference(cuda, golden, bs):
    tensors, stats = small_model(cuda)
    n = -(-sum(t.qvalues.size for t in tensors) // 4096)
    plan = cuda.CompressionPlan.block_plan(4096, n, bs)
    blob = cuda.pack(tensors, stats, chunk_size=4096, plan=plan)
    assert hashlib.sha256(blob).hexdigest() == golden["containers"][f"small_bs{bs}"]["sha"]
    bundle = cuda.unpack(blob)
    for a, b in zip(tensors, bundle.tensors):
        assert np.array_equal(a.qvalues, b.qvalues) and a.w_scale == b.w_scale


def test_short_last_chunk_and_empty(cuda, golden):
    tensors, stats = small_model(cuda, rows=100, cols=41)
    blob = cuda.pack(tensors, stats, chunk_size=4096)
    assert hashlib.sha256(blob).hexdigest() == golden["containers"]["small_short"]["sha"]
    empty = cuda.pack([], {})
    assert empty.hex() == golden["containers"]["empty"]["hex"]
    assert cuda.unpack(empty).tensors == []


@pytest.mark.parametrize("name", ["small_bs0", "small_bs1", "small_bs2", "small_bs5", "small_short"])
def test_unpack_reference_files(cuda, oracle, name):
    data = open(f"{GOLDEN}/{name}.dcc", "rb").read()
    want = oracle.unpack(data)
    got = cuda.unpack(data)
    for (n, q, ws, a, s, cm), t in zip(want, got.tensors):
        assert t.name == n and np.array_equal(t.qvalues, q) and t.w_scale == ws
        assert np.array_equal(t.scale_vec.s, s) and np.array_equal(got.stats[n].channel_max, cm)


def test_split_point_decode_equals_exact(cuda):
    from paper_2502_15443_b200 import container, engine
    rng = np.random.default_rng(3)
    for cs, shift in ((4096, 6), (65536, 9), (1 << 20, 9), (300_000, 10), (123_457, 7)):
        q = np.clip(np.round(rng.normal(0, 9, (700, 1500))), -127, 127).astype(np.int8)
        q[:, :40] = 0  # a run of zeros
        t = cuda.QuantizedTensor("w", q, 0.01, cuda.ScaleVector.identity(1500))
        st = {"w": cuda.ActivationStats("w", np.ones(1500))}
        data, index = container.pack_indexed([t], st, chunk_size=cs, seg_shift=shift)
        assert data == cuda.pack([t], st, chunk_size=cs)
        ent = container._parse(data)[2]
        base = cuda.native.to_device_bytes(data)
        jobs = container.jobs_for(ent)
        exact = engine.decode_jobs(base, jobs, build_index=True, seg_shift=shift)
        fast = engine.decode_jobs(base, jobs, index=index)
        assert (exact.status == 0).all() and (fast.status == 0).all()
        assert torch.equal(exact.out, fast.out)
        assert np.array_equal(exact.out.cpu().numpy().view(np.int8).reshape(q.shape), q)
        # the serially built index equals the encoder's
        a1, b1 = index.host_arrays()
        a2, b2 = exact.index.host_arrays()
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2)
        assert np.array_equal(cuda.unpack(data, index=index).tensors[0].qvalues, q)


@pytest.mark.parametrize("chunk", [16384, 65536])  # warp-task small-chunk kernel / CTA-task kernel
def test_broken_index_falls_back_exactly(cuda, chunk):
    from paper_2502_15443_b200 import container, engine
    rng = np.random.default_rng(4)
    q = np.clip(np.round(rng.normal(0, 9, (300, 1000))), -127, 127).astype(np.int8)
    t = cuda.QuantizedTensor("w", q, 0.01, cuda.ScaleVector.identity(1000))
    st = {"w": cuda.ActivationStats("w", np.ones(1000))}
    data, index = container.pack_indexed([t], st, chunk_size=chunk, seg_shift=8)
    assert engine.small_mode(container.jobs_for(container._parse(data)[2])) == (chunk <= 32768)
    index.d_state[5] += 1  # corrupt one split point
    index.d_off[17] += 3
    assert np.array_equal(cuda.unpack(data, index=index).tensors[0].qvalues, q)


@pytest.mark.parametrize("chunk", [16384, 1 << 20])
def test_mixed_codecs_split_point(cuda, chunk):
    """Single-symbol (all-zero), incompressible (stored) and ordinary chunks in one
    container through the split-point path, small-chunk and CTA-task kernels."""
    from paper_2502_15443_b200 import container, engine
    rng = np.random.default_rng(8)
    parts = [np.zeros((64, 1024), np.int8), rng.integers(-128, 128, (64, 1024)).astype(np.int8),
             np.clip(np.round(rng.normal(0, 7, (512, 1024))), -127, 127).astype(np.int8)]
    ts, st = [], {}
    for i, q in enumerate(parts):
        ts.append(cuda.QuantizedTensor(f"m{i}", q, 0.01, cuda.ScaleVector.identity(1024)))
        st[f"m{i}"] = cuda.ActivationStats(f"m{i}", np.ones(1024))
    data, index = container.pack_indexed(ts, st, chunk_size=chunk, seg_shift=8)
    ent = container._parse(data)[2]
    if chunk == 16384:
        assert (ent["codec"] == 0).any() and (ent["codec"] == 1).any()
    base = cuda.native.to_device_bytes(data)
    jobs = container.jobs_for(ent)
    assert engine.small_mode(jobs) == (chunk <= 32768)
    fast = engine.decode_jobs(base, jobs, index=index)
    assert (fast.status == 0).all()
    want = np.concatenate([q.reshape(-1).view(np.uint8) for q in parts])
    assert np.array_equal(fast.out[: want.size].cpu().numpy(), want)


def test_unpack_from_pinned_tensors(cuda):
    """unpack() straight from pinned host tensors (container + sidecar) gives the
    bytes-input result; a corrupted pinned payload raises the same error."""
    from paper_2502_15443_b200 import container
    rng = np.random.default_rng(6)
    ts, st = [], {}
    for i, (r, c) in enumerate([(300, 1000), (128, 4096), (77, 513)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        ts.append(cuda.QuantizedTensor(f"w{i}", q, 0.01, cuda.ScaleVector.identity(c)))
        st[f"w{i}"] = cuda.ActivationStats(f"w{i}", np.ones(c))
    data, index = container.pack_indexed(ts, st, chunk_size=65536, seg_shift=8)
    side = index.to_bytes(container.binding_of(data))
    pin = torch.empty(len(data), dtype=torch.uint8, pin_memory=True)
    pin.numpy()[:] = np.frombuffer(data, np.uint8)
    pside = torch.empty(len(side), dtype=torch.uint8, pin_memory=True)
    pside.numpy()[:] = np.frombuffer(side, np.uint8)
    a = container.unpack(pin, index=pside)
    b = container.unpack(data, index=side)
    for x, y, t in zip(a.tensors, b.tensors, ts):
        assert np.array_equal(x.qvalues, t.qvalues) and np.array_equal(y.qvalues, t.qvalues)
    last = container._parse(data)[2][-1]
    pin.numpy()[int(last["file_offset"]) + 500] ^= 0x40  # payload bit flip in the last chunk
    with pytest.raises((cuda.CorruptStreamError, cuda.ChecksumError)):
        container.unpack(pin, index=pside)


def test_structural_errors_with_sidecar(cuda):
    """unpack(data, index=sidecar) starts the GPU pipeline from the chunk table
    before walking the header body; header / table / length damage must still
    raise exactly what the index-less path (full ordered parse) raises."""
    from paper_2502_15443_b200 import container
    tensors, stats = small_model(cuda, rows=300)
    data, index = container.pack_indexed(tensors, stats, chunk_size=8192, seg_shift=8)
    side = index.to_bytes(container.binding_of(data))
    (hlen,) = struct.unpack_from("<I", data, 6)
    (count,) = struct.unpack_from("<I", data, 10 + hlen)
    prefix = 14 + hlen + 29 * count
    rng = np.random.default_rng(12)

    def outcome(fn):
        try:
            fn()
            return None
        except cuda.DcompError as e:
            return type(e).__name__, str(e)

    mutants = []
    for _ in range(60):
        b = bytearray(data)
        pos = int(rng.integers(10, 10 + hlen - 4))  # header body: the sidecar still binds
        b[pos] ^= 1 << int(rng.integers(0, 8))
        mutants.append(bytes(b))
    for _ in range(20):
        b = bytearray(data)
        b[int(rng.integers(0, prefix))] ^= 1 << int(rng.integers(0, 8))
        mutants.append(bytes(b))
    mutants += [data[:-1], data + b"\x00", data[:prefix + 5]]
    raised = 0
    pside = torch.empty(len(side), dtype=torch.uint8, pin_memory=True)
    pside.numpy()[:] = np.frombuffer(side, np.uint8)
    for i, m in enumerate(mutants):
        want = outcome(lambda: container.unpack(m))
        got = outcome(lambda: container.unpack(m, index=side))
        assert got == want
        if i % 4 == 0:  # the pinned-tensor input parses a zero-copy view of the prefix
            pin = torch.empty(len(m), dtype=torch.uint8, pin_memory=True)
            pin.numpy()[:] = np.frombuffer(m, np.uint8)
            assert outcome(lambda: container.unpack(pin, index=pside)) == want
        raised += want is not None
    assert raised >= 70


def test_sidecar_roundtrip(cuda, tmp_path):
    rng = np.random.default_rng(5)
    q = np.clip(np.round(rng.normal(0, 9, (200, 1000))), -127, 127).astype(np.int8)
    t = cuda.QuantizedTensor("w", q, 0.01, cuda.ScaleVector.identity(1000))
    st = {"w": cuda.ActivationStats("w", np.ones(1000))}
    p = tmp_path / "m.dcc"
    cuda.write_container(p, [t], st, chunk_size=65536, sidecar=True)
    assert (tmp_path / "m.dcc.dcidx").exists()
    assert np.array_equal(cuda.container.read_container(p).tensors[0].qvalues, q)


def test_corruption_errors_match_oracle(cuda, oracle):
    tensors, stats = small_model(cuda, rows=200)
    data = cuda.pack(tensors, stats, chunk_size=4096)
    info = cuda.inspect(data)
    rng = np.random.default_rng(9)
    checked = 0
    for _ in range(300):
        c = info.chunks[int(rng.integers(0, len(info.chunks)))]
        pos = c.file_offset + int(rng.integers(0, c.comp_len))
        b = bytearray(data)
        b[pos] ^= 1 << int(rng.integers(0, 8))
        b = bytes(b)
        try:
            oracle.unpack(b)
            want = None
        except oracle.OracleError as e:
            want = (e.kind, e.msg)
        try:
            cuda.unpack(b)
            got = None
        except cuda.DcompError as e:
            got = (type(e).__name__, str(e))
        assert got == want
        checked += want is not None
    assert checked > 250


def test_c1_opt125m_digests(cuda, model_digests):
    """C1 parity config: OPT-125M-shaped synthetic weights, alpha 0.5, per-tensor
    prune 0.2: GPU quantize+prune+pack bytes == the reference's (SHA-256)."""
    import importlib
    tens = importlib.import_module("paper_2502_15443_b200.tensors")
    for key, alpha, sp in (("opt125m_a0.5_p0.2", 0.5, 0.2), ("opt125m_a0.0_p0.0", 0.0, 0.0)):
        want = model_digests[key]
        qts, stats = [], {}
        h = hashlib.sha256()
        for i, (name, r, c) in enumerate(tens.model_layout("opt-125m")):
            w, s = cuda.synth_ensemble(cuda.SynthSpec(rows=r, cols=c, name=name), 1000 + i)
            qt = cuda.quantize_scaled(w, s, alpha)
            assert struct.pack("<d", qt.w_scale).hex() == want["w_scales"][i]
            if sp:
                qt = cuda.prune(qt, s, cuda.PruneConfig(sp))
            h.update(qt.qvalues.tobytes())
            qts.append(qt)
            stats[name] = s
        assert h.hexdigest() == want["q_sha"]
        for cs, meta in want["containers"].items():
            blob = cuda.pack(qts, stats, chunk_size=int(cs))
            assert len(blob) == meta["size"]
            assert hashlib.sha256(blob).hexdigest() == meta["sha"]
            back = cuda.unpack(blob)
            assert all(np.array_equal(a.qvalues, b.qvalues) for a, b in zip(qts, back.tensors))


@pytest.mark.parametrize("chunk,mode", [(65536, "narrow"), (98304, "wide"), (32768, "small")])
def test_decoder_mode_selection_exact(cuda, chunk, mode, monkeypatch):
    """Each split-point decoder (warp-task / 4-warp / 8-warp CTAs) is picked by
    chunk size and decodes bit-exactly; forcing the narrow kernel onto larger
    chunks (multi-task chunks) stays exact too."""
    from paper_2502_15443_b200 import container, engine
    rng = np.random.default_rng(chunk)
    ts, st = [], {}
    for i, (r, c) in enumerate([(700, 1000), (256, 2304)]):
        q = np.clip(np.round(rng.normal(0, 7, (r, c))), -127, 127).astype(np.int8)
        ts.append(cuda.QuantizedTensor(f"w{i}", q, 0.01, cuda.ScaleVector.identity(c)))
        st[f"w{i}"] = cuda.ActivationStats(f"w{i}", np.ones(c))
    data, index = container.pack_indexed(ts, st, chunk_size=chunk, seg_shift=8)
    jobs = container.jobs_for(container._parse(data)[2])
    assert engine.decode_mode(jobs) == mode
    side = index.to_bytes(container.binding_of(data))
    out = container.unpack(data, index=side)
    for x, t in zip(out.tensors, ts):
        assert np.array_equal(x.qvalues, t.qvalues)
    monkeypatch.setenv("DCOMP_NARROW_MAX_CHUNK", str(1 << 30))
    if mode == "wide":
        assert engine.decode_mode(jobs) == "narrow"
        out = container.unpack(data, index=side)
        for x, t in zip(out.tensors, ts):
            assert np.array_equal(x.qvalues, t.qvalues)


def test_index_less_unpack_records_index_for_next_call(cuda):
    """unpack(file) with no sidecar runs the serial chains and keeps the split
    points they record; the next unpack of the same container takes the
    parallel path (same bytes), and a payload-corrupted copy (same binding)
    still raises the reference's error."""
    from paper_2502_15443_b200 import container
    container.clear_index_cache()
    tensors, stats = small_model(cuda, rows=400, cols=512)
    data = cuda.pack(tensors, stats, chunk_size=65536)
    a = container.unpack(data)
    assert len(container._INDEX_CACHE) == 1
    assert "table" not in container.LAST_UNPACK_MS
    b = container.unpack(data)
    assert "table" in container.LAST_UNPACK_MS  # pipelined split-point path
    for x, y, t in zip(a.tensors, b.tensors, tensors):
        assert np.array_equal(x.qvalues, t.qvalues) and np.array_equal(y.qvalues, t.qvalues)
    info = cuda.inspect(data)
    bad = bytearray(data)
    bad[info.chunks[1].file_offset + 100] ^= 0x10
    with pytest.raises((cuda.CorruptStreamError, cuda.ChecksumError)):
        container.unpack(bytes(bad))
    container.clear_index_cache()


@pytest.mark.parametrize("chunk", [4096, 5000, 12345, 65537, 100003, 300001])
def test_odd_chunk_sizes_split_point_exact(cuda, oracle, chunk):
    """Chunk sizes that are not multiples of the 256-symbol segment (ragged last
    segments everywhere), every decoder mode: file bytes equal the oracle's pack,
    the sidecar-driven decode equals the tensors."""
    from paper_2502_15443_b200 import container
    rng = np.random.default_rng(chunk)
    ts, st, ents = [], {}, []
    for i, (r, c) in enumerate([(333, 700), (129, 1001)]):
        q = np.clip(np.round(rng.normal(0, 11, (r, c))), -127, 127).astype(np.int8)
        ts.append(cuda.QuantizedTensor(f"t{i}", q, 0.02, cuda.ScaleVector.identity(c)))
        st[f"t{i}"] = cuda.ActivationStats(f"t{i}", np.ones(c))
        ents.append((f"t{i}", q, 0.02, 0.0, np.ones(c), np.ones(c)))
    data, index = container.pack_indexed(ts, st, chunk_size=chunk, seg_shift=8)
    assert data == oracle.pack(ents, chunk)
    out = container.unpack(data, index=index.to_bytes(container.binding_of(data)))
    for x, t in zip(out.tensors, ts):
        assert np.array_equal(x.qvalues, t.qvalues)
