"""A damaged split-point sidecar (.dcidx) must never fault a kernel or change
a result: the kernels never form an address from a split point outside its
chunk's stream span, wild or stale split points are caught by the chain
checks (exact serial re-decode), and a sidecar whose body CRC fails is not
trusted at all."""

import struct
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _model(dc, chunk, seed=0):
    from paper_2502_15443_b200 import container
    rng = np.random.default_rng(seed)
    ts, st = [], {}
    for i, (r, c) in enumerate([(300, 1024), (256, 2048), (77, 512)]):
        q = np.clip(np.round(rng.normal(0, 9, (r, c))), -127, 127).astype(np.int8)
        ts.append(dc.QuantizedTensor(f"w{i}", q, 0.01, dc.ScaleVector.identity(c)))
        st[f"w{i}"] = dc.ActivationStats(f"w{i}", np.ones(c))
    data, index = container.pack_indexed(ts, st, chunk_size=chunk, seg_shift=8)
    return ts, data, index.to_bytes(container.binding_of(data))


def _pinned(b: bytes) -> torch.Tensor:
    t = torch.empty(len(b), dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = np.frombuffer(b, np.uint8)
    return t


def _recrc(side: bytearray) -> bytes:
    n = struct.unpack_from("<Q", side, 14)[0]
    struct.pack_into("<I", side, 22 + 8 * n, zlib.crc32(bytes(side[22:22 + 8 * n])))
    return bytes(side)


@pytest.mark.parametrize("chunk", [16384, 65536, 1 << 20])  # small / narrow / wide decoders
def test_damaged_sidecar_exact_or_fallback(cuda, chunk):
    from paper_2502_15443_b200 import container
    ts, data, side = _model(cuda, chunk)
    n = struct.unpack_from("<Q", side, 14)[0]
    rng = np.random.default_rng(chunk)
    cases = []
    for _ in range(12):  # random bit flips anywhere in the body (CRC now fails)
        b = bytearray(side)
        b[22 + int(rng.integers(0, 8 * n))] ^= 1 << int(rng.integers(0, 8))
        cases.append(bytes(b))
    for _ in range(12):  # wild offsets / states with a consistent CRC: the kernels see them
        b = bytearray(side)
        k = int(rng.integers(0, n))
        if rng.random() < 0.7:  # stream offset: high byte flipped (far outside the stream)
            b[22 + 4 * n + 4 * k + 3] ^= 1 << int(rng.integers(0, 8))
        else:
            b[22 + 4 * k + int(rng.integers(0, 4))] ^= 1 << int(rng.integers(0, 8))
        cases.append(_recrc(b))
    b = bytearray(side)  # every offset of the body set to 0xFFFFFFF0
    b[22 + 4 * n:22 + 8 * n] = np.full(n, 0xFFFFFFF0, np.uint32).tobytes()
    cases.append(_recrc(b))
    for bad in cases:
        for sidecar in (bad, _pinned(bad)):
            got = container.unpack(_pinned(data) if isinstance(sidecar, torch.Tensor) else data, index=sidecar)
            for a, t in zip(got.tensors, ts):
                assert np.array_equal(a.qvalues, t.qvalues)
    torch.cuda.synchronize()  # no sticky fault


def test_sidecar_crc_checked_before_trust(cuda):
    from paper_2502_15443_b200 import container, engine
    ts, data, side = _model(cuda, 65536)
    ent = container._parse(data)[2]
    jobs = container.jobs_for(ent)
    bind = container.binding_of(data)
    assert engine.SegmentIndex.from_bytes(side, jobs, bind) is not None
    b = bytearray(side)
    b[30] ^= 4
    assert engine.SegmentIndex.from_bytes(bytes(b), jobs, bind) is None
    assert engine.SegmentIndex.from_bytes(_pinned(bytes(b)), jobs, bind) is None
    lazy = engine.SegmentIndex.from_bytes(_pinned(bytes(b)), jobs, bind, lazy=True)
    lazy.ensure_uploaded()
    assert not lazy.body_crc_ok()


def test_fused_ring_wild_split_points(cuda):
    """The fused decode -> tcgen05 kernel flags (never dereferences) split
    points outside the stream; run_checked() then gives the exact product."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(1)
    shapes = [(1024, 1024), (512, 2048)]
    ws = [torch.round(torch.randn(r, k, generator=g) * 9).clamp_(-127, 127).to(torch.int8) for r, k in shapes]
    xs = [torch.randint(-127, 128, (2, k), generator=g, dtype=torch.int8) for _, k in shapes]
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, 1 << 21, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    enc.index.d_off[5] = 0x7FFFFFF0
    enc.index.d_off[700] = -16
    fr = FusedRing(image, jobs, enc.index, 1 << 21, shapes, t_offs, [x.cuda() for x in xs], 2)
    fr.run()
    torch.cuda.synchronize()
    assert (fr.check() != 0).any()
    assert not fr.run_checked()
    for w, x, acc in zip(ws, xs, fr.accs):
        assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)
