"""GPU parity of the rANS codec against the reference's golden blobs and the
C oracle: bit-exact blobs, tables, decoded bytes and error verdicts."""

import hashlib

import numpy as np
import pytest

from conftest import split_concat

pytestmark = pytest.mark.gpu


def test_for_data_and_blobs_bit_exact(cuda, codec_golden):
    datas = split_concat(codec_golden["data"], codec_golden["data_len"])
    blobs = split_concat(codec_golden["blob"], codec_golden["blob_len"])
    for d, b, f in zip(datas, blobs, codec_golden["freq"]):
        assert np.array_equal(cuda.AnsTable.for_data(d).frequencies, f)
        assert cuda.compress_blob(d) == b.tobytes()
        assert cuda.decompress_blob(b.tobytes(), d.size) == d.tobytes()


def test_corrupt_verdicts_match_reference(cuda, golden):
    for case in golden["corrupt"]["cases"]:
        blob = bytes.fromhex(case["blob_hex"])
        want = case["verdict"]
        try:
            out = cuda.decompress_blob(blob, case["out_len"])
            got = {"ok": True, "sha": hashlib.sha256(out).hexdigest()}
        except cuda.DcompError as e:
            got = {"ok": False, "cls": type(e).__name__, "msg": str(e)}
        assert got == want, (case["kind"], case["arg"])


def test_random_roundtrips_match_oracle(cuda, oracle):
    rng = np.random.default_rng(11)
    for _ in range(60):
        n = int(rng.integers(1, 40_000))
        kind = rng.integers(0, 3)
        if kind == 0:
            d = rng.integers(0, int(rng.integers(2, 257)), n).astype(np.uint8)
        elif kind == 1:
            d = np.clip(np.abs(rng.laplace(0, float(rng.uniform(0.3, 40)), n)), 0, 255).astype(np.uint8)
        else:
            d = np.clip(np.round(rng.normal(0, float(rng.uniform(1, 30)), n)), -127, 127).astype(np.int8).view(np.uint8)
        blob = cuda.compress_blob(d)
        assert blob == oracle.compress_blob(d)
        assert cuda.decompress_blob(blob, n) == d.tobytes()


def test_decode_blobs_into_grouping_and_isolation(cuda):
    rng = np.random.default_rng(12)
    datas = [rng.integers(0, int(rng.integers(2, 200)), 4096).astype(np.uint8) for _ in range(11)]
    outs = [np.empty(4096, np.uint8) for _ in datas]
    cuda.ans.decode_blobs_into([(cuda.compress_blob(d), o) for d, o in zip(datas, outs)])
    for d, o in zip(datas, outs):
        assert np.array_equal(d, o)
    # corrupt one lane of four: the error names it
    datas = [rng.integers(0, 30, 4096).astype(np.uint8) for _ in range(4)]
    blobs = [bytearray(cuda.compress_blob(d)) for d in datas]
    blobs[2][cuda.ans.HEADER_BYTES + 5] ^= 0x55
    outs = [np.empty(4096, np.uint8) for _ in range(4)]
    with pytest.raises(cuda.CorruptStreamError, match="chunk c2"):
        cuda.ans.decode_blobs_into([(bytes(b), o) for b, o in zip(blobs, outs)], labels=["c0", "c1", "c2", "c3"])
    # mixed lengths
    datas = [rng.integers(0, 50, n).astype(np.uint8) for n in (100, 100, 100, 100, 7, 7, 9)]
    outs = [np.empty(d.size, np.uint8) for d in datas]
    cuda.ans.decode_blobs_into([(cuda.compress_blob(d), o) for d, o in zip(datas, outs)])
    assert all(np.array_equal(d, o) for d, o in zip(datas, outs))


def test_edge_cases(cuda):
    with pytest.raises(cuda.DcompError, match="empty input"):
        cuda.ans_compress(np.empty(0, np.uint8))
    for b in (0, 7, 255):
        d = np.array([b], np.uint8)
        assert cuda.decompress_blob(cuda.compress_blob(d), 1) == d.tobytes()
    big = np.full(10_000, 9, np.uint8)
    blob = cuda.compress_blob(big)
    assert len(blob) <= 420
    q = np.random.default_rng(6).integers(-128, 128, 1000).astype(np.int8)
    assert np.array_equal(np.frombuffer(cuda.decompress_blob(cuda.compress_blob(q), 1000), np.int8), q)
    t = cuda.AnsTable.for_data(np.array([3, 9] * 51 + [3], np.uint8))
    assert t.frequencies[3] > t.frequencies[9]


def test_long_stream(cuda):
    d = np.abs(np.random.default_rng(7).laplace(0, 6, 2**20)).astype(np.uint8)
    assert cuda.decompress_blob(cuda.compress_blob(d), d.size) == d.tobytes()


def test_singleton_symbols_f1_bit_exact(cuda, oracle):
    """Symbols whose normalized frequency is 1 (rare bytes in a long skewed
    chunk) take the encoder's f == 1 reciprocal form; blobs equal the oracle's
    and decode back."""
    rng = np.random.default_rng(17)
    for n, k in ((1 << 16, 12), (1 << 20, 40), (300_000, 3)):
        data = np.zeros(n, np.uint8)
        data[: n // 3] = rng.integers(1, 4, n // 3)
        pos = rng.choice(n, size=k, replace=False)
        data[pos] = rng.integers(100, 256, k).astype(np.uint8)  # each appears ~once -> f == 1
        rng.shuffle(data)
        blob = cuda.compress_blob(data.tobytes())
        assert blob == oracle.compress_blob(data.tobytes())
        table = cuda.AnsTable.from_bytes(blob[:384])
        assert (table.frequencies == 1).sum() >= 1
        assert cuda.decompress_blob(blob, n) == data.tobytes()


def _shannon_bits(d):
    p = np.bincount(d, minlength=256).astype(np.float64) / d.size
    p = p[p > 0]
    return float(-(p * np.log2(p)).sum())


def test_entropy_window_and_distributions(cuda, oracle):
    """The reference's size bounds (test_ans.py TestSizeBounds, test_acceptance.py
    codec optimality): every GPU blob within [0.99 H - 16, 1.03 H + 400] bytes of
    the Shannon bound, and byte-identical to the oracle, on ten distributions."""
    rng = np.random.default_rng(2024)
    n = 100_000
    streams = {
        "uniform256": rng.integers(0, 256, n, dtype=np.uint8),
        "uniform16": rng.integers(0, 16, n).astype(np.uint8),
        "uniform2": rng.integers(0, 2, n).astype(np.uint8),
        "constant": np.full(n, 7, dtype=np.uint8),
        "bernoulli": rng.choice([0, 1], n, p=[0.97, 0.03]).astype(np.uint8),
        "geometric": np.minimum(rng.geometric(0.2, n) - 1, 255).astype(np.uint8),
        "zipf": np.minimum(rng.zipf(1.4, n) - 1, 255).astype(np.uint8),
        "binomial": rng.binomial(255, 0.5, n).astype(np.uint8),
        "poisson": np.minimum(rng.poisson(30, n), 255).astype(np.uint8),
        "gauss_int8": np.clip(np.rint(rng.normal(0, 9, n)), -127, 127).astype(np.int8).view(np.uint8),
    }
    for name, data in streams.items():
        ideal = n * _shannon_bits(data) / 8
        blob = cuda.compress_blob(data)
        assert 0.99 * ideal - 16 <= len(blob) <= 1.03 * ideal + 400, name
        assert blob == oracle.compress_blob(data), name
        assert cuda.decompress_blob(blob, n) == data.tobytes(), name


@pytest.mark.parametrize("chunk", [16 << 10, 64 << 10, 1 << 20])
def test_segment_range_tasks_decode_exactly_those_segments(cuda, chunk):
    """SegmentIndex.tasks(seg_range=...) (the fused fallback's partial-chunk
    decode): every chunk's [first, end) segment range, including ranges that
    start and end mid-chunk, is decoded exactly and nothing outside it is
    written -- for the small, narrow and wide decoders."""
    import torch

    from paper_2502_15443_b200 import container, engine
    rng = np.random.default_rng(chunk)
    n_bytes = 5 * chunk + 4321
    payload = torch.from_numpy(np.clip(np.round(rng.normal(0, 6, n_bytes)), -127, 127).astype(np.int8)
                               .view(np.uint8)).cuda()
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    nseg = (jobs.out_len.astype(np.int64) + 255) // 256
    lo = np.array([(3 * i) % max(int(s), 1) for i, s in enumerate(nseg)], dtype=np.int64)
    hi = np.minimum(nseg, lo + 1 + (nseg // 3))
    tasks = enc.index.tasks(jobs, np.ones(jobs.n, bool), seg_range=(lo, hi))
    out = torch.full_like(payload, 0xA5)
    status = torch.zeros(jobs.n, dtype=torch.int32, device=payload.device)
    engine.decode_segments(image, jobs, enc.index, tasks, out, status)
    torch.cuda.synchronize()
    assert int(status.abs().sum()) == 0
    got, want = out.cpu().numpy(), payload.cpu().numpy()
    mask = np.zeros(n_bytes, bool)
    for c in range(jobs.n):
        a = int(jobs.out_off[c]) + 256 * int(lo[c])
        b = min(int(jobs.out_off[c]) + 256 * int(hi[c]), int(jobs.out_off[c] + jobs.out_len[c]))
        mask[a:b] = True
    assert np.array_equal(got[mask], want[mask])
    assert (got[~mask] == 0xA5).all()
