"""bench_codecs (reference bench.py:25-72): same rows/columns/errors; the
GPU-resident row is opt-in."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bench_codecs_rows(cuda):
    rng = np.random.default_rng(0)
    data = np.clip(np.round(rng.normal(0, 6, 3 << 20)), -127, 127).astype(np.int8).view(np.uint8)
    assert [r.codec for r in cuda.bench_codecs(data, repetitions=3, chunk_size=1 << 20)] == ["store", "ans"]
    rows = cuda.bench_codecs(data, repetitions=3, chunk_size=1 << 20, gpu_row=True)
    assert [r.codec for r in rows] == ["store", "ans", "ans-gpu"]
    assert rows[0].cr == 1.0 and rows[1].cr > 1.5 and rows[2].cr == pytest.approx(rows[1].cr, rel=1e-3)
    assert all(r.compress_mbps > 0 and r.decompress_mbps > 0 for r in rows)
    assert set(rows[1].to_dict()) == {"codec", "cr", "compress_mbps", "decompress_mbps"}
    with pytest.raises(cuda.DcompError):
        cuda.bench_codecs(data[:1000])
    with pytest.raises(cuda.DcompError):
        cuda.bench_codecs(data, repetitions=2)
