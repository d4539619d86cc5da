"""Device CRC-32 (zlib.crc32, the reference's chunk checksum, container.py:169,
:329) of many byte ranges: the lane-piece kernel (16-B aligned range ends,
whole 4 KB pieces) and the 256-byte piece kernel (heads, unaligned ends)
together equal zlib on every range."""

import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _crcs(buf: np.ndarray, offs, lens):
    from paper_2502_15443_b200 import engine
    d = torch.from_numpy(buf).cuda()
    o = torch.tensor(offs, dtype=torch.int64).cuda()
    n = torch.tensor(lens, dtype=torch.int64).cuda()
    got = engine.crc32_ranges(d, o, n, max(lens) if lens else 0).cpu().numpy().view(np.uint32)
    want = [zlib.crc32(buf[a:a + b]) for a, b in zip(offs, lens)]
    return got, np.array(want, dtype=np.uint32)


def test_crc_ranges_mixed(cuda):
    rng = np.random.default_rng(0)
    buf = rng.integers(0, 256, 40 << 20, dtype=np.uint8)
    offs, lens = [], []
    for L in [1, 15, 16, 4095, 4096, 4097, 8192, 131072, 131072 + 16, 131071, 1 << 20, (1 << 20) + 48,
              (3 << 20) + 4096 * 7 + 16, 16 << 20, 0]:
        for _ in range(2):
            a = int(rng.integers(0, buf.size - L - 1))
            if rng.random() < 0.5:  # 16-B aligned end -> lane kernel
                a -= (a + L) % 16
            offs.append(a)
            lens.append(L)
    got, want = _crcs(buf, offs, lens)
    assert np.array_equal(got, want)


def test_crc_chunk_table_layout(cuda):
    """Back-to-back chunks of one payload, as unpack checks them."""
    rng = np.random.default_rng(1)
    chunk = 1 << 20
    total = 37 * chunk + 12345
    buf = (rng.normal(0, 6, total).astype(np.int8)).view(np.uint8)
    offs = list(range(0, total, chunk))
    lens = [min(chunk, total - o) for o in offs]
    got, want = _crcs(buf, offs, lens)
    assert np.array_equal(got, want)
