"""CRC-32 of N x 16 MiB device ranges (the bench's per-chunk checksum pass):
times dc_crc32_ranges with CUDA events; run under ncu for the kernel profile.

    python tools/profile_crc.py [n_chunks] [chunk_bytes]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_15443_b200 import engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 384
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 16 << 20
g = torch.Generator(device="cuda").manual_seed(0)
buf = torch.randint(0, 256, (n * chunk,), dtype=torch.uint8, device="cuda", generator=g)
off = torch.arange(n, dtype=torch.int64, device="cuda") * chunk
ln = torch.full((n,), chunk, dtype=torch.int64, device="cuda")
for _ in range(3):
    engine.crc32_ranges(buf, off, ln, chunk)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    engine.crc32_ranges(buf, off, ln, chunk)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"crc {n} x {chunk} B: {ms:.3f} ms, {n * chunk / ms / 1e6:.1f} GB/s")
