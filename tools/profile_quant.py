"""Time the quantize kernels (absmax pass + quantize pass) on an OPT-6.7B fc1-shaped
tensor for each input dtype; prints HBM GB/s per kernel (ncu target too).

    python tools/profile_quant.py [rows cols]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import native as nv  # noqa: E402
from paper_2502_15443_b200.scaling import _DTYPE_CODE  # noqa: E402

rows, cols = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16384, 4096)
g = torch.Generator(device="cuda")
g.manual_seed(0)
s = torch.rand(cols, generator=g, device="cuda", dtype=torch.float64) + 0.5
bits = torch.zeros(1, dtype=torch.int64, device="cuda")
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
q = torch.empty(rows, cols, dtype=torch.int8, device="cuda")
for dt in (torch.float64, torch.float32, torch.bfloat16):
    w = (torch.randn(rows, cols, generator=g, device="cuda", dtype=torch.float32) * 0.2).to(dt)
    n = w.numel()

    def absmax():
        nv.call("dc_quant_absmax", w.data_ptr(), _DTYPE_CODE[dt], s.data_ptr(), rows, cols, bits.data_ptr(),
                bad.data_ptr(), nv.stream_ptr())

    def quant():
        nv.call("dc_quantize", w.data_ptr(), _DTYPE_CODE[dt], s.data_ptr(), rows, cols, ctypes.c_double(0.01),
                q.data_ptr(), nv.stream_ptr())

    for name, fn, nbytes in (("absmax", absmax, n * w.element_size()),
                             ("quantize", quant, n * w.element_size() + n)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{str(dt):15s} {name:9s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:8.1f} GB/s", flush=True)
