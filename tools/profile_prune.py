"""Time prune_device (per-tensor and per-row) on an OPT-6.7B fc1-shaped int8 tensor.

    python tools/profile_prune.py [rows cols sparsity]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200.pruning import prune_device  # noqa: E402

rows, cols, sp = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (16384, 4096, 0.2)
g = torch.Generator(device="cuda")
g.manual_seed(0)
q = torch.clamp(torch.round(torch.randn(rows, cols, generator=g, device="cuda") * 30), -127, 127).to(torch.int8)
cm = torch.exp(torch.randn(cols, generator=g, device="cuda", dtype=torch.float64) - 1)
for per_row in (False, True):
    for _ in range(2):
        out = prune_device(q, cm, sp, per_row)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        out = prune_device(q, cm, sp, per_row)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    n = q.numel()
    z = int((out == 0).sum())
    print(f"per_row={per_row}: {ms:.3f} ms  {2 * n / ms / 1e6:.1f} GB/s (read q + write out)  zeros={z / n:.4f}",
          flush=True)
