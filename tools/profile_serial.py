"""Exact serial decode of every chunk (no split-point index), OPT-1.3B layers."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15443_b200 import engine, synth  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
model = sys.argv[2] if len(sys.argv) > 2 else "opt-1.3b"
m = synth.build_model(model, layers=layers or None)
pm = synth.pack_model(m, 16 << 20, seg_shift=None)
for i in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = engine.decode_jobs(pm.image, pm.jobs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"serial decode {pm.jobs.n} chunks: {ms:.1f} ms  {m.nbytes / ms / 1e6:.2f} GB/s  "
          f"per chunk {16.77e6 / (ms / 1e3) / 1e6:.1f} MB/s", flush=True)
assert (res.status == 0).all() and torch.equal(res.out[: m.nbytes], m.payload)
