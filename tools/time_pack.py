"""Time the GPU pack path (quantized payload -> DCC1 image + split-point index)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import synth  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b"
m = synth.build_model(model)
for i in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"pack {model}: {dt * 1e3:.1f} ms  {m.nbytes / dt / 1e9:.2f} GB/s  chunks={pm.jobs.n} CR={pm.raw_bytes / pm.file_bytes:.3f}",
          flush=True)
