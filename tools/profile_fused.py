"""Run the fused TMEM-ring decode-GEMM on OPT-1.3B-shaped layers (ncu target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import synth  # noqa: E402
from paper_2502_15443_b200.gemm import FusedRing  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4  # 0 = every layer
model = sys.argv[2] if len(sys.argv) > 2 else "opt-1.3b"
m = synth.build_model(model, layers=layers or None)
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 16 << 20
pm = synth.pack_model(m, chunk, seg_shift=8)
g = torch.Generator(device="cuda")
g.manual_seed(1)
xs = [torch.randint(-127, 128, (1, c), generator=g, device="cuda", dtype=torch.int8) for _, c in m.shapes]
fr = FusedRing(pm.image, pm.jobs, pm.index, pm.chunk_size, m.shapes, m.offsets()[:-1], xs, 1)
for i in range(int(os.environ.get("ITERS", 3))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fr.run()
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {i}: {e0.elapsed_time(e1):.3f} ms  {m.nbytes / e0.elapsed_time(e1) / 1e6:.1f} GB/s", flush=True)
assert (fr.check() == 0).all()
print(f"native layers {fr.native_layers}, fallback layers {len(fr._fb_layers)}")
print("ok")
