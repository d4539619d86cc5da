"""Time the TP-8 rank-0 LLaMA-13B shard step (fused vs INT8) on one GPU.

    python tools/profile_tp.py [model] [world]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import tp_step  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "llama-13b"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tps = tp_step.TPDecodeStep(model, world, 0, ntok=1, device=torch.device("cuda", 0))
f = tps.fused
print("native layers", f.native_layers, "fallback layers", len(f._fb_layers),
      "fallback groups", len(f._fb.groups) if f._fb else 0)
r = tp_step.measure_local(tps, iters=10)
print(r)
if len(sys.argv) > 3:  # extra fused launches for ncu (-k regex:k_fused_ring -s N)
    for _ in range(int(sys.argv[3])):
        tps.fused.run()
    torch.cuda.synchronize()
