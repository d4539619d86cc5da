"""Host/GPU profile of container.pack at the C1 shape (OPT-125M, 256 KiB chunks).

    python tools/profile_pack_c1.py
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2502_15443_b200 as dc  # noqa: E402
from paper_2502_15443_b200.tensors import model_layout  # noqa: E402

qts, stats = [], {}
for i, (n, r, c) in enumerate(model_layout("opt-125m")):
    w, s = dc.synth_ensemble(dc.SynthSpec(rows=r, cols=c, name=n), 1000 + i)
    qts.append(dc.prune(dc.quantize_scaled(w, s, 0.5), s, dc.PruneConfig(0.2)))
    stats[n] = s
for cs in (256 << 10, 16 << 20):
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blob = dc.pack(qts, stats, chunk_size=cs)
        print(f"chunk {cs >> 10} KiB pack {1e3 * (time.perf_counter() - t0):.1f} ms ({len(blob)} B)", flush=True)
for i in range(3):  # fresh host arrays every call (as a caller re-quantizing would pass)
    fresh = [dc.QuantizedTensor(q.name, q.qvalues.copy(), q.w_scale, q.scale_vec) for q in qts]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dc.pack(fresh, stats, chunk_size=256 << 10)
    print(f"fresh arrays pack {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
fresh = [dc.QuantizedTensor(q.name, q.qvalues.copy(), q.w_scale, q.scale_vec) for q in qts]
pr = cProfile.Profile()
pr.enable()
dc.pack(fresh, stats, chunk_size=256 << 10)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
