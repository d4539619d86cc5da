"""container.pack (the reference API: host QuantizedTensors in, DCC1 bytes out)
on the GPU vs the oracle's pack (the reference algorithm, all host threads),
on an OPT-1.3B-shaped model (one synthetic layer tiled over every layer)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2502_15443_b200 import container  # noqa: E402
from paper_2502_15443_b200.scaling import QuantizedTensor, ScaleVector  # noqa: E402
from paper_2502_15443_b200.tensors import ActivationStats, SynthSpec, model_layout, synth_ensemble  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b"
full = model_layout(model)
layer = full[:6]
made = []
for i, (name, r, c) in enumerate(layer):
    w, st = synth_ensemble(SynthSpec(rows=r, cols=c, name=name), 1000 + i)
    s = O.compute_scale(st.channel_max, 0.5)
    q, ws = O.quantize(w.values, s)
    made.append((q, ws, s, st.channel_max))
n_layers = len(full) // 6
tensors, stats, entries = [], {}, []
for L in range(n_layers):
    for (name, _, _), (q, ws, s, cm) in zip(layer, made):
        nm = f"layers.{L}.{name.split('.')[-1]}"
        tensors.append(QuantizedTensor(nm, q, ws, ScaleVector(0.5, s)))
        stats[nm] = ActivationStats(nm, cm)
        entries.append((nm, q, ws, 0.5, s, cm))
raw = sum(t.qvalues.size for t in tensors)
for i in range(3):
    t0 = time.perf_counter()
    data = container.pack(tensors, stats)
    dt = time.perf_counter() - t0
    print(f"GPU container.pack: {dt * 1e3:.0f} ms  {raw / dt / 1e9:.2f} GB/s  ({len(data)} bytes)", flush=True)
threads = os.cpu_count() or 1
t0 = time.perf_counter()
ref = O.pack(entries, 16 << 20, threads=threads)
dt = time.perf_counter() - t0
print(f"oracle pack ({threads} threads): {dt * 1e3:.0f} ms  {raw / dt / 1e9:.2f} GB/s", flush=True)
print("bytes identical:", ref == data)

if os.environ.get("PROFILE"):
    import cProfile
    import pstats
    import torch
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    container.pack(tensors, stats)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
