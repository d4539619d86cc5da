"""Phase times of container.pack through the API (OPT-1.3B shape, 16 MiB chunks):
header, payload staging + H2D, encode (+ assemble), D2H, bytes."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_15443_b200 as dc  # noqa: E402
from paper_2502_15443_b200 import container, native as nv  # noqa: E402
from paper_2502_15443_b200.tensors import model_layout  # noqa: E402

full = model_layout(sys.argv[1] if len(sys.argv) > 1 else "opt-1.3b")
made = []
for i, (name, r, c) in enumerate(full[:6]):
    w, st = dc.synth_ensemble(dc.SynthSpec(rows=r, cols=c, name=name), 1000 + i)
    made.append((dc.quantize_scaled(w, st, 0.5), st.channel_max))
tensors, stats = [], {}
for L in range(len(full) // 6):
    for (name, _, _), (qt, cm) in zip(full[:6], made):
        nm = f"layers.{L}.{name.split('.')[-1]}"
        tensors.append(dc.QuantizedTensor(nm, qt.qvalues, qt.w_scale, qt.scale_vec))
        stats[nm] = dc.ActivationStats(nm, cm)
for it in range(3):
    t = [time.perf_counter()]
    header = container._header(tensors, stats, 16 << 20)
    t.append(time.perf_counter())
    payload = container._device_payload(tensors)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    image, enc, _ = container.pack_device(payload, header, 16 << 20, None, None)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    host = nv.to_host(image)
    t.append(time.perf_counter())
    data = host.tobytes()
    t.append(time.perf_counter())
    names = ["header", "stage+h2d", "encode+assemble", "d2h", "tobytes"]
    print(f"iter {it}: " + "  ".join(f"{n} {1e3 * (b - a):.1f} ms" for n, a, b in zip(names, t, t[1:])) +
          f"  total {1e3 * (t[-1] - t[0]):.1f} ms", flush=True)
    t0 = time.perf_counter()
    d2 = container.pack(tensors, stats)
    print(f"   pack() {1e3 * (time.perf_counter() - t0):.1f} ms, equal {d2 == data}", flush=True)
