"""dcomp sweep on the GPU at model scale: CR / near-zero / layer error over the
alpha grid for one transformer layer of a model shape (the CPU-oracle comparison
and CR equality live in tests/test_perf_vs_oracle_gpu.py).

    python tools/alpha_sweep.py [--model opt-1.3b] [--sparsity 0.0] [--out profiles/r1_alpha_sweep.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import sweep  # noqa: E402
from paper_2502_15443_b200.tensors import SynthSpec, model_layout, synth_ensemble  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-1.3b")
    p.add_argument("--sparsity", type=float, default=0.0)
    p.add_argument("--out", default=None)
    a = p.parse_args()
    layer = model_layout(a.model)[:6]
    ws, st = [], {}
    for i, (name, r, c) in enumerate(layer):
        w, s = synth_ensemble(SynthSpec(rows=r, cols=c, name=name), 1000 + i)
        ws.append(w)
        st[w.name] = s
    sweep.alpha_sweep(ws, st, (0.5,), a.sparsity, calib_rows=8)  # warm (first launches, allocator)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = sweep.alpha_sweep(ws, st, sparsity=a.sparsity)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    for r in rows:
        print(json.dumps(r), flush=True)
    doc = {"model": a.model, "tensors": [f"{n} {r}x{c}" for n, r, c in layer], "sparsity": a.sparsity,
           "rows": rows, "gpu_seconds_all_alphas": gpu_s, "gpu_seconds_per_alpha": gpu_s / len(rows)}
    print(json.dumps({k: v for k, v in doc.items() if k != "rows"}))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
