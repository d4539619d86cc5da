"""Host profile of the drop-in quantize_scaled + prune calls at the C1 shape (OPT-125M).

    python tools/profile_quant_api.py
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_15443_b200 as dc  # noqa: E402
from paper_2502_15443_b200.tensors import model_layout  # noqa: E402

ws = [dc.synth_ensemble(dc.SynthSpec(rows=r, cols=c, name=n), 1000 + i) for i, (n, r, c) in enumerate(model_layout("opt-125m"))]


def run():
    return [dc.prune(dc.quantize_scaled(w, s, 0.5), s, dc.PruneConfig(0.2)) for w, s in ws]


run()
for _ in range(2):
    t = time.perf_counter()
    run()
    print(f"quantize_scaled + prune, 72 tensors: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
