"""Golden simulate_layer reports (W8A8 numerics, scaling.py:127-152) computed by
the REFERENCE (run here, where /root/reference is importable; output committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_simulate_golden.py
"""
import dataclasses
import json
import os

import numpy as np
from dcomp import SynthSpec, simulate_layer, synth_ensemble

HERE = os.path.dirname(os.path.abspath(__file__))
out = []
for seed, (r, c, b) in enumerate([(64, 96, 8), (256, 512, 16), (384, 128, 3)]):
    w, st = synth_ensemble(SynthSpec(rows=r, cols=c, name=f"t{seed}"), 40 + seed)
    x = np.random.default_rng([seed, 7]).normal(0.0, 1.0, (b, c)) * st.channel_max[None, :]
    for alpha in (0.0, 0.5, 0.9):
        rep = simulate_layer(x, w, st, alpha)
        out.append({"seed": seed, "rows": r, "cols": c, "batch": b, "alpha": alpha, **dataclasses.asdict(rep)})
with open(os.path.join(HERE, "simulate.json"), "w") as f:
    json.dump(out, f, indent=1)
