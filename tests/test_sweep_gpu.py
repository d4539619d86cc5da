"""GPU alpha sweep (dcomp sweep, cli.py:201-230): exact blob lengths and
near-zero fractions equal the oracle's on the same inputs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_alpha_sweep_matches_oracle(cuda, oracle):
    from paper_2502_15443_b200 import sweep
    from paper_2502_15443_b200.tensors import SynthSpec, synth_ensemble
    ws, st = [], {}
    for i, (r, c) in enumerate([(96, 128), (64, 256), (200, 64)]):
        w, s = synth_ensemble(SynthSpec(rows=r, cols=c, name=f"t{i}"), 100 + i)
        ws.append(w)
        st[w.name] = s
    alphas = (0.0, 0.5, 1.0)
    for sp, per_row in ((0.0, False), (0.3, False), (0.25, True)):
        rows = sweep.alpha_sweep(ws, st, alphas, sparsity=sp, per_row=per_row, calib_rows=8)
        for row, a in zip(rows, alphas):
            u = c = nz = 0
            for w in ws:
                cm = st[w.name].channel_max
                q, _ = oracle.quantize(w.values, oracle.compute_scale(cm, a))
                if sp > 0:
                    q = oracle.prune(q, cm, sp, per_row)
                u += q.size
                c += len(oracle.compress_blob(q.reshape(-1).view(np.uint8)))
                nz += int((np.abs(q.astype(np.int16)) <= 1).sum())
            assert row["raw_bytes"] == u and row["blob_bytes"] == c, (a, sp)
            assert row["near_zero"] == pytest.approx(nz / u, abs=0)
            assert np.isfinite(row["layer_error"]) and row["layer_error"] > 0
