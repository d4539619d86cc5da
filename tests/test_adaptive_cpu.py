"""Speed-adaptive planner on a B200-like measured profile (host logic only):
the reference's plan_partial fed by measured rates, and the per-layer mapping."""

import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _profile():
    from paper_2502_15443_b200 import adaptive
    curve = json.load(open(os.path.join(ROOT, "profiles", "r1_c3_chunks.json")))["curve"]
    return adaptive.b200_profile(curve, int8_weight_gbs=6200.0, hbm_gbs=6546.6, h2d_gbs=55.0, mem_gpu=180e9)


def test_profile_fit_from_measured_curve():
    mp = _profile()
    d_max, c_sat = mp.fit
    pts = {p["chunk_size"]: p["gbs"] for p in mp.curve}
    assert 0.9 * max(pts.values()) < d_max < 1.1 * max(pts.values())
    assert c_sat < 1 << 20  # split points: saturated well below 1 MiB chunks
    assert json.loads(mp.to_json())["profile"]["B_gpu"] == 6546.6


def test_budget_monotone_and_feasibility():
    from paper_2502_15443_b200 import adaptive
    h = _profile().profile
    cs, n, cr = 16 << 20, 384, 2.2
    none = adaptive.CompressionPlan.block_plan(cs, n, 0)
    t_raw = adaptive.predicted_step(h, none, 1.0)
    fracs = []
    for slack in (0.5, 1.0, 1.5, 3.0, 10.0, 100.0):
        pr = adaptive.plan_for_budget(h, n, cs, cr, slack * t_raw)
        assert pr.feasible == (slack >= 1.0)
        fracs.append(pr.plan.compressed_fraction)
        if pr.feasible:
            assert pr.report.per_sample_latency <= slack * t_raw * (1 + 1e-9)
    assert fracs == sorted(fracs) and fracs[-1] == 1.0  # looser budget -> more compressed


def test_plan_layers_nested_and_covering():
    from paper_2502_15443_b200 import adaptive
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 100, 40) * 4096
    crs = rng.uniform(1.5, 3.0, 40)
    prev = np.zeros(40, bool)
    for f in np.linspace(0, 1, 11):
        m = adaptive.plan_layers(sizes, crs, f)
        assert sizes[m].sum() >= f * sizes.sum() - 1e-6
        assert np.all(prev <= m)  # nested as the fraction grows
        if m.any() and (~m).any():
            assert crs[m].min() >= crs[~m].max()  # highest-CR layers first
        prev = m
