"""analyze_quantized's report from a 256-bin histogram (the GPU path's host
half) equals the REFERENCE's analyze_quantized (golden reports written by
tests/golden/make_analyze_golden.py) -- integers exactly, floats to 1e-12 --
and the percentile restatement equals numpy.percentile bit for bit."""

import dataclasses
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2502_15443_b200.tensors import _percentile_linear, report_from_histogram


def int8_cases():
    rng = np.random.default_rng(11)
    yield "gauss9", np.clip(np.round(rng.normal(0, 9, (300, 517))), -127, 127).astype(np.int8)
    yield "gauss2", np.clip(np.round(rng.normal(0, 2, (1024, 1024))), -127, 127).astype(np.int8)
    yield "uniform", rng.integers(-127, 128, (64, 4099)).astype(np.int8)
    yield "const", np.full((7, 9), -3, np.int8)
    yield "one", np.array([[5]], np.int8)
    yield "sparse", (rng.random((200, 300)) < 0.01).astype(np.int8) * 100
    yield "pm127", np.array([[127, -127, 0, 1, -1, 2]], np.int8)


def check_report(got: dict, want: dict):
    for k, w in want.items():
        g = got[k]
        if isinstance(w, int) and not isinstance(w, bool):
            assert g == w, k
        else:
            assert g == pytest.approx(w, rel=1e-12, abs=0.0) or g == w, (k, g, w)


@pytest.mark.parametrize("name,v", list(int8_cases()))
def test_histogram_report_equals_reference(name, v):
    with open(os.path.join(GOLDEN, "analyze.json")) as f:
        want = json.load(f)["int8"][name]
    hist = np.bincount(v.reshape(-1).view(np.uint8), minlength=256)
    check_report(dataclasses.asdict(report_from_histogram(hist)), want)


def test_percentile_restatement_is_numpy():
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 4, 5, 7, 10, 101, 1000, 4099):
        for _ in range(20):
            mag = rng.integers(0, 129, n).astype(np.int16)
            counts = np.bincount(mag, minlength=129)
            vals = np.arange(129, dtype=np.int16)
            for q in (0.25, 0.75):
                want = float(np.percentile(mag, 100 * q))
                assert _percentile_linear(vals, counts, n, q) == want
