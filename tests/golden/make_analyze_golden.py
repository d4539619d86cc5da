"""Golden analyze_quantized / analyze_float reports computed by the REFERENCE
(run here, where /root/reference is importable; the output is committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_analyze_golden.py

Inputs are regenerated from the seeds in the tests."""
import dataclasses
import json
import os

import numpy as np
from dcomp import WeightTensor, analyze_float, analyze_quantized

HERE = os.path.dirname(os.path.abspath(__file__))


def int8_cases():
    rng = np.random.default_rng(11)
    yield "gauss9", np.clip(np.round(rng.normal(0, 9, (300, 517))), -127, 127).astype(np.int8)
    yield "gauss2", np.clip(np.round(rng.normal(0, 2, (1024, 1024))), -127, 127).astype(np.int8)
    yield "uniform", rng.integers(-127, 128, (64, 4099)).astype(np.int8)
    yield "const", np.full((7, 9), -3, np.int8)
    yield "one", np.array([[5]], np.int8)
    yield "sparse", (rng.random((200, 300)) < 0.01).astype(np.int8) * 100
    yield "pm127", np.array([[127, -127, 0, 1, -1, 2]], np.int8)


def float_cases():
    rng = np.random.default_rng(12)
    yield "gauss", rng.normal(0, 0.2, (256, 384))
    yield "const", np.full((5, 5), 0.25)
    yield "heavy", rng.standard_t(3, (128, 1000)) * 0.05


out = {"int8": {k: dataclasses.asdict(analyze_quantized(v)) for k, v in int8_cases()},
       "float": {k: dataclasses.asdict(analyze_float(WeightTensor(k, v))) for k, v in float_cases()}}
with open(os.path.join(HERE, "analyze.json"), "w") as f:
    json.dump(out, f, indent=1)
