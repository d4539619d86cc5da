"""The bench workload is the same container in both arms: GPU hash weights +
GPU quantize + GPU pack give the bytes the oracle's C generator + quantize +
pack give (what bench.py --impl reference decodes)."""

import importlib.util
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_bench_container_identical_to_reference_arm(cuda, oracle):
    import torch

    from paper_2502_15443_b200 import synth
    bench = _bench()
    layout, keys, cms = bench.synth_spec("opt-125m", 1234, 1)
    m = synth.build_hash_model("opt-125m", layout, keys, cms, alpha=0.5, device=torch.device("cuda"))
    chunk = 1 << 20
    pm = synth.pack_model(m, chunk)
    ours = pm.image.cpu().numpy().tobytes()
    entries = []
    for (name, r, c), key, cm in zip(layout, keys, cms):
        s = oracle.compute_scale(cm, 0.5)
        q, ws = oracle.gen_quantize(key, r, c, s)
        entries.append((name, q, ws, 0.5, s, cm))
    ref = oracle.pack(entries, chunk, threads=4)
    assert bench.container_digest(ours) == bench.container_digest(ref)
    assert ours == ref
