"""bench.py contract on CPU: the reference arm prints one JSON line with the
keys the driver reads (small model, one layer)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--model", "opt-125m", "--layers", "1",
                        "--steps", "2", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["config"]["workload"]


def test_hash_weights_match_oracle_generator(oracle):
    """bench.py's two arms draw the same weights: the torch restatement of the
    integer-hash generator (GPU arm) equals the oracle's C one (reference arm)
    bit for bit, including indices past 2^26 and keys near 2^32."""
    import numpy as np

    from paper_2502_15443_b200 import synth
    for key in (0, 0x632BE5AB, 0xFFFFFFF0):
        for start, n in ((0, 4096), (70_000_000, 3000)):
            a = oracle.gen_weights(key, n, start)
            b = synth.hash_weights(key, start, n, "cpu").numpy()
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    w = oracle.gen_weights(7, 1 << 20)
    assert abs(w.std() - 0.2) < 0.002 and abs(w).max() < 1.0


def test_synth_spec_digest_shared():
    """Both arms build the workload from bench.synth_spec (same keys and
    channel maxima for the same seed)."""
    import importlib.util

    import numpy as np
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    a = bench.synth_spec("opt-125m", 1234, 1)
    b = bench.synth_spec("opt-125m", 1234, 1)
    assert a[0] == b[0] and a[1] == b[1] and all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))
    assert len(a[0]) == 6 and len(set(a[1])) == 6
