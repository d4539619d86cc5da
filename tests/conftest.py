import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long-running GPU case")
    config.addinivalue_line("markers", "perf: opt-in timing comparison (DCOMP_PERF=1)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def codec_golden():
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def model_digests():
    with open(os.path.join(GOLDEN, "model_digests.json")) as f:
        return json.load(f)


def split_concat(flat, lens):
    out, pos = [], 0
    for n in lens:
        out.append(flat[pos:pos + int(n)])
        pos += int(n)
    return out


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.lib()
    return o


@pytest.fixture(scope="session")
def cuda():
    """The CUDA product library; GPU tests only."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_15443_b200 as dc
    dc.native.lib()  # fails loudly if the extension is missing
    return dc
