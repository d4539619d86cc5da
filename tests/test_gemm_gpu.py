"""tcgen05 W8A8 GEMM: exact int32 accumulators vs an int64 CPU product, and
simulate_layer vs the reference's f64 formula (scaling.py:127-152)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,N,K", [(1, 128, 128), (3, 200, 256), (16, 1024, 2048), (17, 384, 640),
                                   (32, 2048, 1024), (5, 130, 4096), (8, 77, 1000)])
def test_w8a8_exact(cuda, T, N, K):
    from paper_2502_15443_b200.gemm import w8a8_matmul_exact
    g = torch.Generator().manual_seed(T * 7919 + N * 13 + K)
    qx = torch.randint(-127, 128, (T, K), generator=g, dtype=torch.int8)
    qw = torch.randint(-127, 128, (N, K), generator=g, dtype=torch.int8)
    want = qx.long() @ qw.long().T
    got = w8a8_matmul_exact(qx.cuda(), qw.cuda()).cpu().long()
    assert torch.equal(got, want)


@pytest.mark.parametrize("kslice", [128, 256, 1024])
def test_w8a8_split_k_exact(cuda, kslice):
    from paper_2502_15443_b200.gemm import w8a8_gemm_into
    g = torch.Generator().manual_seed(kslice)
    qx = torch.randint(-128, 128, (16, 1024), generator=g, dtype=torch.int8).cuda()
    qw = torch.randint(-128, 128, (512, 1024), generator=g, dtype=torch.int8).cuda()
    acc = torch.empty((16, 512), dtype=torch.int32, device="cuda")
    w8a8_gemm_into(qx, qw, acc, kslice=kslice)
    assert torch.equal(acc.cpu().long(), qx.cpu().long() @ qw.cpu().long().T)


def test_simulate_layer_matches_reference_formula(cuda):
    rng = np.random.default_rng(5)
    for alpha in (0.0, 0.5, 1.0):
        w, st = cuda.synth_ensemble(cuda.SynthSpec(rows=96, cols=160), 17)
        x = rng.normal(0, 1, (8, 160)) * st.channel_max
        rep = cuda.simulate_layer(x, w, st, alpha)
        # reference arithmetic (scaling.py:139-152) in numpy f64
        sv = cuda.compute_scale(st, alpha)
        y = x @ w.values.T
        xs = x / sv.s[None, :]
        ws = w.values * sv.s[None, :]
        fp = np.linalg.norm(xs @ ws.T - y) / np.linalg.norm(y)
        qw = cuda.quantize(cuda.WeightTensor("w", ws))
        qx = cuda.quantize(cuda.WeightTensor("x", xs))
        yq = (qx.qvalues.astype(np.float64) * qx.w_scale) @ (qw.qvalues.astype(np.float64) * qw.w_scale).T
        qe = np.linalg.norm(yq - y) / np.linalg.norm(y)
        assert rep.fp_identity_error == pytest.approx(fp, rel=1e-6, abs=1e-15)
        assert rep.quantized_error == pytest.approx(qe, rel=1e-9)


def test_simulate_layer_equals_reference_golden(cuda):
    """simulate_layer (GPU quantize + tcgen05 W8A8, f64 references on the GPU)
    against reports the REFERENCE computed on the same seeded inputs
    (tests/golden/make_simulate_golden.py); only the f64 summation order
    differs, so the errors agree to 1e-9 relative."""
    import json
    import os

    import numpy as np
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "simulate.json")) as f:
        gold = json.load(f)
    for g in gold:
        w, st = cuda.synth_ensemble(cuda.SynthSpec(rows=g["rows"], cols=g["cols"], name=f"t{g['seed']}"),
                                    40 + g["seed"])
        x = np.random.default_rng([g["seed"], 7]).normal(0.0, 1.0, (g["batch"], g["cols"])) * st.channel_max[None, :]
        rep = cuda.simulate_layer(x, w, st, g["alpha"])
        assert rep.alpha == g["alpha"]
        # fp_identity_error is pure f64 round-off (~1e-16): absolute tolerance
        assert abs(rep.fp_identity_error - g["fp_identity_error"]) <= 1e-9 * g["fp_identity_error"] + 1e-14
        assert abs(rep.quantized_error - g["quantized_error"]) <= 1e-9 * g["quantized_error"]
