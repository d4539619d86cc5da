"""GPU parity of quantization and pruning against reference golden vectors
and the C oracle (bit-exact q, bit-exact f64 w_scale, identical zero sets)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_quantize_golden(cuda, golden):
    for c in golden["transforms"]["quantize"]:
        w = cuda.WeightTensor("g", np.array(c["w"], dtype=np.float64))
        if "cm" in c:
            qt = cuda.quantize_scaled(w, cuda.ActivationStats("g", np.array(c["cm"])), c["alpha"])
            assert np.array_equal(qt.scale_vec.s, np.array(c["s"]))
        else:
            qt = cuda.quantize(w)
        assert np.array_equal(qt.qvalues, np.array(c["q"], dtype=np.int8))
        assert qt.w_scale.hex() == c["w_scale"]


def test_quantize_matches_oracle_random(cuda, oracle):
    rng = np.random.default_rng(21)
    for _ in range(12):
        r, c = int(rng.integers(1, 300)), int(rng.integers(1, 3000))
        w, st = cuda.synth_ensemble(cuda.SynthSpec(rows=r, cols=c), int(rng.integers(0, 1 << 30)))
        alpha = float(rng.choice([0.0, 0.25, 0.5, 0.9, 1.0]))
        qt = cuda.quantize_scaled(w, st, alpha)
        q, ws = oracle.quantize(w.values, oracle.compute_scale(st.channel_max, alpha))
        assert np.array_equal(qt.qvalues, q) and qt.w_scale == ws
        assert qt.qvalues.min() >= -127


def test_quantize_errors(cuda):
    with pytest.raises(cuda.DcompError, match="zero dynamic range"):
        cuda.quantize(cuda.WeightTensor("z", np.zeros((3, 3))))
    with pytest.raises(cuda.DcompError, match="empty input"):
        cuda.quantize(cuda.WeightTensor("e", np.zeros((0, 3))))
    # max element maps to +-127 exactly; half-away rounding
    qt = cuda.quantize(cuda.WeightTensor("h", np.array([[1.0, -1.0, 0.0]])))
    assert qt.qvalues.tolist() == [[127, -127, 0]] and qt.w_scale == 1 / 127


def test_device_dtypes_match_f64(cuda):
    from paper_2502_15443_b200.scaling import quantize_device
    rng = np.random.default_rng(2)
    w32 = torch.from_numpy(rng.normal(0, 0.2, (257, 1031)).astype(np.float32)).cuda()
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        wd = w32.to(dt)
        q1, s1 = quantize_device(wd)
        q2, s2 = quantize_device(wd.to(torch.float64))
        assert torch.equal(q1, q2) and s1 == s2


def test_vector_path_half_integers_match_oracle(cuda, oracle):
    """The 8-column vector kernels (cols % 8 == 0) on every input dtype, with
    values placed on, just below and just above half-integers of w*s/w_scale,
    so the branch-free f32-product rounding hands those groups to the exact
    f64 path; q must equal the reference's rounding of the widened values."""
    from paper_2502_15443_b200.scaling import quantize_device
    rng = np.random.default_rng(77)
    rows, cols = 96, 256
    base = rng.integers(-126, 126, (rows, cols)).astype(np.float64)
    frac = rng.choice([0.5, 0.5 - 2 ** -14, 0.5 + 2 ** -14, 0.49999, 0.50001, 0.25, 0.0], (rows, cols))
    w = (base + np.sign(base + 0.1) * frac) / 127.0
    w[0, 0] = 1.0  # max |w| = 1 -> w_scale = 1/127
    for dt in (torch.float64, torch.float32, torch.bfloat16, torch.float16):
        wd = torch.from_numpy(w).to(dt).cuda()
        wide = wd.to(torch.float64).cpu().numpy()
        for s in (None, rng.uniform(0.5, 2.0, cols)):
            q, ws = quantize_device(wd, None if s is None else torch.from_numpy(s))
            qo, wso = oracle.quantize(wide, s)
            assert ws == wso, dt
            assert np.array_equal(q.cpu().numpy(), qo), (dt, s is None)


def test_dequantize_and_scale(cuda):
    rng = np.random.default_rng(8)
    w, st = cuda.synth_ensemble(cuda.SynthSpec(rows=64, cols=96), 3)
    qt = cuda.quantize_scaled(w, st, 0.5)
    dq = cuda.dequantize(qt)
    want = qt.qvalues.astype(np.float64) * qt.w_scale / qt.scale_vec.s[None, :]
    assert np.array_equal(dq.values, want)
    sw = cuda.scale_weights(w, qt.scale_vec)
    assert np.array_equal(sw.values, w.values * qt.scale_vec.s[None, :])
    del rng


def test_prune_golden(cuda, golden):
    for c in golden["transforms"]["prune"]:
        q = np.array(c["q"], dtype=np.int8)
        qt = cuda.QuantizedTensor("p", q, 0.1, cuda.ScaleVector.identity(q.shape[1]))
        st = cuda.ActivationStats("p", np.array(c["cm"]))
        scope = cuda.PruneScope.PER_ROW if c["per_row"] else cuda.PruneScope.PER_TENSOR
        out = cuda.prune(qt, st, cuda.PruneConfig(c["sparsity"], scope)).qvalues
        assert np.array_equal(out, np.array(c["out"], dtype=np.int8))


def test_prune_matches_oracle_random(cuda, oracle):
    rng = np.random.default_rng(33)
    for _ in range(16):
        r, c = int(rng.integers(1, 400)), int(rng.integers(1, 900))
        q = np.clip(np.round(rng.normal(0, float(rng.uniform(1, 40)), (r, c))), -127, 127).astype(np.int8)
        if rng.random() < 0.3:
            q[0, 0] = -128
        cm = rng.choice([0.0, 0.5, 1.0, 2.0, 3.0], c) if rng.random() < 0.5 else rng.lognormal(-1, 1, c)
        sp = float(rng.choice([0.0, 0.05, 0.2, 0.5, 0.999, 1.0]))
        per_row = bool(rng.random() < 0.4)
        qt = cuda.QuantizedTensor("p", q, 0.1, cuda.ScaleVector.identity(c))
        st = cuda.ActivationStats("p", cm)
        scope = cuda.PruneScope.PER_ROW if per_row else cuda.PruneScope.PER_TENSOR
        got = cuda.prune(qt, st, cuda.PruneConfig(sp, scope)).qvalues
        assert np.array_equal(got, oracle.prune(q, cm, sp, per_row)), (r, c, sp, per_row)
        if not per_row:
            newly = (got == 0) & (q != 0)
            assert (q == 0).sum() + newly.sum() >= int(np.floor(sp * q.size))


def test_prune_per_row_wide_rows_match_oracle(cuda, oracle):
    """Per-row selection on wide rows (the register path, up to 4096 columns):
    rows whose keys are all equal, rows dominated by ties, rows of distinct
    scores (the early exit when a bucket holds one key) -- zero sets equal the
    reference's stable-argsort result."""
    rng = np.random.default_rng(55)
    for cols, sp in ((4096, 0.2), (4000, 0.5), (3000, 0.01), (4096, 0.999)):
        rows = 24
        q = np.clip(np.round(rng.normal(0, 25, (rows, cols))), -127, 127).astype(np.int8)
        q[0, :] = 7                       # with constant cm: every key equal
        q[1, :] = rng.choice([-3, 3, 5], cols)  # heavy ties
        cm = rng.lognormal(-1, 1.5, cols)
        cm_const = np.full(cols, 0.75)
        for c_vec in (cm, cm_const):
            qt = cuda.QuantizedTensor("r", q, 0.1, cuda.ScaleVector.identity(cols))
            st = cuda.ActivationStats("r", c_vec)
            got = cuda.prune(qt, st, cuda.PruneConfig(sp, cuda.PruneScope.PER_ROW)).qvalues
            assert np.array_equal(got, oracle.prune(q, c_vec, sp, True)), (cols, sp)


def test_prune_per_tensor_ties_match_oracle(cuda, oracle):
    """Per-tensor selection where the k-th score is shared by many entries:
    constant cm (every column holds ties: the tie cut scans whole rows), a
    few cm levels, zero channel maxima (score-0 keys), 16-aligned and ragged
    widths (vector and scalar apply) -- zero sets equal the reference's."""
    rng = np.random.default_rng(66)
    for rows, cols in ((300, 1024), (257, 777), (64, 4096)):
        q = np.clip(np.round(rng.normal(0, 9, (rows, cols))), -127, 127).astype(np.int8)
        for cm in (np.full(cols, 0.75), rng.choice([0.0, 0.5, 1.0, 2.0], cols), rng.lognormal(-1, 1, cols)):
            for sp in (0.013, 0.2, 0.5, 0.93):
                qt = cuda.QuantizedTensor("t", q, 0.1, cuda.ScaleVector.identity(cols))
                st = cuda.ActivationStats("t", cm)
                got = cuda.prune(qt, st, cuda.PruneConfig(sp)).qvalues
                assert np.array_equal(got, oracle.prune(q, cm, sp, False)), (rows, cols, sp, cm[:3])


def test_prune_per_row_warp_kernel_shapes_match_oracle(cuda, oracle):
    """The warp-per-row kernel (16-aligned widths up to 4096, full and ragged
    512-column chunks) on continuous, few-level and constant channel maxima,
    zero columns, heavy ties and sparsities from 1/cols to 1: zero sets equal
    the reference's stable-argsort result."""
    rng = np.random.default_rng(88)
    for cols in (16, 48, 512, 1040, 2064, 4096):
        rows = 37
        q = np.clip(np.round(rng.normal(0, 12, (rows, cols))), -127, 127).astype(np.int8)
        q[0, :] = 5
        q[1, :] = rng.choice([-2, 2, 9], cols)
        q[2, : cols // 2] = 0
        for cm in (rng.lognormal(-1, 1, cols), rng.choice([0.0, 0.25, 1.0, 4.0], cols), np.full(cols, 0.3)):
            for sp in (1.0 / cols, 0.2, 0.5, 0.97, 1.0):
                qt = cuda.QuantizedTensor("r", q, 0.1, cuda.ScaleVector.identity(cols))
                st = cuda.ActivationStats("r", cm)
                got = cuda.prune(qt, st, cuda.PruneConfig(sp, cuda.PruneScope.PER_ROW)).qvalues
                assert np.array_equal(got, oracle.prune(q, cm, sp, True)), (cols, sp, cm[:2])


def test_prune_properties(cuda):
    rng = np.random.default_rng(44)
    q = np.clip(np.round(rng.normal(0, 20, (256, 512))), -127, 127).astype(np.int8)
    qt = cuda.QuantizedTensor("p", q, 0.1, cuda.ScaleVector.identity(512))
    st = cuda.ActivationStats("p", rng.lognormal(-1, 1, 512))
    a = cuda.prune(qt, st, cuda.PruneConfig(0.2))
    b = cuda.prune(a, st, cuda.PruneConfig(0.2))
    assert np.array_equal(a.qvalues, b.qvalues)  # idempotent
    c = cuda.prune(qt, st, cuda.PruneConfig(0.4))
    assert np.all((a.qvalues == 0) <= (c.qvalues == 0))  # nested zero sets


def test_prune_scores_reference_cases(cuda):
    """pruning.py:37-40 through dc_prune_scores, with the reference's own
    known answers (test_pruning.py:28-58) and an f64 numpy restatement."""
    dc = cuda

    def qt(vals, cm=None):
        v = np.asarray(vals, dtype=np.int8)
        cm = np.ones(v.shape[1]) if cm is None else np.asarray(cm, dtype=np.float64)
        return (dc.QuantizedTensor("t", v, 1.0, dc.ScaleVector.identity(v.shape[1])),
                dc.ActivationStats("t", cm))

    q, st = qt([[10, -10]], [1.0, 2.0])
    assert dc.prune_scores(q, st).tolist() == [[10.0, 20.0]]
    q, st = qt([[0, 5]], [100.0, 1.0])
    assert dc.prune_scores(q, st)[0, 0] == 0.0
    q, _ = qt([[1, 2]])
    with pytest.raises(dc.DcompError):
        dc.prune_scores(q, dc.ActivationStats("t", np.ones(3)))
    rng = np.random.default_rng(4)
    for r, c in [(6, 5), (33, 77), (512, 1024), (3, 4099)]:
        v = rng.integers(-127, 128, (r, c)).astype(np.int8)
        cm = rng.uniform(0.0, 3.0, c)
        q, st = qt(v, cm)
        got = dc.prune_scores(q, st)
        want = cm[None, :] * np.abs(v.astype(np.float64))
        assert got.dtype == np.float64 and np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_analyze_quantized_gpu_equals_reference(cuda):
    """analyze_quantized on the B200 (k_hist + report_from_histogram) equals
    the reference's reports (tests/golden/analyze.json), for host arrays,
    QuantizedTensors and int8 CUDA tensors alike."""
    import json
    import os
    import dataclasses
    import torch
    from conftest import GOLDEN
    from test_analyze_cpu import check_report, int8_cases
    with open(os.path.join(GOLDEN, "analyze.json")) as f:
        gold = json.load(f)["int8"]
    for name, v in int8_cases():
        check_report(dataclasses.asdict(cuda.analyze_quantized(v)), gold[name])
        check_report(dataclasses.asdict(cuda.analyze_quantized(torch.from_numpy(v).cuda())), gold[name])
        qt = cuda.QuantizedTensor(name, v, 1.0, cuda.ScaleVector.identity(v.shape[1]))
        check_report(dataclasses.asdict(cuda.analyze_quantized(qt)), gold[name])
    with pytest.raises(cuda.DcompError):
        cuda.analyze_quantized(np.zeros((0, 3), np.int8))


@pytest.mark.parametrize("shape", [(300, 264), (1500, 1000), (64, 4104), (1200, 2048)])
def test_column_max_absmax_equals_f64(cuda, shape):
    """f32 / bf16 / f16 absmax through the column-max pass (cols % 8 == 0):
    max|W*s| bit-equal to the f64 elementwise formula (max over columns of
    RN(max|W[:,c]| * s[c]) -- rounding is monotone), the max placed in
    different columns and rows, and the non-finite flag for inf and NaN."""
    from paper_2502_15443_b200.scaling import _absmax
    rng = np.random.default_rng(shape[1])
    rows, cols = shape
    s = torch.from_numpy(rng.uniform(0.05, 3.0, cols)).cuda()
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        for trial in range(3):
            w = torch.from_numpy(rng.normal(0, 0.2, (rows, cols)).astype(np.float32)).to(dt).cuda()
            r, c = int(rng.integers(rows)), int(rng.integers(cols))
            w[r, c] = -1.5 if trial == 1 else w[r, c]
            wide = w.to(torch.float64).cpu().numpy() * s.cpu().numpy()
            want = float(np.abs(wide).max())
            got, bad = _absmax(w, s)
            assert not bad and got == want, (dt, trial, got, want)
            got_f64, _ = _absmax(w.to(torch.float64), s)
            assert got_f64 == got
        for v in (float("inf"), float("nan"), float("-inf")):
            w2 = w.clone()
            w2[rows // 2, cols - 1] = v
            assert _absmax(w2, s)[1], (dt, v)
