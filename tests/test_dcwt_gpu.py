"""DCWT ingest on the B200: device read == host read, GPU quantize from the
file == the reference's read + quantize (oracle), and the on-device
activation-stats hook == a CPU f64 max over the same activations
(exporter export.py:77-123)."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_read_weights_device_equals_host(cuda):
    for name in ("ref_f64", "ref_f32", "ref_i8"):
        path = os.path.join(GOLDEN, name + ".dcwt")
        host = cuda.dcwt.read_weights(path)
        dev = cuda.dcwt.read_weights_device(path)
        for h, (n, d) in zip(host, dev):
            assert h.name == n and np.array_equal(h.values, d.cpu().numpy().astype(np.float64))


@pytest.mark.parametrize("name", ["ref_f64", "ref_f32"])
def test_quantize_file_matches_reference_path(cuda, oracle, name):
    path = os.path.join(GOLDEN, name + ".dcwt")
    qts, stats = cuda.dcwt.quantize_file(path, os.path.join(GOLDEN, "ref_stats.json"), 0.5)
    for t, w in zip(qts, cuda.dcwt.read_weights(path)):  # reference: widen to f64 on the host, then quantize
        s = oracle.compute_scale(stats[t.name].channel_max, 0.5)
        q, ws = oracle.quantize(w.values, s)
        assert np.array_equal(t.qvalues, q) and t.w_scale == ws


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
def test_collect_activation_stats_device(cuda, dtype):
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(96, 256), torch.nn.GELU(), torch.nn.Linear(256, 64)).cuda().to(dtype)
    samples = [torch.randn(3, 17, 96, device="cuda", dtype=dtype) * (i + 1) for i in range(4)]
    samples[2][0, 0, 5] = -1e3  # a large negative activation: max|x| must catch it
    got = cuda.dcwt.collect_activation_stats(model, samples)
    want = {"0": None, "2": None}
    with torch.no_grad():
        for x in samples:
            h = model[1](model[0](x))
            for k, v in (("0", x), ("2", h)):
                m = v.double().abs().reshape(-1, v.shape[-1]).amax(0).cpu().numpy()
                want[k] = m if want[k] is None else np.maximum(want[k], m)
    assert set(got) == {"0", "2"}
    for k in got:
        assert np.array_equal(got[k], want[k])
    assert got["0"][5] == 1e3 if dtype == torch.float32 else got["0"][5] > 900


def test_export_then_quantize_roundtrip(cuda, oracle, tmp_path):
    torch.manual_seed(1)
    model = torch.nn.Sequential(torch.nn.Linear(128, 64), torch.nn.ReLU(), torch.nn.Linear(64, 32)).cuda()
    wp, sp = tmp_path / "m.dcwt", tmp_path / "m.json"
    names = cuda.dcwt.export_weights(model, wp)
    assert [n["name"] for n in names] == ["0", "2"]
    cuda.dcwt.collect_activation_stats(model, [torch.randn(8, 128, device="cuda")], out_path=sp)
    qts, stats = cuda.dcwt.quantize_file(wp, sp, 0.5)
    for t, mod in zip(qts, (model[0], model[2])):
        w = mod.weight.detach().float().cpu().numpy().astype(np.float64)
        q, ws = oracle.quantize(w, oracle.compute_scale(stats[t.name].channel_max, 0.5))
        assert np.array_equal(t.qvalues, q) and t.w_scale == ws
