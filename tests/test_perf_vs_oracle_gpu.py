"""Opt-in timing comparisons against the CPU oracle (the reference algorithm on
the host's cores), each also asserting bit-exactness.  Skipped unless
DCOMP_PERF=1; results go to $DCOMP_PERF_OUT (default gpurun_out/) as JSON.

    DCOMP_PERF=1 python -m pytest tests/test_perf_vs_oracle_gpu.py -s

The oracle is the checker and the CPU comparator here, never the product path.
"""
import json
import os
import time

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(os.environ.get("DCOMP_PERF") != "1",
                                                  reason="timing comparison: set DCOMP_PERF=1")]


def _save(name, doc):
    out = os.environ.get("DCOMP_PERF_OUT", "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, name), "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc))


def _sync():
    import torch
    torch.cuda.synchronize()


def test_c1_pipeline_vs_oracle(cuda, oracle):
    """SURVEY 8d C1 (OPT-125M, alpha 0.5, per-tensor prune 0.2, 256 KiB chunks):
    quantize + prune + pack + unpack through the drop-in API on the GPU vs the
    oracle's same four steps (all host threads for pack/unpack)."""
    from paper_2502_15443_b200.tensors import model_layout
    layout = model_layout("opt-125m")
    ws = [cuda.synth_ensemble(cuda.SynthSpec(rows=r, cols=c, name=n), 1000 + i) for i, (n, r, c) in enumerate(layout)]
    cs, alpha, sp = 256 << 10, 0.5, 0.2
    t = {"quantize_prune": [], "pack": [], "unpack": []}
    for _ in range(4):  # the first pass warms allocators, pinned pools and kernel attributes
        _sync()
        t0 = time.perf_counter()
        qts, stats = [], {}
        for w, s in ws:
            qts.append(cuda.prune(cuda.quantize_scaled(w, s, alpha), s, cuda.PruneConfig(sp)))
            stats[s.name] = s
        t["quantize_prune"].append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        blob = cuda.pack(qts, stats, chunk_size=cs)
        t["pack"].append(time.perf_counter() - t0)
        cuda.container.clear_index_cache()  # time the reference's call as a first call (serial chains)
        t0 = time.perf_counter()
        back = cuda.unpack(blob)
        t["unpack"].append(time.perf_counter() - t0)
    t = {k: min(v[1:]) for k, v in t.items()}  # best warm pass per stage
    threads = os.cpu_count() or 1
    c = {}
    t0 = time.perf_counter()
    ents = []
    for (w, s) in ws:
        sv = oracle.compute_scale(s.channel_max, alpha)
        q, wsc = oracle.quantize(w.values, sv)
        q = oracle.prune(q, s.channel_max, sp, False)
        ents.append((w.name, q, wsc, alpha, sv, s.channel_max))
    c["quantize_prune"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref = oracle.pack(ents, cs, threads=threads)
    c["pack"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.unpack(ref, threads=threads)
    c["unpack"] = time.perf_counter() - t0
    assert blob == ref
    assert all(np.array_equal(a.qvalues, b.qvalues) for a, b in zip(qts, back.tensors))
    raw = sum(q.qvalues.size for q in qts)
    _save("c1_pipeline.json", {"config": "C1 opt-125m alpha 0.5 prune 0.2 per-tensor, 256 KiB chunks",
                               "raw_bytes": raw, "file_bytes": len(blob), "cr": raw / len(blob),
                               "gpu_seconds": t, "gpu_total_s": sum(t.values()),
                               "oracle_seconds": c, "oracle_total_s": sum(c.values()), "oracle_threads": threads,
                               "bytes_identical": True})


def test_pack_api_vs_oracle(cuda, oracle):
    """container.pack on the GPU vs the oracle's pack (all host threads), OPT-1.3B
    shape (one synthetic layer tiled over every layer), 16 MiB chunks."""
    from paper_2502_15443_b200.tensors import model_layout
    full = model_layout("opt-1.3b")
    layer = full[:6]
    made = []
    for i, (name, r, c) in enumerate(layer):
        w, st = cuda.synth_ensemble(cuda.SynthSpec(rows=r, cols=c, name=name), 1000 + i)
        qt = cuda.quantize_scaled(w, st, 0.5)
        made.append((qt, st.channel_max))
    tensors, stats, ents = [], {}, []
    for L in range(len(full) // 6):
        for (name, _, _), (qt, cm) in zip(layer, made):
            nm = f"layers.{L}.{name.split('.')[-1]}"
            tensors.append(cuda.QuantizedTensor(nm, qt.qvalues, qt.w_scale, qt.scale_vec))
            stats[nm] = cuda.ActivationStats(nm, cm)
            ents.append((nm, qt.qvalues, qt.w_scale, 0.5, qt.scale_vec.s, cm))
    raw = sum(t.qvalues.size for t in tensors)
    gpu = []
    for _ in range(3):
        t0 = time.perf_counter()
        data = cuda.pack(tensors, stats)
        gpu.append(time.perf_counter() - t0)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    ref = oracle.pack(ents, 16 << 20, threads=threads)
    cpu = time.perf_counter() - t0
    assert ref == data
    _save("pack_api.json", {"model": "opt-1.3b", "raw_bytes": raw, "gpu_seconds": min(gpu), "gpu_gbs": raw / min(gpu) / 1e9,
                            "oracle_seconds": cpu, "oracle_threads": threads, "bytes_identical": True})


def test_alpha_sweep_vs_oracle(cuda, oracle):
    """dcomp sweep on one OPT-1.3B layer: GPU alpha sweep (all 11 alphas) vs the
    oracle's quantize + compress per alpha; CR identical."""
    import torch
    from paper_2502_15443_b200 import sweep
    from paper_2502_15443_b200.tensors import model_layout
    layer = model_layout("opt-1.3b")[:6]
    ws, st = [], {}
    for i, (name, r, c) in enumerate(layer):
        w, s = cuda.synth_ensemble(cuda.SynthSpec(rows=r, cols=c, name=name), 1000 + i)
        ws.append(w)
        st[w.name] = s
    sweep.alpha_sweep(ws, st, (0.5,), 0.0, calib_rows=8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = sweep.alpha_sweep(ws, st, sparsity=0.0)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    for alpha in (0.0, 0.5):
        u = c = 0
        for w in ws:
            q, _ = oracle.quantize(w.values, oracle.compute_scale(st[w.name].channel_max, alpha))
            u += q.size
            c += len(oracle.compress_blob(q.reshape(-1).view(np.uint8)))
        g = next(r for r in rows if r["alpha"] == alpha)
        assert g["cr"] == u / c
    cpu_s = (time.perf_counter() - t0) / 2
    _save("alpha_sweep_vs_oracle.json", {"model": "opt-1.3b", "layer_tensors": len(ws), "alphas": len(rows),
                                         "gpu_seconds_all_alphas": gpu_s,
                                         "oracle_seconds_per_alpha_quantize_compress": cpu_s,
                                         "cr_identical": True})
