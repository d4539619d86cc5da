"""Generate golden vectors by running the CPU REFERENCE itself.

Run in the dev container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes small fixtures next to this file.  Large cases are pinned by
SHA-256 digests of the reference's output bytes, with their inputs
regenerated deterministically from the reference's seeded generator
(`synth_ensemble`, tensors.py:154-171) -- the product reimplements the same
RNG call sequence, so the digests are reproducible on the GPU box.

Nothing on the GPU box runs this script; only its outputs travel.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

import numpy as np

import dcomp  # the reference
from dcomp import ans, container
from dcomp.errors import DcompError

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def codec_cases():
    rng = np.random.default_rng(2024)
    cases = []
    cases.append(np.array([0], np.uint8))
    cases.append(np.array([255], np.uint8))
    cases.append(np.array([7, 7, 7], np.uint8))
    cases.append(np.full(10_000, 9, np.uint8))
    cases.append(np.array([3, 9] * 51 + [3], np.uint8))
    z = np.zeros(100_000, np.uint8)
    z[0] = 255
    cases.append(z)
    cases.append(rng.integers(0, 256, 65_536).astype(np.uint8))  # incompressible
    for top in (2, 3, 16, 64, 200, 256):
        cases.append(rng.integers(0, top, int(rng.integers(1, 30_000))).astype(np.uint8))
    for scale in (0.3, 2.0, 6.0, 40.0):
        cases.append(np.clip(np.abs(rng.laplace(0, scale, 20_000)), 0, 255).astype(np.uint8))
    # int8 weight-like bytes (Gaussian quantized), sizes around chunk boundaries
    for n in (4095, 4096, 4097, 65_536, 131_072):
        cases.append(np.clip(np.round(rng.normal(0, 12, n)), -127, 127).astype(np.int8).view(np.uint8))
    for n in (1, 2, 5, 100, 1000):
        cases.append(rng.integers(0, 256, n).astype(np.uint8))
    return cases


def make_codec():
    cases = codec_cases()
    datas, blobs, freqs = [], [], []
    for d in cases:
        blob = ans.compress_blob(d)
        assert ans.decompress_blob(blob, d.size) == d.tobytes()
        datas.append(d)
        blobs.append(np.frombuffer(blob, np.uint8))
        freqs.append(ans.AnsTable.for_data(d).frequencies)
    # normalization-only cases (histograms straight into _normalize)
    rng = np.random.default_rng(77)
    hists = []
    for _ in range(200):
        h = np.zeros(256, np.int64)
        k = int(rng.integers(1, 257))
        idx = rng.choice(256, k, replace=False)
        h[idx] = rng.integers(1, int(rng.choice([3, 50, 10_000, 1 << 22])), k)
        hists.append(h)
    normed = [ans._normalize(h) for h in hists]
    np.savez_compressed(
        os.path.join(HERE, "codec.npz"),
        data=np.concatenate(datas), data_len=np.array([d.size for d in datas]),
        blob=np.concatenate(blobs), blob_len=np.array([b.size for b in blobs]),
        freq=np.stack(freqs), hist=np.stack(hists), normed=np.stack(normed),
    )


def corrupt_verdicts():
    """Reference verdicts for mutated blobs (ans.py:333-372)."""
    rng = np.random.default_rng(99)
    data = rng.integers(0, 40, 5000).astype(np.uint8)
    blob = ans.compress_blob(data)
    out = []
    muts = []
    for cut in (100, len(blob) - 1, len(blob) - 10, ans.TABLE_BYTES + 4):
        muts.append(("cut", cut, blob[:cut], data.size))
    for pos in rng.integers(ans.HEADER_BYTES, len(blob), 40):
        b = bytearray(blob)
        b[int(pos)] ^= 0xFF
        muts.append(("flip", int(pos), bytes(b), data.size))
    for pos in rng.integers(0, ans.TABLE_BYTES, 10):
        b = bytearray(blob)
        b[int(pos)] ^= 0x5A
        muts.append(("flip_table", int(pos), bytes(b), data.size))
    for st in (0xFFFF, 1 << 29, (1 << 20) + 1):
        b = bytearray(blob)
        b[ans.TABLE_BYTES:ans.TABLE_BYTES + 4] = struct.pack("<I", st)
        muts.append(("state", st, bytes(b), data.size))
    for wrong in (data.size - 1, data.size + 1, 1):
        muts.append(("outlen", wrong, blob, wrong))
    for kind, arg, b, n in muts:
        try:
            res = ans.decompress_blob(b, n)
            verdict = {"ok": True, "sha": sha(res)}
        except DcompError as e:
            verdict = {"ok": False, "cls": type(e).__name__, "msg": str(e)}
        out.append({"kind": kind, "arg": arg, "blob_hex": b.hex(), "out_len": n, "verdict": verdict})
    return {"data_hex": data.tobytes().hex(), "cases": out}


def small_model(seed=0, rows=64, cols=96):
    """Same construction as the reference's test fixture (test_container.py:25-33)."""
    rng = np.random.default_rng(seed)
    tensors, stats = [], {}
    for i, name in enumerate(("alpha", "beta", "gamma")):
        q = rng.integers(-30, 31, (rows + i, cols)).astype(np.int8)
        sv = dcomp.ScaleVector(0.5, np.exp(rng.normal(0, 0.2, cols)))
        tensors.append(dcomp.QuantizedTensor(name, q, float(rng.uniform(0.001, 0.1)), sv))
        stats[name] = dcomp.ActivationStats(name, np.abs(rng.normal(0, 1, cols)))
    return tensors, stats


def make_containers():
    meta = {}
    tensors, stats = small_model()
    total = sum(t.qvalues.size for t in tensors)
    n = -(-total // 4096)
    for bs in (0, 1, 2, 5):
        plan = dcomp.CompressionPlan.block_plan(4096, n, bs)
        blob = container.pack(tensors, stats, chunk_size=4096, plan=plan)
        with open(os.path.join(HERE, f"small_bs{bs}.dcc"), "wb") as f:
            f.write(blob)
        meta[f"small_bs{bs}"] = {"sha": sha(blob), "size": len(blob)}
    blob = container.pack([], {})
    meta["empty"] = {"hex": blob.hex()}
    # short last chunk
    tensors2, stats2 = small_model(rows=100, cols=41)
    blob = container.pack(tensors2, stats2, chunk_size=4096)
    with open(os.path.join(HERE, "small_short.dcc"), "wb") as f:
        f.write(blob)
    meta["small_short"] = {"sha": sha(blob), "size": len(blob)}
    return meta


OPT_SHAPES = {
    "opt-125m": (768, 3072, 12),
}


def model_shapes(model: str):
    h, ffn, L = OPT_SHAPES[model]
    out = []
    for l in range(L):
        for proj, r, c in (("q_proj", h, h), ("k_proj", h, h), ("v_proj", h, h), ("out_proj", h, h),
                           ("fc1", ffn, h), ("fc2", h, ffn)):
            out.append((f"layers.{l}.{proj}", r, c))
    return out


def make_model_digests():
    """C1 parity config: OPT-125M-shaped, alpha=0.5, per-tensor prune 0.2."""
    res = {}
    shapes = model_shapes("opt-125m")
    for alpha, sparsity in ((0.5, 0.2), (0.0, 0.0)):
        qts, stats = [], {}
        qdig = hashlib.sha256()
        wdig = []
        for i, (name, r, c) in enumerate(shapes):
            w, st = dcomp.synth_ensemble(dcomp.SynthSpec(rows=r, cols=c, name=name), 1000 + i)
            qt = dcomp.quantize_scaled(w, st, alpha)
            if sparsity:
                qt = dcomp.prune(qt, st, dcomp.PruneConfig(sparsity))
            qdig.update(qt.qvalues.tobytes())
            wdig.append(struct.pack("<d", qt.w_scale).hex())
            qts.append(qt)
            stats[name] = st
        key = f"opt125m_a{alpha}_p{sparsity}"
        res[key] = {"q_sha": qdig.hexdigest(), "w_scales": wdig, "containers": {}}
        for cs in (256 * 1024, 16 * 2**20):
            blob = container.pack(qts, stats, chunk_size=cs)
            res[key]["containers"][str(cs)] = {"sha": sha(blob), "size": len(blob),
                                                "cr": sum(t.qvalues.size for t in qts) / len(blob)}
        print(key, {k: v["cr"] for k, v in res[key]["containers"].items()}, file=sys.stderr)
    return res


def make_transforms():
    rng = np.random.default_rng(5150)
    qcases = []
    kat = [np.array([[1.0, -1.0, 0.0]]), np.array([[0.5, 1.0]]), np.array([[-0.5, 1.0]])]
    for w in kat:
        qt = dcomp.quantize(dcomp.WeightTensor("k", w))
        qcases.append({"w": w.tolist(), "s": None, "q": qt.qvalues.tolist(), "w_scale": qt.w_scale.hex()})
    for _ in range(12):
        r, c = int(rng.integers(1, 40)), int(rng.integers(1, 70))
        w, st = dcomp.synth_ensemble(dcomp.SynthSpec(rows=r, cols=c), int(rng.integers(0, 10_000)))
        alpha = float(rng.choice([0.0, 0.3, 0.5, 0.9, 1.0]))
        qt = dcomp.quantize_scaled(w, st, alpha)
        qcases.append({"w": w.values.tolist(), "cm": st.channel_max.tolist(), "alpha": alpha,
                       "s": qt.scale_vec.s.tolist(), "q": qt.qvalues.tolist(), "w_scale": qt.w_scale.hex()})
    # half-way rounding stress: values exactly at k+0.5 after division
    w = np.array([[127.0, 0.5, 1.5, -2.5, 126.5, -0.49999999999999994, 3.5000000000000004]])
    qt = dcomp.quantize(dcomp.WeightTensor("h", w))
    qcases.append({"w": w.tolist(), "s": None, "q": qt.qvalues.tolist(), "w_scale": qt.w_scale.hex()})

    pcases = []
    for _ in range(40):
        r, c = int(rng.integers(1, 24)), int(rng.integers(1, 40))
        q = rng.integers(-6, 7, (r, c)).astype(np.int8)
        cm = rng.choice([0.0, 0.5, 1.0, 2.0, 0.25], c) if rng.random() < 0.5 else rng.uniform(0, 3, c)
        sp = float(rng.choice([0.0, 0.1, 0.25, 0.5, 0.77, 1.0]))
        per_row = bool(rng.random() < 0.4)
        qt = dcomp.QuantizedTensor("p", q, 0.1, dcomp.ScaleVector.identity(c))
        st = dcomp.ActivationStats("p", cm)
        scope = dcomp.PruneScope.PER_ROW if per_row else dcomp.PruneScope.PER_TENSOR
        out = dcomp.prune(qt, st, dcomp.PruneConfig(sp, scope)).qvalues
        pcases.append({"q": q.tolist(), "cm": cm.tolist(), "sparsity": sp, "per_row": per_row,
                       "out": out.tolist()})
    return {"quantize": qcases, "prune": pcases}


def make_planner():
    L = sys.modules["dcomp.latency"]
    rng = np.random.default_rng(31337)
    cases = []
    for _ in range(60):
        h = L.HardwareProfile(
            B_stoc=float(rng.uniform(1, 10)), B_ctog=float(rng.uniform(5, 60)), B_gpu=float(rng.uniform(100, 8000)),
            D_max=float(rng.uniform(20, 4000)), c_sat=float(rng.uniform(1e5, 1e9)), I_gpu=float(rng.uniform(50, 8000)),
            mem_gpu=float(rng.uniform(1e9, 2e11)), mem_cpu=float(rng.uniform(1e9, 5e11)))
        n = int(rng.integers(1, 60))
        cs = int(rng.choice([16384, 1 << 20, 16 << 20]))
        cr = float(rng.uniform(1.0, 3.0))
        arch = list(L.Architecture)[int(rng.integers(0, 4))]
        bs = int(rng.integers(0, n + 1))
        plan = L.CompressionPlan.block_plan(cs, n, bs)
        rep = L.latency(h, plan, arch, np.where(plan.compressed_mask, cr, 1.0))
        full = L.latency(h, L.CompressionPlan.block_plan(cs, n, 1), arch, cr).per_sample_latency
        store = L.latency(h, L.CompressionPlan.block_plan(cs, n, 0), arch, 1.0).per_sample_latency
        budget = float(rng.uniform(min(full, store) * 0.8, max(full, store) * 1.2))
        pr = L.plan_partial(h, n, cs, cr, budget, arch)
        cases.append({"profile": json.loads(h.to_json()), "n": n, "cs": cs, "cr": cr, "arch": arch.value,
                      "bs": bs, "latency": rep.per_sample_latency, "bottleneck": rep.bottleneck.value,
                      "mem_gpu": rep.memory_used_gpu, "mem_cpu": rep.memory_used_cpu,
                      "stages": rep.stage_seconds, "budget": budget, "plan_bs": pr.plan.block_size,
                      "feasible": pr.feasible, "plan_latency": pr.report.per_sample_latency,
                      "footprint": L.memory_footprint(plan, np.where(plan.compressed_mask, cr, 1.0))})
    fit = L.fit_speed_curve([(48.05e6, 97.76), (75.08e6, 109.64), (192.13e6, 144.01), (300.16e6, 156.08)])
    return {"cases": cases, "fit_paper": list(fit)}


def main():
    make_codec()
    meta = {
        "corrupt": corrupt_verdicts(),
        "containers": make_containers(),
        "transforms": make_transforms(),
        "planner": make_planner(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f)
    with open(os.path.join(HERE, "model_digests.json"), "w") as f:
        json.dump(make_model_digests(), f, indent=1)


if __name__ == "__main__":
    main()
