"""Measurement sweeps for BASELINE configs C3 and C4 (writes JSON under profiles/).

  python tools/sweeps.py chunks  [--model opt-2.7b]   # C3: decode GB/s vs chunk size, fitted (D_max, c_sat)
  python tools/sweeps.py partial [--model opt-6.7b]   # C4: compressed fraction vs memory and tokens/s,
                                                      #     plus the speed-adaptive planner's choice
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15443_b200 import adaptive, container, synth  # noqa: E402
from paper_2502_15443_b200.gemm import FusedRing, GroupedInt8, MixedStep  # noqa: E402
from paper_2502_15443_b200.latency import CompressionPlan  # noqa: E402


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        return None


def cmd_chunks(a):
    t0 = time.time()
    curve = adaptive.measure_decode_curve(a.model, chunk_sizes=[int(x) for x in a.sizes.split(",")],
                                          layers=a.layers, seg_shift=8)
    int8 = a.int8_gbs
    mp = adaptive.b200_profile(curve, int8_weight_gbs=int8, hbm_gbs=hbm_peak())
    doc = json.loads(mp.to_json())
    doc.update({"config": "C3", "model": a.model, "layers": a.layers, "wall_s": time.time() - t0,
                "paper_fit_A40": {"D_max": 156.08, "c_sat": 76.72e6}})
    print(json.dumps(doc))
    return doc


def cmd_partial(a):
    t0 = time.time()
    m = synth.build_model(a.model, layers=a.layers)
    offs = m.offsets()[:-1]
    sizes = np.array([r * c for r, c in m.shapes], dtype=np.int64)
    w_views = [m.payload[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
    cs = a.chunk_size
    # per-layer CR estimate from a full pack (chunk stats mapped to layers)
    pm_all = synth.pack_model(m, cs, seg_shift=8)
    cr_all = pm_all.raw_bytes / pm_all.comp_bytes
    del pm_all
    points = []
    B = a.tokens
    gx = torch.Generator(device="cuda")
    gx.manual_seed(11)
    xs = [torch.randint(-127, 128, (B, c), generator=gx, device="cuda", dtype=torch.int8) for _, c in m.shapes]
    t_int8 = None
    for f in [i / 10 for i in range(11)]:
        mask = adaptive.plan_layers(sizes, np.full(len(sizes), cr_all), f)
        comp_idx = np.nonzero(mask)[0]
        plain_idx = np.nonzero(~mask)[0]
        mem = int(sizes[plain_idx].sum())
        fns = []
        checks = []
        gi = fc = None
        if len(plain_idx):
            gi = GroupedInt8([w_views[i] for i in plain_idx], [xs[i] for i in plain_idx], B)
            fns.append(gi.run)
        if len(comp_idx):
            sub = torch.cat([m.payload[offs[i]:offs[i] + sizes[i]] for i in comp_idx])
            sub_offs = np.concatenate([[0], np.cumsum(sizes[comp_idx])[:-1]])
            header = b"\0" * 8
            image, enc, entries = container.pack_device(sub, header, cs, None, seg_shift=8)
            jobs = container.jobs_for(entries, image.device)
            fc = FusedRing(image, jobs, enc.index, cs, [m.shapes[i] for i in comp_idx], sub_offs,
                                 [xs[i] for i in comp_idx], B)
            fns.append(fc.run)
            checks.append(fc)
            mem += int(entries["comp_len"].sum()) + enc.index.nbytes
        ms_seq = adaptive.time_ms(lambda: [fn() for fn in fns], iters=a.iters)
        for c in checks:
            if (c.check() != 0).any():
                raise SystemExit("fused chain check failed")
        split, ms = None, ms_seq
        if gi is not None and fc is not None:  # overlapped: fused on part of the SMs, INT8 GEMM on the rest
            ref = [x.clone() for x in gi.accs + fc.accs]
            mx = MixedStep(fc, gi)
            tries = mx.tune(iters=a.iters)
            split, ms = mx.fused_ctas, min(tries.values())
            mx.run()
            torch.cuda.synchronize()
            if (fc.check() != 0).any() or not all(torch.equal(x, y) for x, y in zip(ref, gi.accs + fc.accs)):
                raise SystemExit("overlapped step differs from the sequential one")
        if f == 0.0:
            t_int8 = ms
        points.append({"fraction": f, "layers_compressed": int(mask.sum()), "resident_bytes": mem,
                       "memory_vs_int8": mem / int(sizes.sum()), "step_ms": ms, "tokens_per_s": B / (ms / 1e3),
                       "vs_int8": t_int8 / ms if t_int8 else None, "sequential_step_ms": ms_seq,
                       "fused_sms": split})
        print(json.dumps(points[-1]), flush=True)
        fns.clear()
        torch.cuda.empty_cache()
    # the speed-adaptive planner on the measured profile (budget = INT8 step x slack)
    curve = json.load(open(a.curve))["curve"] if a.curve and os.path.exists(a.curve) else \
        adaptive.measure_decode_curve("opt-2.7b", layers=4)
    int8_gbs = int(sizes.sum()) / (t_int8 / 1e3) / 1e9
    mp = adaptive.b200_profile(curve, int8_weight_gbs=int8_gbs, hbm_gbs=hbm_peak())
    n_chunks = -(-int(sizes.sum()) // cs)
    plans = []
    for slack in (1.05, 1.25, 2.0, 5.0, 20.0):
        budget = slack * t_int8 / 1e3
        pr = adaptive.plan_for_budget(mp.profile, n_chunks, cs, cr_all, budget)
        plans.append({"budget_vs_int8": slack, "block_size": pr.plan.block_size,
                      "compressed_fraction": pr.plan.compressed_fraction, "feasible": pr.feasible,
                      "predicted_ms": pr.report.per_sample_latency * 1e3, "bottleneck": pr.report.bottleneck.value})
    doc = {"config": "C4", "model": a.model, "layers": a.layers, "tokens": B, "chunk_size": cs, "cr": cr_all,
           "points": points, "planner": plans, "profile": json.loads(mp.profile.to_json()),
           "wall_s": time.time() - t0}
    print(json.dumps(doc))
    return doc


def main():
    p = argparse.ArgumentParser()
    p.add_argument("cmd", choices=["chunks", "partial"])
    p.add_argument("--model", default=None)
    p.add_argument("--layers", type=int, default=None)
    p.add_argument("--sizes", default=",".join(str(x) for x in (16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20)))
    p.add_argument("--chunk-size", type=int, default=16 << 20)
    p.add_argument("--tokens", type=int, default=1)
    p.add_argument("--iters", type=int, default=10)
    p.add_argument("--int8-gbs", type=float, default=6200.0)
    p.add_argument("--curve", default=None)
    p.add_argument("--out", default=None)
    a = p.parse_args()
    if a.model is None:
        a.model = "opt-2.7b" if a.cmd == "chunks" else "opt-6.7b"
    doc = cmd_chunks(a) if a.cmd == "chunks" else cmd_partial(a)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
