"""Grouped INT8 GEMM: wave kernel vs persistent kernel, and the persistent
kernel's weight GB/s as a function of the SMs it may use (per-SM bandwidth
decides how well it overlaps with the fused decode kernel).

    python tools/int8_scaling.py [--model opt-6.7b]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import adaptive, synth  # noqa: E402
from paper_2502_15443_b200.gemm import GroupedInt8  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-6.7b")
    p.add_argument("--ntok", type=int, default=1)
    p.add_argument("--out", default=None)
    a = p.parse_args()
    m = synth.build_model(a.model)
    offs = m.offsets()[:-1]
    ws = [m.payload[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    xs = [torch.randint(-127, 128, (a.ntok, c), generator=g, device="cuda", dtype=torch.int8) for _, c in m.shapes]
    gi = GroupedInt8(ws, xs, a.ntok)
    gi.run()
    ref = [x.clone() for x in gi.accs]
    gi.run(max_ctas=0)
    torch.cuda.synchronize()
    assert all(torch.equal(x, y) for x, y in zip(ref, gi.accs)), "persistent != wave kernel"
    out = {"model": a.model, "weight_bytes": m.nbytes}
    t = adaptive.time_ms(gi.run, iters=20)
    out["wave_ms"], out["wave_gbs"] = t, m.nbytes / t / 1e6
    rows = []
    for c in (16, 24, 32, 48, 64, 80, 96, 112, 128, 148):
        t = adaptive.time_ms(lambda: gi.run(max_ctas=c), iters=20)
        rows.append({"sms": c, "ms": t, "gbs": m.nbytes / t / 1e6, "gbs_per_sm": m.nbytes / t / 1e6 / c})
        print(json.dumps(rows[-1]), flush=True)
    out["persistent"] = rows
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
