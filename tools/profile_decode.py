"""Run the resident split-point decode a few times (for ncu / timing runs).

    python tools/profile_decode.py --layers 4 --iters 5 [--seg-shift 9] [--chunk-size N]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import engine, synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-1.3b")
    p.add_argument("--layers", type=int, default=4)
    p.add_argument("--iters", type=int, default=5)
    p.add_argument("--seg-shift", type=int, default=8)
    p.add_argument("--chunk-size", type=int, default=16 * 2**20)
    a = p.parse_args()
    m = synth.build_model(a.model, layers=a.layers)
    pm = synth.pack_model(m, a.chunk_size, seg_shift=a.seg_shift)
    out = torch.empty_like(m.payload)
    st = torch.zeros(pm.jobs.n, dtype=torch.int32, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(a.iters):
        ev[0].record()
        engine.decode_segments(pm.image, pm.jobs, pm.index, pm.tasks, out, st)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1])
        ans = int(pm.entries["uncomp_len"][pm.entries["codec"] == 1].sum())
        print(f"iter {i}: {ms:.3f} ms  {ans / ms / 1e6:.1f} GB/s decompressed  tasks={pm.tasks.shape[0]}", flush=True)
    assert torch.equal(out, m.payload) and int(st.abs().sum()) == 0
    print("ok")


if __name__ == "__main__":
    main()
