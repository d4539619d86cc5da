"""Stage timeline of the public e2e call container.unpack(pinned file, index=pinned sidecar).

    DCOMP_TIMELINE=1 python tools/e2e_timeline.py [--model opt-1.3b] [--groups 16]

Prints host phase times and, per chunk group, when its H2D / decode / D2H
started and ended on the device (ms from PipelinedDecode construction).
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DCOMP_TIMELINE"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_15443_b200 import container, synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-1.3b")
    p.add_argument("--layers", type=int, default=None)
    p.add_argument("--reps", type=int, default=4)
    a = p.parse_args()
    m = synth.build_model(a.model, layers=a.layers)
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    host_file = pm.image.cpu().numpy().tobytes()
    side = pm.index.to_bytes(container.binding_of(host_file))
    pin_file = torch.empty(len(host_file), dtype=torch.uint8, pin_memory=True)
    pin_file.numpy()[:] = np.frombuffer(host_file, np.uint8)
    pin_side = torch.empty(len(side), dtype=torch.uint8, pin_memory=True)
    pin_side.numpy()[:] = np.frombuffer(side, np.uint8)
    for i in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        container.unpack(pin_file, index=pin_side)
        dt = time.perf_counter() - t0
        print(f"call {i}: {dt * 1e3:.2f} ms  {m.nbytes / dt / 1e9:.1f} GB/s  {container.LAST_UNPACK_MS}", flush=True)
    for name, h, d in container.LAST_UNPACK_TIMELINE:
        print(f"  {name:16s} host {h:8.3f}  dev {d:8.3f}")


if __name__ == "__main__":
    main()
