"""Host-side profile of the public e2e path container.unpack(host bytes, index=sidecar).

    python tools/profile_e2e.py [--model opt-1.3b] [--layers N]

Prints the unpack phase split and the top cProfile entries of one warm call.
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2502_15443_b200 import container, synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-1.3b")
    p.add_argument("--layers", type=int, default=None)
    a = p.parse_args()
    m = synth.build_model(a.model, layers=a.layers)
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    host_file = pm.image.cpu().numpy().tobytes()
    side = pm.index.to_bytes(container.binding_of(host_file))
    raw = m.nbytes
    import numpy as np
    pin_file = torch.empty(len(host_file), dtype=torch.uint8, pin_memory=True)
    pin_file.numpy()[:] = np.frombuffer(host_file, np.uint8)
    pin_side = torch.empty(len(side), dtype=torch.uint8, pin_memory=True)
    pin_side.numpy()[:] = np.frombuffer(side, np.uint8)
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        container.unpack(pin_file, index=pin_side)
        dt = time.perf_counter() - t0
        print(f"pinned call {i}: {dt * 1e3:.1f} ms  {raw / dt / 1e9:.1f} GB/s  phases {container.LAST_UNPACK_MS}",
              flush=True)
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        container.unpack(host_file, index=side)
        dt = time.perf_counter() - t0
        print(f"call {i}: {dt * 1e3:.1f} ms  {raw / dt / 1e9:.1f} GB/s  phases {container.LAST_UNPACK_MS}", flush=True)
    from paper_2502_15443_b200 import engine

    def t(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        print(f"  {name:24s} {(time.perf_counter() - t0) * 1e3:8.2f} ms", flush=True)
        return r

    for _ in range(2):
        _, _, ent, _ = t("_parse", lambda: container._parse(host_file))
        jobs = t("jobs_for", lambda: container.jobs_for(ent))
        b = t("binding_of", lambda: container.binding_of(host_file))
        ix = t("from_bytes", lambda: engine.SegmentIndex.from_bytes(side, jobs, b))
        t("tasks", lambda: ix.tasks(jobs, __import__("numpy").ones(jobs.n, bool)))
    import numpy as np

    from paper_2502_15443_b200 import native as nv
    src = np.frombuffer(host_file, np.uint8)
    stage = torch.empty(src.size, dtype=torch.uint8, pin_memory=True)
    dbuf = torch.empty(max(src.size, raw), dtype=torch.uint8, device="cuda")
    hout = torch.empty(raw, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        t("host memcpy -> pinned", lambda: nv._parallel_copy(stage.numpy(), src, piece=8 << 20))
        t(f"H2D {src.size >> 20} MiB", lambda: dbuf[: src.size].copy_(stage, non_blocking=True))
        t(f"D2H {raw >> 20} MiB", lambda: hout.copy_(dbuf[:raw], non_blocking=True))
        t("pipelined decode", lambda: engine.decode_file_pipelined(src, jobs, ix))
    pr = cProfile.Profile()
    pr.enable()
    container.unpack(host_file, index=side)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
    pstats.Stats(pr).sort_stats("tottime").print_stats(20)


if __name__ == "__main__":
    main()
