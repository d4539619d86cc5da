"""GPU_DISK tier measurement: raw INT8 vs compressed DCC1 read from disk every step.

    python tools/disk_tier.py [--model opt-1.3b] [--workdir DIR] [--buffered]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_15443_b200 import streaming, synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--model", default="opt-1.3b")
    p.add_argument("--workdir", default=None)
    p.add_argument("--buffered", action="store_true")
    p.add_argument("--out", default=None)
    a = p.parse_args()
    m = synth.build_model(a.model)
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    r = streaming.measure_disk(m.payload, m.shapes, m.offsets()[:-1], pm.image, pm.jobs, pm.index, ntok=1,
                               iters=3, workdir=a.workdir, direct=not a.buffered)
    r["model"] = a.model
    print(json.dumps(r))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(r, f, indent=1)


if __name__ == "__main__":
    main()
