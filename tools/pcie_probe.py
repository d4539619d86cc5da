"""PCIe copy-engine probe: D2H / H2D GB/s alone, split over k streams, and both directions at once.

    python tools/pcie_probe.py
"""
import torch


def run(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        for s in STREAMS:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


STREAMS = [torch.cuda.Stream() for _ in range(4)]


def main():
    n = 1 << 30
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
    for s in STREAMS:
        s.wait_stream(torch.cuda.current_stream())

    def split(dst, src, k):
        step = dst.numel() // k
        for i in range(k):
            with torch.cuda.stream(STREAMS[i]):
                dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)

    for k in (1, 2, 4):
        t = run(lambda: split(host, dev, k))
        print(f"D2H 1 GiB over {k} stream(s): {t:.2f} ms  {n / t / 1e6:.1f} GB/s", flush=True)
        t = run(lambda: split(dev, host, k))
        print(f"H2D 1 GiB over {k} stream(s): {t:.2f} ms  {n / t / 1e6:.1f} GB/s", flush=True)

    def both():
        with torch.cuda.stream(STREAMS[0]):
            host.copy_(dev, non_blocking=True)
        with torch.cuda.stream(STREAMS[1]):
            dev2.copy_(host2, non_blocking=True)
    t = run(both)
    print(f"D2H 1 GiB + H2D 0.5 GiB concurrently: {t:.2f} ms", flush=True)
    # pieces, as the pipeline issues them (75 MB D2H pieces)
    piece = 75 << 20

    def pieces():
        with torch.cuda.stream(STREAMS[0]):
            for o in range(0, n, piece):
                host[o:o + piece].copy_(dev[o:o + piece], non_blocking=True)
    t = run(pieces)
    print(f"D2H 1 GiB in 75 MiB pieces: {t:.2f} ms  {n / t / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()


def overlap_detail():
    """Per-direction finish times when D2H and H2D run together (and with an
    HBM-heavy kernel stream alongside)."""
    n = 1 << 30
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    host2 = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
    big_a = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
    big_b = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
    for with_kernel in (False, True):
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = torch.cuda.Event(enable_timing=True)
            e_d2h = torch.cuda.Event(enable_timing=True)
            e_h2d = torch.cuda.Event(enable_timing=True)
            t0.record()
            for s in STREAMS:
                s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(STREAMS[0]):
                host.copy_(dev, non_blocking=True)
                e_d2h.record()
            with torch.cuda.stream(STREAMS[1]):
                dev2.copy_(host2, non_blocking=True)
                e_h2d.record()
            if with_kernel:
                with torch.cuda.stream(STREAMS[2]):
                    for _ in range(20):
                        big_b.copy_(big_a)
            torch.cuda.synchronize()
        td, th = t0.elapsed_time(e_d2h), t0.elapsed_time(e_h2d)
        print(f"together (hbm kernel {with_kernel}): H2D 0.5 GiB done {th:.2f} ms ({n / 2 / th / 1e6:.1f} GB/s), "
              f"D2H 1 GiB done {td:.2f} ms", flush=True)


if __name__ == "__main__":
    overlap_detail()
