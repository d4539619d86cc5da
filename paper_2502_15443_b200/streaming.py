"""Host-resident weights streamed to the GPU every step (the reference's GPU_CPU
tier, latency.py:33 and :140-146).

The reference models a model too large for GPU memory: weights live in host
memory and cross PCIe once per forward pass, so a compressed chunk costs
S/cr on the link plus S/d_gpu(S) of decode, overlapped chunk by chunk
(``latency()``: per chunk max(load, dec, compute)).  This module runs that
pipeline for real on the B200:

* ``StreamedCompressed``: the DCC1 image sits in pinned host memory; each
  step copies chunk group g+1 over PCIe (copy stream) while group g is
  validated and decoded by the split-point decoder (compute stream), then the
  grouped tcgen05 W8A8 GEMM consumes the decoded weights.
* ``StreamedRaw``: the baseline -- raw INT8 weights in pinned host memory,
  copied every step, then the same GEMM.

Both keep one device copy of their input as the landing buffer (the
measurement is the per-step link + decode pipeline, which is what the
planner's GPU_CPU latency models; a rolling buffer of a few chunk groups
would bound device memory without changing the timing).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import engine
from . import native as nv
from .gemm import GroupedInt8


def _group_bounds(sizes: np.ndarray, groups: int) -> list[tuple[int, int]]:
    n = len(sizes)
    cuts = np.searchsorted(np.cumsum(sizes.astype(np.float64)),
                           np.linspace(0, float(sizes.sum()), groups + 1)[1:-1]).tolist()
    b = sorted(set([0] + [min(max(int(c), 0), n) for c in cuts] + [n]))
    return [(g0, g1) for g0, g1 in zip(b, b[1:]) if g1 > g0]


class StreamedCompressed:
    """Per-step PCIe streaming of a compressed container + on-GPU decode."""

    def __init__(self, host_image: torch.Tensor, jobs: engine.JobTable, index: engine.SegmentIndex,
                 groups: int = 16):
        if not host_image.is_pinned():
            raise ValueError("host_image must be pinned host memory")
        self.host, self.jobs, self.index = host_image, jobs, index
        dev = jobs.d_blob_off.device
        self.dev = dev
        self.image = nv.device_bytes(host_image.numel(), dev)
        self.out = nv.device_bytes(jobs.total_out, dev)
        self.status = torch.zeros(max(jobs.n, 1), dtype=torch.int32, device=dev)
        self.tasks = index.tasks(jobs, np.ones(jobs.n, bool))
        t_chunk = self.tasks[:, 0].cpu().numpy() if self.tasks.shape[0] else np.zeros(0, np.int32)
        ends = jobs.blob_off + jobs.blob_len
        self.groups = []
        for g0, g1 in _group_bounds(jobs.blob_len, groups):
            f0, f1 = int(jobs.blob_off[g0]), int(ends[g1 - 1])
            t0, t1 = int(np.searchsorted(t_chunk, g0)), int(np.searchsorted(t_chunk, g1))
            self.groups.append((g0, g1, f0, f1, t0, t1))
        self.s_copy = torch.cuda.Stream(dev)
        self.has_store = bool((jobs.codec == 0).any())
        self.bytes_per_step = int(host_image.numel())

    def step(self) -> None:
        j, ix = self.jobs, self.index
        s_comp = torch.cuda.current_stream(self.dev)
        s_copy = self.s_copy
        s_copy.wait_stream(s_comp)  # the previous step's decode is done reading the image
        sp = s_comp.cuda_stream
        for g0, g1, f0, f1, t0, t1 in self.groups:
            with torch.cuda.stream(s_copy):
                self.image[f0:f1].copy_(self.host[f0:f1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_copy)
            s_comp.wait_event(ev)
            k = g1 - g0
            off8 = lambda t: t.data_ptr() + 8 * g0  # noqa: E731
            nv.call("dc_ans_validate", self.image.data_ptr(), off8(j.d_blob_off), off8(j.d_blob_len),
                    off8(j.d_out_len), j.d_codec.data_ptr() + g0, k, self.status.data_ptr() + 4 * g0, sp)
            if t1 > t0:
                nv.call(engine.segment_kernel(j), self.image.data_ptr(), j.d_blob_off.data_ptr(),
                        j.d_blob_len.data_ptr(), j.d_out_off.data_ptr(), j.d_out_len.data_ptr(), ix.seg_shift,
                        ix.d_seg_base.data_ptr(), ix.d_state.data_ptr(), ix.d_off.data_ptr(),
                        self.tasks[t0:t1].data_ptr(), t1 - t0, self.out.data_ptr(), self.status.data_ptr(), sp)
            if self.has_store:
                nv.call("dc_store_copy", self.image.data_ptr(), off8(j.d_blob_off), off8(j.d_out_off),
                        off8(j.d_out_len), j.d_codec.data_ptr() + g0, k, self.out.data_ptr(), sp)

    def check(self) -> np.ndarray:
        return self.status[: self.jobs.n].cpu().numpy()


class StreamedRaw:
    """Baseline: raw INT8 weights in pinned host memory, copied every step."""

    def __init__(self, host_weights: torch.Tensor, device, groups: int = 16):
        if not host_weights.is_pinned():
            raise ValueError("host_weights must be pinned host memory")
        self.host = host_weights
        self.out = torch.empty(host_weights.numel(), dtype=torch.uint8, device=device)
        n = host_weights.numel()
        step = -(-n // groups)
        self.groups = [(a, min(n, a + step)) for a in range(0, n, step)]
        self.bytes_per_step = int(n)

    def step(self) -> None:
        for a, b in self.groups:
            self.out[a:b].copy_(self.host[a:b], non_blocking=True)


class StreamedFused:
    """Bounded-memory GPU_CPU tier: the compressed container stays in pinned
    host memory and every step streams it, group of layers by group, through
    a ring of ``slots`` device buffers; each group is consumed by the fused
    decode -> tcgen05 W8A8 kernel as soon as it lands (decoded weights never
    exist in HBM).  Device memory: the slots + the split-point index + the
    activations/accumulators -- the reference's buffer-chunk term of
    ``memory_footprint`` (latency.py:225-232) instead of the whole model.

    A group is a run of whole layers; its chunk span [c0, c1) is copied as one
    contiguous file range, and the group's FusedRing sees chunk-relative
    offsets (t_off - c0*chunk_size) and job/index arrays sliced at c0 with
    blob offsets rebased to its slot."""

    def __init__(self, host_image: torch.Tensor, jobs: engine.JobTable, index: engine.SegmentIndex,
                 chunk_size: int, shapes, t_offs, xs, ntok: int, slots: int = 3, group_bytes: int = 32 << 20):
        from .gemm import FusedRing
        if host_image is not None and not host_image.is_pinned():
            raise ValueError("host_image must be pinned host memory")
        self.host, self.slots = host_image, slots
        dev = index.d_state.device
        cs = int(chunk_size)
        ends = jobs.blob_off + jobs.blob_len
        spans = []  # (l0, l1, c0, c1)
        l0 = 0
        n = len(shapes)

        def span(a, b):
            c0 = int(t_offs[a]) // cs
            r, k = shapes[b - 1]
            c1 = (int(t_offs[b - 1]) + int(r) * int(k) - 1) // cs + 1
            return c0, c1

        while l0 < n:
            l1 = l0 + 1
            while l1 < n:
                c0, c1 = span(l0, l1 + 1)
                if int(ends[c1 - 1] - jobs.blob_off[c0]) > group_bytes:
                    break
                l1 += 1
            spans.append((l0, l1, *span(l0, l1)))
            l0 = l1
        self.slot_bytes = max(int(ends[c1 - 1] - jobs.blob_off[c0]) for _, _, c0, c1 in spans)
        self.ring = nv.device_bytes(slots * self.slot_bytes, dev)
        self.groups = []
        self.accs = []
        for g, (a, b, c0, c1) in enumerate(spans):
            f0, f1 = int(jobs.blob_off[c0]), int(ends[c1 - 1])
            slot = self.ring[(g % slots) * self.slot_bytes:(g % slots) * self.slot_bytes + (f1 - f0)]
            sub = engine.JobTable.build(jobs.blob_off[c0:c1] - np.uint64(f0), jobs.blob_len[c0:c1],
                                        jobs.out_off[c0:c1], jobs.out_len[c0:c1], jobs.codec[c0:c1], dev)
            six = engine.SegmentIndex(index.seg_shift, index.seg_base[c0:c1], index.n_segs,
                                      index.d_seg_base[c0:c1], index.d_state, index.d_off)
            fr = FusedRing(slot, sub, six, cs, shapes[a:b], [int(t) - c0 * cs for t in t_offs[a:b]], xs[a:b], ntok)
            self.groups.append((g % slots, f0, f1, fr))
            self.accs.extend(fr.accs)
        self.s_copy = torch.cuda.Stream(dev)
        self.ev_free = [None] * slots
        self.bytes_per_step = int(sum(f1 - f0 for _, f0, f1, _ in self.groups))
        self.device_bytes = int(self.ring.numel()) + 8 * index.n_segs

    def step(self) -> None:
        s_comp = torch.cuda.current_stream()
        for slot, f0, f1, fr in self.groups:
            with torch.cuda.stream(self.s_copy):
                if self.ev_free[slot] is not None:
                    self.s_copy.wait_event(self.ev_free[slot])  # the slot's previous group is decoded
                fr.image.copy_(self.host[f0:f1], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_copy)
            s_comp.wait_event(ev)
            fr.run()
            self.ev_free[slot] = torch.cuda.Event()
            self.ev_free[slot].record(s_comp)

    def check(self) -> bool:
        return all(not (fr.check() != 0).any() for _, _, _, fr in self.groups)


_PAGE = 4096


def _open(path: str, direct: bool) -> tuple[int, bool]:
    """Open for reading, O_DIRECT when asked and supported (tmpfs is not)."""
    if direct:
        try:
            return os.open(path, os.O_RDONLY | os.O_DIRECT), True
        except OSError:
            pass
    return os.open(path, os.O_RDONLY), False


def _read_range(fd: int, buf: torch.Tensor, f0: int, f1: int) -> int:
    """Read file bytes [f0, f1) into the page-aligned pinned ``buf`` starting at
    a page boundary (O_DIRECT needs aligned offset, size and address); returns
    the offset of f0 inside ``buf``."""
    a = f0 & ~(_PAGE - 1)
    b = (f1 + _PAGE - 1) & ~(_PAGE - 1)
    mv = memoryview(buf.numpy())[: b - a]
    got = 0
    while got < b - a:
        n = os.preadv(fd, [mv[got:]], a + got)
        if n <= 0:
            break
        got += n
    if got < f1 - a:
        raise OSError(f"short read at {a + got} (wanted through {f1})")
    return f0 - a


class StreamedFusedFile(StreamedFused):
    """GPU_DISK tier (the reference's storage -> CPU -> GPU path, B_stoc /
    B_ctog, latency.py:33-37): the container file stays on disk; every step
    reads each layer group's byte range (O_DIRECT by default, so the page
    cache does not stand in for the disk) into one of ``slots`` pinned host
    buffers on reader threads, copies it to a device slot and runs the fused
    decode -> GEMM on it.  Reads, H2D and decode of different groups overlap."""

    def __init__(self, path: str, jobs: engine.JobTable, index: engine.SegmentIndex, chunk_size: int, shapes,
                 t_offs, xs, ntok: int, slots: int = 4, group_bytes: int = 32 << 20, direct: bool = True,
                 threads: int = 4):
        from concurrent.futures import ThreadPoolExecutor
        super().__init__(None, jobs, index, chunk_size, shapes, t_offs, xs, ntok, slots, group_bytes)
        self.fd, self.direct = _open(path, direct)
        self.hslots = [torch.empty(self.slot_bytes + 2 * _PAGE, dtype=torch.uint8, pin_memory=True)
                       for _ in range(slots)]
        self.h2d_done = [None] * slots
        self.pool = ThreadPoolExecutor(max_workers=threads)

    def close(self) -> None:
        if getattr(self, "fd", None) is not None:
            self.pool.shutdown()
            os.close(self.fd)
            self.fd = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _read(self, g: int) -> int:
        slot, f0, f1, _ = self.groups[g]
        ev = self.h2d_done[slot]
        if ev is not None:
            ev.synchronize()  # the slot's previous H2D has read the pinned buffer
        return _read_range(self.fd, self.hslots[slot], f0, f1)

    def step(self) -> None:
        s_comp = torch.cuda.current_stream()
        G, S = len(self.groups), self.slots
        futs = {g: self.pool.submit(self._read, g) for g in range(min(S, G))}
        for g, (slot, f0, f1, fr) in enumerate(self.groups):
            off = futs.pop(g).result()
            with torch.cuda.stream(self.s_copy):
                if self.ev_free[slot] is not None:
                    self.s_copy.wait_event(self.ev_free[slot])
                fr.image.copy_(self.hslots[slot][off:off + (f1 - f0)], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_copy)
            self.h2d_done[slot] = ev
            s_comp.wait_event(ev)
            fr.run()
            self.ev_free[slot] = torch.cuda.Event()
            self.ev_free[slot].record(s_comp)
            if g + S < G:
                futs[g + S] = self.pool.submit(self._read, g + S)


class StreamedRawFile:
    """Baseline of the disk tier: raw INT8 weights read from a file every step
    (same reader threads / pinned slots / O_DIRECT), copied to the device
    weight buffer, then the grouped INT8 GEMM."""

    def __init__(self, path: str, nbytes: int, device, slots: int = 4, group_bytes: int = 64 << 20,
                 direct: bool = True, threads: int = 4):
        from concurrent.futures import ThreadPoolExecutor
        self.fd, self.direct = _open(path, direct)
        self.out = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.groups = [(a, min(nbytes, a + group_bytes)) for a in range(0, nbytes, group_bytes)]
        self.slots = slots
        self.hslots = [torch.empty(group_bytes + 2 * _PAGE, dtype=torch.uint8, pin_memory=True)
                       for _ in range(slots)]
        self.h2d_done = [None] * slots
        self.pool = ThreadPoolExecutor(max_workers=threads)
        self.s_copy = torch.cuda.Stream(device)
        self.bytes_per_step = nbytes

    def close(self) -> None:
        if getattr(self, "fd", None) is not None:
            self.pool.shutdown()
            os.close(self.fd)
            self.fd = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _read(self, g: int) -> int:
        slot = g % self.slots
        if self.h2d_done[slot] is not None:
            self.h2d_done[slot].synchronize()
        a, b = self.groups[g]
        return _read_range(self.fd, self.hslots[slot], a, b)

    def step(self) -> None:
        G, S = len(self.groups), self.slots
        # the previous step's GEMM (compute stream) must be done reading self.out
        # before this step's copies overwrite it (same rule as StreamedCompressed)
        self.s_copy.wait_stream(torch.cuda.current_stream())
        futs = {g: self.pool.submit(self._read, g) for g in range(min(S, G))}
        for g, (a, b) in enumerate(self.groups):
            off = futs.pop(g).result()
            slot = g % S
            with torch.cuda.stream(self.s_copy):
                self.out[a:b].copy_(self.hslots[slot][off:off + (b - a)], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_copy)
            self.h2d_done[slot] = ev
            if g + S < G:
                futs[g + S] = self.pool.submit(self._read, g + S)
        torch.cuda.current_stream().wait_stream(self.s_copy)


def measure_disk(model_payload: torch.Tensor, shapes, offs, image: torch.Tensor, jobs, index, ntok: int = 1,
                 iters: int = 3, workdir: str | None = None, direct: bool = True) -> dict:
    """Per-step time of the disk tier: raw INT8 file vs compressed DCC1 image
    file, each read every step (O_DIRECT), fused decode -> GEMM vs INT8 GEMM."""
    import tempfile
    from .adaptive import time_ms
    dev = model_payload.device
    workdir = workdir or tempfile.gettempdir()
    os.makedirs(workdir, exist_ok=True)
    raw_path = os.path.join(workdir, "dcomp_disk_raw.bin")
    img_path = os.path.join(workdir, "dcomp_disk_img.dcc")
    model_payload.cpu().numpy().tofile(raw_path)
    image.cpu().numpy().tofile(img_path)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    xs = [torch.randint(-127, 128, (ntok, c), generator=g, device=dev, dtype=torch.int8) for _, c in shapes]
    out = {"direct_io": direct}
    raw = StreamedRawFile(raw_path, model_payload.numel(), dev, direct=direct)
    gemm_raw = GroupedInt8(layer_views(raw.out, shapes, offs), xs, ntok)
    chunk = int(jobs.out_len.max())
    comp = StreamedFusedFile(img_path, jobs, index, chunk, shapes, offs, xs, ntok, direct=direct)
    try:
        raw.step()
        gemm_raw.run()
        comp.step()
        torch.cuda.synchronize()
        ok = comp.check() and all(torch.equal(a, b) for a, b in zip(gemm_raw.accs, comp.accs))
        t_raw = time_ms(lambda: (raw.step(), gemm_raw.run()), iters, warmup=1)
        t_comp = time_ms(comp.step, iters, warmup=1)
        out["direct_io"] = raw.direct and comp.direct
        out.update({"raw_step_ms": t_raw, "compressed_step_ms": t_comp, "speedup": t_raw / t_comp,
                    "raw_read_bytes": raw.bytes_per_step, "compressed_read_bytes": comp.bytes_per_step,
                    "raw_read_gbs": raw.bytes_per_step / t_raw / 1e6, "outputs_equal": ok,
                    "device_bytes_compressed": comp.device_bytes})
    finally:
        raw.close()
        comp.close()
        for p in (raw_path, img_path):
            try:
                os.remove(p)
            except OSError:
                pass
    return out


def layer_views(buf: torch.Tensor, shapes, offs) -> list[torch.Tensor]:
    return [buf[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, shapes)]


def measure(model_payload: torch.Tensor, shapes, offs, image: torch.Tensor, jobs, index, ntok: int = 1,
            iters: int = 5, groups: int = 16) -> dict:
    """Per-step time of raw vs compressed host streaming, each followed by the
    grouped W8A8 GEMM over every linear (CUDA events on the compute stream)."""
    from .adaptive import time_ms
    dev = model_payload.device
    host_raw = torch.empty(model_payload.numel(), dtype=torch.uint8, pin_memory=True)
    host_raw.copy_(model_payload)
    host_img = torch.empty(image.numel(), dtype=torch.uint8, pin_memory=True)
    host_img.copy_(image)
    raw = StreamedRaw(host_raw, dev, groups)
    comp = StreamedCompressed(host_img, jobs, index, groups)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    xs = [torch.randint(-127, 128, (ntok, c), generator=g, device=dev, dtype=torch.int8) for _, c in shapes]
    gemm_raw = GroupedInt8(layer_views(raw.out, shapes, offs), xs, ntok)
    gemm_comp = GroupedInt8(layer_views(comp.out, shapes, offs), xs, ntok)
    # correctness: the streamed, decoded weights are the model's weights
    comp.step()
    raw.step()
    torch.cuda.synchronize()
    if (comp.check() != 0).any() or not torch.equal(comp.out, model_payload) or not torch.equal(raw.out,
                                                                                               model_payload):
        raise RuntimeError("streamed weights differ from the model")
    t_raw = time_ms(lambda: (raw.step(), gemm_raw.run()), iters)
    t_comp = time_ms(lambda: (comp.step(), gemm_comp.run()), iters)
    gemm_raw.run()
    gemm_comp.run()
    torch.cuda.synchronize()
    same = all(torch.equal(a, b) for a, b in zip(gemm_raw.accs, gemm_comp.accs))
    out = {"raw_step_ms": t_raw, "compressed_step_ms": t_comp, "speedup": t_raw / t_comp,
           "raw_h2d_bytes": raw.bytes_per_step, "compressed_h2d_bytes": comp.bytes_per_step,
           "raw_tok_s": ntok / (t_raw / 1e3), "compressed_tok_s": ntok / (t_comp / 1e3), "ntok": ntok,
           "groups": groups, "outputs_equal": same,
           "device_bytes": {"raw": int(raw.out.numel()), "compressed": int(comp.image.numel() + comp.out.numel())}}
    del comp, gemm_comp
    # bounded memory: fused decode -> GEMM per streamed layer group, 3 device slots
    chunk = int(jobs.out_len.max())
    try:
        sf = StreamedFused(host_img, jobs, index, chunk, shapes, offs, xs, ntok)
        sf.step()
        torch.cuda.synchronize()
        ok = sf.check() and all(torch.equal(a, b) for a, b in zip(gemm_raw.accs, sf.accs))
        t_f = time_ms(sf.step, iters)
        out.update({"fused_bounded_step_ms": t_f, "fused_bounded_speedup": t_raw / t_f,
                    "fused_bounded_outputs_equal": ok, "fused_bounded_groups": len(sf.groups),
                    "fused_bounded_device_bytes": sf.device_bytes})
    except ValueError as e:  # chunking unsuitable for the fused path
        out["fused_bounded"] = f"skipped: {e}"
    return out
