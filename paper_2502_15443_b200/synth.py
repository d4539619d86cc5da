"""Device-side synthetic model builder for the benchmarks.

Large configs (OPT-1.3B .. LLaMA-13B) are far too big for the host numpy
generator in f64 (10-100 GB), so the bench draws the same distribution as
``SynthSpec`` (N(0, 0.2) clipped to +-1 weights, log-normal(-1, 1) channel
maxima with 2% outlier channels x20) with torch's CUDA generator, then
quantizes with the compression-aware scale (kernel 1) and packs with the
GPU encoder (kernel 2).  Parity of those kernels is established on the
reference's own generator in the tests; here only the shapes matter.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from . import container, engine
from .scaling import quantize_device
from .tensors import model_layout


@dataclasses.dataclass
class DeviceModel:
    model: str
    names: list[str]
    shapes: list[tuple[int, int]]
    payload: torch.Tensor       # uint8, concatenated int8 weights (row-major, exporter order)
    w_scales: list[float]
    s: list[torch.Tensor]       # f64 per-column scale vectors (device)
    cm: list[torch.Tensor]      # f64 channel maxima (device)
    alpha: float

    @property
    def nbytes(self) -> int:
        return int(self.payload.numel())

    def offsets(self) -> np.ndarray:
        sizes = np.array([r * c for r, c in self.shapes], dtype=np.int64)
        return np.concatenate([[0], np.cumsum(sizes)])


def build_model(model: str, alpha: float = 0.5, seed: int = 0, device=None, layers: int | None = None) -> DeviceModel:
    layout = model_layout(model)
    if layers is not None:
        per = sum(1 for n, _, _ in layout if n.startswith("layers.0."))
        layout = layout[: per * layers]
    return build_from_layout(model, layout, alpha, seed, device)


def build_from_layout(model: str, layout, alpha: float = 0.5, seed: int = 0, device=None) -> DeviceModel:
    """Random-init (SynthSpec distribution) weights of the given (name, rows,
    cols) list, compression-aware quantized on the GPU."""
    dev = device or torch.device("cuda")
    total = sum(r * c for _, r, c in layout)
    from .native import device_bytes
    payload = device_bytes(total, dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    names, shapes, scales, svec, cms = [], [], [], [], []
    pos = 0
    for name, r, c in layout:
        w = torch.randn((r, c), generator=g, device=dev, dtype=torch.float32).mul_(0.2).clamp_(-1.0, 1.0)
        cm = torch.exp(torch.randn(c, generator=g, device=dev, dtype=torch.float64) * 1.0 - 1.0)
        k = int(round(0.02 * c))
        if k:
            idx = torch.randperm(c, generator=g, device=dev)[:k]
            cm[idx] *= 20.0
        s = torch.clamp(cm, min=1e-8) ** alpha if alpha else torch.ones(c, dtype=torch.float64, device=dev)
        q = payload[pos:pos + r * c].view(torch.int8).view(r, c)
        _, ws = quantize_device(w, s, name, out=q)
        names.append(name)
        shapes.append((r, c))
        scales.append(ws)
        svec.append(s)
        cms.append(cm)
        pos += r * c
        del w
    return DeviceModel(model, names, shapes, payload, scales, svec, cms, alpha)


# ---- hash-generated weights (bench.py: both arms build identical containers) ----
GEN_SCALE = 4.315837287515549e-06   # 0.2 / (65536 * sqrt(6/12)): Irwin-Hall(6) ~ N(0, 0.2)
_M32 = 0xFFFFFFFF


def _fmix32(h: torch.Tensor) -> torch.Tensor:
    # uint32 arithmetic held in int64 (products wrap mod 2^64, the mask keeps the low word)
    h = h ^ (h >> 16)
    h = (h * 0x85EBCA6B) & _M32
    h = h ^ (h >> 13)
    h = (h * 0xC2B2AE35) & _M32
    return h ^ (h >> 16)


def hash_weights(key: int, start: int, n: int, device=None) -> torch.Tensor:
    """f64 weights [start, start+n) of the bench's integer-hash generator:
    u = sum of the six 16-bit halves of fmix32(key + 3j + t), t = 0..2, and
    w = (u - 196605) * GEN_SCALE.  Restated in C by oracle/dcomp_oracle.c
    (or_gen_weights) so the reference arm draws the same bytes on the host."""
    j = torch.arange(start, start + n, dtype=torch.int64, device=device)
    base = (j * 3 + (key & _M32)) & _M32
    u = torch.zeros(n, dtype=torch.int64, device=device)
    for t in range(3):
        h = _fmix32((base + t) & _M32)
        u += (h & 0xFFFF) + (h >> 16)
    return (u - 196605).to(torch.float64) * GEN_SCALE


def build_hash_model(model: str, layout, keys, cms, alpha: float = 0.5, device=None) -> DeviceModel:
    """Device model from hash weights (``keys[i]`` per tensor) and host f64
    channel maxima ``cms[i]``: s = compute_scale(cm, alpha) on the host (the
    reference's numpy pow), scale + quantize on the GPU (kernel 1)."""
    from .native import device_bytes
    from .scaling import compute_scale
    from .tensors import ActivationStats
    dev = device or torch.device("cuda")
    total = sum(r * c for _, r, c in layout)
    payload = device_bytes(total, dev)
    names, shapes, scales, svec, cmt = [], [], [], [], []
    pos = 0
    piece = 1 << 24
    for (name, r, c), key, cm in zip(layout, keys, cms):
        s_host = compute_scale(ActivationStats(name, np.asarray(cm, np.float64)), alpha).s
        s = torch.from_numpy(np.ascontiguousarray(s_host)).to(dev)
        w = torch.empty(r * c, dtype=torch.float64, device=dev)
        for a in range(0, r * c, piece):
            b = min(r * c, a + piece)
            w[a:b] = hash_weights(key, a, b - a, dev)
        q = payload[pos:pos + r * c].view(torch.int8).view(r, c)
        _, ws = quantize_device(w.view(r, c), s, name, out=q)
        del w
        names.append(name)
        shapes.append((r, c))
        scales.append(ws)
        svec.append(s)
        cmt.append(torch.from_numpy(np.ascontiguousarray(cm, dtype=np.float64)).to(dev))
        pos += r * c
    return DeviceModel(model, names, shapes, payload, scales, svec, cmt, alpha)


def header_for(m: DeviceModel, chunk_size: int) -> bytes:
    """DCC1 header body for a device model (f32 s / cm as the format stores)."""
    import struct
    import zlib
    parts = [struct.pack("<II", chunk_size, len(m.names))]
    for name, (r, c), ws, s, cm in zip(m.names, m.shapes, m.w_scales, m.s, m.cm):
        nb = name.encode()
        parts += [struct.pack("<H", len(nb)), nb, struct.pack("<IIdd", r, c, ws, m.alpha),
                  s.cpu().numpy().astype("<f4").tobytes(), cm.cpu().numpy().astype("<f4").tobytes()]
    body = b"".join(parts)
    return body + struct.pack("<I", zlib.crc32(body))


@dataclasses.dataclass
class PackedModel:
    image: torch.Tensor          # device DCC1 file image
    entries: np.ndarray
    jobs: engine.JobTable
    index: engine.SegmentIndex | None
    tasks: torch.Tensor | None
    chunk_size: int

    @property
    def file_bytes(self) -> int:
        return int(self.image.numel())

    @property
    def comp_bytes(self) -> int:
        return int(self.entries["comp_len"].sum())

    @property
    def raw_bytes(self) -> int:
        return int(self.entries["uncomp_len"].sum())


def pack_model(m: DeviceModel, chunk_size: int, plan=None, seg_shift: int = engine.DEFAULT_SEG_SHIFT) -> PackedModel:
    header = header_for(m, chunk_size)
    image, enc, entries = container.pack_device(m.payload, header, chunk_size, plan, seg_shift)
    jobs = container.jobs_for(entries, image.device)
    tasks = None
    if enc.index is not None:
        ok = np.ones(jobs.n, bool)
        tasks = enc.index.tasks(jobs, ok)
    return PackedModel(image, entries, jobs, enc.index, tasks, chunk_size)


def n_chunks(total: int, chunk_size: int) -> int:
    return math.ceil(total / chunk_size)
