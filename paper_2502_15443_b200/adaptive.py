"""Speed-adaptive partial compression on B200 (north-star kernel 4).

The reference plans from an *illustrative* A40 profile (latency.py:78-87).
Here every HardwareProfile field the planner uses is measured on the GPU it
will run on:

  B_gpu   HBM copy bandwidth (MEASURED_PEAKS.json, or a device copy here)
  D_max,  fit_speed_curve() (the reference's own least-squares fit,
  c_sat   latency.py:279-292) over a measured decode-GB/s vs chunk-size sweep
  I_gpu   INT8 weight-streaming rate of the tcgen05 W8A8 GEMM
  B_ctog  pinned host -> device copy bandwidth

``plan_partial`` (unchanged reference algorithm) then picks the block plan,
and ``plan_layers`` turns a compressed fraction into a per-layer decision
(whole layers compressed, the largest-CR layers first) for engines that keep
uncompressed layers as plain INT8 tensors.
"""

from __future__ import annotations

import dataclasses
import json

import numpy as np
import torch

from .latency import Architecture, CompressionPlan, HardwareProfile, fit_speed_curve, latency, plan_partial


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_ms(fn, iters: int = 10, warmup: int = 2) -> float:
    for _ in range(warmup):
        fn()
    e0, e1 = _events()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def measure_h2d_gbs(nbytes: int = 1 << 30) -> float:
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ms = time_ms(lambda: dev.copy_(host, non_blocking=True), iters=5)
    return nbytes / (ms / 1e3) / 1e9


def measure_hbm_gbs(nbytes: int = 1 << 30) -> float:
    a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    ms = time_ms(lambda: b.copy_(a), iters=10)
    return 2 * nbytes / (ms / 1e3) / 1e9


def measure_decode_curve(model: str = "opt-2.7b", chunk_sizes=(16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20),
                         layers: int | None = 8, alpha: float = 0.5, seg_shift: int = 8, iters: int = 10):
    """Decode GB/s (decompressed) of a resident container at each chunk size."""
    from . import engine, synth
    m = synth.build_model(model, alpha=alpha, layers=layers)
    out = torch.empty_like(m.payload)
    pts = []
    for cs in chunk_sizes:
        pm = synth.pack_model(m, cs, seg_shift=seg_shift)
        st = torch.zeros(pm.jobs.n, dtype=torch.int32, device="cuda")
        has_store = bool((pm.entries["codec"] == 0).any())

        def step():
            engine.decode_segments(pm.image, pm.jobs, pm.index, pm.tasks, out, st)
            if has_store:
                engine.store_copy(pm.image, pm.jobs, out)

        ms = time_ms(step, iters)
        torch.cuda.synchronize()
        ok = bool(torch.equal(out, m.payload)) and int(st.abs().sum()) == 0
        pts.append({"chunk_size": cs, "gbs": pm.raw_bytes / (ms / 1e3) / 1e9, "ms": ms, "cr": pm.raw_bytes / pm.file_bytes,
                    "n_chunks": int(pm.jobs.n), "bit_exact": ok})
        del pm
    return pts


@dataclasses.dataclass
class MeasuredProfile:
    profile: HardwareProfile
    curve: list
    fit: tuple

    def to_json(self) -> str:
        return json.dumps({"profile": json.loads(self.profile.to_json()), "curve": self.curve,
                           "fit": {"D_max": self.fit[0], "c_sat": self.fit[1]}}, indent=1)


def b200_profile(curve, int8_weight_gbs: float, hbm_gbs: float | None = None, h2d_gbs: float | None = None,
                 storage_gbs: float = 7.0, mem_gpu: float | None = None) -> MeasuredProfile:
    """HardwareProfile from measurements (GB/s with GB = 1e9); rates not given
    are measured on the current GPU."""
    pts = [(p["chunk_size"], p["gbs"]) for p in curve]
    d_max, c_sat = fit_speed_curve(pts)
    if mem_gpu is None:
        mem_gpu = float(torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)
    import os
    host_mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    h = HardwareProfile(B_stoc=storage_gbs, B_ctog=h2d_gbs or measure_h2d_gbs(), B_gpu=hbm_gbs or measure_hbm_gbs(),
                        D_max=d_max, c_sat=c_sat, I_gpu=int8_weight_gbs, mem_gpu=float(mem_gpu),
                        mem_cpu=float(host_mem))
    return MeasuredProfile(h, curve, (d_max, c_sat))


def plan_for_budget(h: HardwareProfile, n_chunks: int, chunk_size: int, cr: float, budget_s: float,
                    arch: Architecture = Architecture.GPU_BUFFER):
    """The reference's planner on the measured profile (latency.py:244-276)."""
    return plan_partial(h, n_chunks, chunk_size, cr, budget_s, arch)


def plan_layers(layer_bytes, layer_cr, fraction: float) -> np.ndarray:
    """Per-layer keep-compressed decision for a target compressed fraction of
    the weight bytes: compress the layers that save the most memory per byte
    decoded (highest CR) first."""
    layer_bytes = np.asarray(layer_bytes, dtype=np.float64)
    layer_cr = np.asarray(layer_cr, dtype=np.float64)
    order = np.argsort(-layer_cr, kind="stable")
    want = fraction * layer_bytes.sum()
    mask = np.zeros(len(layer_bytes), dtype=bool)
    acc = 0.0
    for i in order:
        if acc >= want - 1e-9:
            break
        mask[i] = True
        acc += layer_bytes[i]
    return mask


def predicted_step(h: HardwareProfile, plan: CompressionPlan, cr: float) -> float:
    return latency(h, plan, Architecture.GPU_BUFFER, np.where(plan.compressed_mask, cr, 1.0)).per_sample_latency
