"""Tensor-parallel compressed-weight decode step (config C5), one process per GPU.

Each rank holds ITS shard of every linear (parallel.tp_layout) as a DCC1
container (GPU-encoded, with the split-point index) and as plain INT8 for the
baseline.  A step runs every local linear for ``ntok`` tokens in one grouped
launch (fused decode -> TMEM -> tcgen05, or the INT8 tcgen05 GEMM), then
all-reduces each row-parallel layer's int32 partial outputs over NCCL
(2 per transformer layer; exact integer sums).

``graph(compressed)`` captures that whole step -- the one grouped GEMM
launch and the row-parallel all-reduces (80 for LLaMA-13B) -- in ONE CUDA
graph, so a decode step is a single graph launch instead of ~80 eager NCCL
calls from Python.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import container, synth
from .gemm import FusedRing, GroupedInt8
from .parallel import tp_layout


class TPDecodeStep:
    def __init__(self, model: str, world: int, rank: int, ntok: int = 1, chunk_size: int = 16 << 20,
                 layers: int | None = None, alpha: float = 0.5, device=None):
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.shards = tp_layout(model, world, rank, layers)
        layout = [(s.name, *s.local_shape) for s in self.shards]
        self.model = synth.build_from_layout(model, layout, alpha, seed=4321 + rank, device=self.dev)
        m = self.model
        offs = m.offsets()[:-1]
        header = b"\0" * 8
        image, enc, entries = container.pack_device(m.payload, header, chunk_size, None, seg_shift=8)
        self.image, self.entries, self.index = image, entries, enc.index
        self.jobs = container.jobs_for(entries, image.device)
        g = torch.Generator(device=self.dev)
        g.manual_seed(99)
        # one activation per input: q/k/v read the same hidden state, as do gate/up
        shared = {}
        self.xs = []
        for s, (_, c) in zip(self.shards, m.shapes):
            layer, proj = s.name.rsplit(".", 1)
            key = (layer, "attn" if proj in ("q_proj", "k_proj", "v_proj") else
                   "mlp" if proj in ("gate_proj", "up_proj") else proj)
            if key not in shared:
                shared[key] = torch.randint(-127, 128, (ntok, c), generator=g, device=self.dev, dtype=torch.int8)
            self.xs.append(shared[key])
        w_views = [m.payload[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
        self.int8 = GroupedInt8(w_views, self.xs, ntok)
        self.fused = FusedRing(image, self.jobs, enc.index, chunk_size, m.shapes, offs, self.xs, ntok)
        self.row_idx = [i for i, s in enumerate(self.shards) if s.kind == "row"]
        self.raw_bytes = m.nbytes
        self.comp_bytes = int(entries["comp_len"].sum())

    def compute(self, compressed: bool) -> None:
        (self.fused if compressed else self.int8).run()

    def allreduce(self, compressed: bool) -> None:
        accs = (self.fused if compressed else self.int8).accs
        for i in self.row_idx:
            dist.all_reduce(accs[i], op=dist.ReduceOp.SUM)

    def step(self, compressed: bool) -> None:
        self.compute(compressed)
        self.allreduce(compressed)

    def graph(self, compressed: bool) -> torch.cuda.CUDAGraph:
        """The step captured in a CUDA graph (warmed up on a side stream first,
        as capture requires); replay() re-runs it on the same buffers."""
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            for _ in range(2):
                self.step(compressed)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(compressed)
        return g

    def check(self) -> bool:
        """Fused and INT8 paths give identical reduced outputs."""
        self.step(False)
        ref = [a.clone() for a in self.int8.accs]
        self.step(True)
        torch.cuda.synchronize()
        return bool((self.fused.check() == 0).all()) and all(torch.equal(a, b) for a, b in zip(ref, self.fused.accs))


def check_local(step: TPDecodeStep) -> bool:
    """Single-process check of one rank's shard: fused == INT8 partial outputs."""
    step.compute(False)
    ref = [a.clone() for a in step.int8.accs]
    step.compute(True)
    torch.cuda.synchronize()
    return bool((step.fused.check() == 0).all()) and all(torch.equal(a, b) for a, b in zip(ref, step.fused.accs))


def measure_local(step: TPDecodeStep, iters: int = 10) -> dict:
    """One rank's compute (no collective) timed alone -- the per-GPU work of a
    TP step when only one GPU is available; CUDA events."""
    def timed(fn):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    return {"int8_compute_ms": timed(lambda: step.compute(False)),
            "compressed_fused_compute_ms": timed(lambda: step.compute(True)),
            "allreduces_per_step": len(step.row_idx), "local_weight_bytes": step.raw_bytes,
            "local_file_bytes": step.comp_bytes}


def measure(step: TPDecodeStep, iters: int = 10) -> dict:
    """Max-over-ranks step times (CUDA events), compute vs all-reduce split."""
    def timed(fn):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=step.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {}
    for name, comp in (("int8", False), ("compressed_fused", True)):
        out[f"{name}_step_ms"] = timed(lambda: step.step(comp))
        out[f"{name}_compute_ms"] = timed(lambda: step.compute(comp))
        try:  # the whole step (GEMM launch + every all-reduce) as one CUDA graph
            g = step.graph(comp)
            out[f"{name}_graph_step_ms"] = timed(g.replay)
            del g
        except Exception as e:  # report, never hide
            out[f"{name}_graph_error"] = repr(e)[:200]
    out["allreduce_ms"] = timed(lambda: step.allreduce(True))
    out["allreduces_per_step"] = len(step.row_idx)
    out["local_weight_bytes"] = step.raw_bytes
    out["local_file_bytes"] = step.comp_bytes
    return out
