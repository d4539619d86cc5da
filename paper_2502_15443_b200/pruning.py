"""Activation-aware pruning of quantized weights (reference pruning.py API;
kernels in csrc/prune.cu).

Score of entry (r, c) is channel_max[c] * |q[r, c]|.  Exactly
floor(sparsity * n) lowest-scoring entries per scope are zeroed, ties
broken by row-major position, so the result equals a stable full sort --
computed on the GPU with a (column, |q|) histogram and a radix select
instead of a sort.
"""

from __future__ import annotations

import ctypes
import dataclasses
import enum
import math

import numpy as np
import torch

from . import native as nv
from .errors import DcompError
from .scaling import QuantizedTensor
from .tensors import ActivationStats


class PruneScope(enum.Enum):
    PER_TENSOR = "per_tensor"
    PER_ROW = "per_row"


@dataclasses.dataclass(frozen=True)
class PruneConfig:
    sparsity: float
    scope: PruneScope = PruneScope.PER_TENSOR

    def __post_init__(self):
        if not 0.0 <= self.sparsity <= 1.0:
            raise DcompError(f"sparsity must be in [0, 1], got {self.sparsity}")


def prune_scores(q: QuantizedTensor, stats: ActivationStats) -> np.ndarray:
    if len(stats.channel_max) != q.cols:
        raise DcompError(f"{q.name}: stats length {len(stats.channel_max)} != cols {q.cols}")
    dev = nv.require_cuda()
    dq = torch.from_numpy(np.ascontiguousarray(q.qvalues)).to(dev)
    cm = torch.from_numpy(np.ascontiguousarray(stats.channel_max, dtype=np.float64)).to(dev)
    out = torch.empty(q.qvalues.shape, dtype=torch.float64, device=dev)
    nv.call("dc_prune_scores", dq.data_ptr(), cm.data_ptr(), q.rows, q.cols, out.data_ptr(), nv.stream_ptr())
    return out.cpu().numpy()


def prune_device(q: torch.Tensor, cm: torch.Tensor, sparsity: float, per_row: bool = False,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """Prune a CUDA int8 tensor in one GPU pass (k from the same float
    arithmetic as the reference: floor(sparsity * n))."""
    rows, cols = q.shape
    q = q.contiguous()
    cm = cm.to(device=q.device, dtype=torch.float64).contiguous()
    out = out if out is not None else torch.empty_like(q)
    sp = nv.stream_ptr()
    if per_row:
        k = int(math.floor(sparsity * cols))
        nv.call("dc_prune_rows", q.data_ptr(), cm.data_ptr(), rows, cols, k, out.data_ptr(), sp)
    else:
        k = int(np.floor(sparsity * (rows * cols)))
        need = ctypes.c_uint64(0)
        nv.call("dc_prune_scratch_bytes", rows, cols, ctypes.byref(need))
        scratch = torch.empty(need.value, dtype=torch.uint8, device=q.device)
        nv.call("dc_prune_tensor", q.data_ptr(), cm.data_ptr(), rows, cols, k, out.data_ptr(),
                scratch.data_ptr(), sp)
    return out


def prune(q: QuantizedTensor, stats: ActivationStats, cfg: PruneConfig) -> QuantizedTensor:
    """Zero exactly floor(sparsity * n) lowest-scoring entries per scope.
    Other entries, w_scale and scale_vec are unchanged; idempotent."""
    if len(stats.channel_max) != q.cols:
        raise DcompError(f"{q.name}: stats length {len(stats.channel_max)} != cols {q.cols}")
    if q.qvalues.size == 0:
        return QuantizedTensor(q.name, q.qvalues.copy(), q.w_scale, q.scale_vec)
    dev = nv.require_cuda()
    dq = torch.from_numpy(np.ascontiguousarray(q.qvalues)).to(dev)
    cm = torch.from_numpy(stats.channel_max).to(dev)
    out = prune_device(dq, cm, cfg.sparsity, cfg.scope is PruneScope.PER_ROW)
    return QuantizedTensor(q.name, out.cpu().numpy(), q.w_scale, q.scale_vec)
