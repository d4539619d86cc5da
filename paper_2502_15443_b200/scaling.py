"""Compression-aware scaling and symmetric INT8 quantization (reference
scaling.py API; kernels in csrc/quant.cu).

Column c of W is multiplied by s_c = max(channel_max[c], 1e-8) ** alpha
before per-tensor absmax quantization; activations are divided by s_c at
run time, so X @ W.T is unchanged while most weight columns shrink -- which
is what makes the entropy coder win.

``compute_scale`` stays host numpy on purpose: libm pow and CUDA pow may
differ by an ulp, and s must be bit-identical to the reference.  The f64
multiply, absmax, IEEE division and half-away-from-zero rounding run on the
GPU (``quantize_device`` is the device-tensor entry point).
"""

from __future__ import annotations

import ctypes
import dataclasses
import struct

import numpy as np
import torch

from . import native as nv
from .errors import DcompError
from .tensors import ActivationStats, WeightTensor

EPS_SCALE = 1e-8
ALPHA_GRID = tuple(round(0.1 * i, 1) for i in range(11))

_DTYPE_CODE = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2, torch.float16: 3}


def compute_scale(stats: ActivationStats, alpha: float) -> ScaleVector:
    """s_i = max(channel_max_i, 1e-8) ** alpha; alpha = 0 is the identity."""
    if not 0.0 <= alpha <= 1.0:
        raise DcompError(f"alpha must be in [0, 1], got {alpha}")
    if alpha == 0.0:
        return ScaleVector.identity(len(stats.channel_max))
    return ScaleVector(alpha, np.maximum(stats.channel_max, EPS_SCALE) ** alpha)


# ------------------------------------------------------------- device API
def _absmax(w: torch.Tensor, s: torch.Tensor | None) -> tuple[float, bool]:
    rows, cols = w.shape
    bits = torch.empty(1, dtype=torch.int64, device=w.device)
    flag = torch.empty(1, dtype=torch.int32, device=w.device)
    nv.call("dc_quant_absmax", w.data_ptr(), _DTYPE_CODE[w.dtype], nv.ptr(s), rows, cols, bits.data_ptr(),
            flag.data_ptr(), nv.stream_ptr())
    m = struct.unpack("<d", struct.pack("<q", int(bits.item())))[0]
    return m, bool(flag.item())


def quantize_device(w: torch.Tensor, s: torch.Tensor | None = None, name: str = "w",
                    out: torch.Tensor | None = None) -> tuple[torch.Tensor, float]:
    """Quantize a CUDA weight tensor (f64/f32/bf16/f16), optionally scaled by
    the f64 column vector ``s``.  Returns (int8 device tensor, w_scale)."""
    if w.dim() != 2:
        raise DcompError(f"{name}: expected a 2-D tensor")
    w = w.contiguous()
    if w.numel() == 0:
        raise DcompError(f"{name}: empty input")
    if s is not None:
        s = s.to(device=w.device, dtype=torch.float64).contiguous()
    m, nonfinite = _absmax(w, s)
    if nonfinite:
        raise ValueError(f"{name}: non-finite values")
    if m == 0.0:
        raise DcompError(f"{name}: zero dynamic range")
    w_scale = m / 127.0  # scaling.py:102, host f64 like the reference
    q = out if out is not None else torch.empty(w.shape, dtype=torch.int8, device=w.device)
    nv.call("dc_quantize", w.data_ptr(), _DTYPE_CODE[w.dtype], nv.ptr(s), w.shape[0], w.shape[1],
            ctypes.c_double(w_scale), q.data_ptr(), nv.stream_ptr())
    return q, w_scale


def _dev_f64(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(nv.require_cuda())


# ------------------------------------------------------------ reference API
def scale_weights(w: WeightTensor, sv: ScaleVector) -> WeightTensor:
    if len(sv.s) != w.cols:
        raise DcompError(f"{w.name}: scale length {len(sv.s)} != cols {w.cols}")
    if w.values.size == 0:
        return WeightTensor(w.name, w.values.copy())
    dw, ds = _dev_f64(w.values), _dev_f64(sv.s)
    out = torch.empty_like(dw)
    nv.call("dc_scale_weights", dw.data_ptr(), ds.data_ptr(), w.rows, w.cols, out.data_ptr(), nv.stream_ptr())
    return WeightTensor(w.name, out.cpu().numpy())


def _quantize_host(w: WeightTensor, s: np.ndarray | None, sv: ScaleVector) -> QuantizedTensor:
    if w.values.size == 0:
        raise DcompError(f"{w.name}: empty input")
    q, w_scale = quantize_device(_dev_f64(w.values), None if s is None else _dev_f64(s), w.name)
    return QuantizedTensor(w.name, q.cpu().numpy(), w_scale, sv)


def quantize(w: WeightTensor, scale_vec: ScaleVector | None = None) -> QuantizedTensor:
    """Per-tensor symmetric INT8: q = clamp(round_half_away(v / w_scale), -127, 127),
    w_scale = max|v| / 127.  ``scale_vec`` records scaling already applied to w."""
    sv = scale_vec if scale_vec is not None else ScaleVector.identity(w.cols)
    return _quantize_host(w, None, sv)


def quantize_scaled(w: WeightTensor, stats: ActivationStats, alpha: float) -> QuantizedTensor:
    """compute_scale + scale_weights + quantize, fused in one GPU pass
    (the f64 product W*s is formed in registers, never stored)."""
    sv = compute_scale(stats, alpha)
    if len(sv.s) != w.cols:
        raise DcompError(f"{w.name}: scale length {len(sv.s)} != cols {w.cols}")
    return _quantize_host(w, sv.s, sv)


def dequantize(q: QuantizedTensor) -> WeightTensor:
    """v = q * w_scale / s[c]."""
    if q.qvalues.size == 0:
        return WeightTensor(q.name, np.zeros(q.qvalues.shape))
    dev = nv.require_cuda()
    dq = torch.from_numpy(np.ascontiguousarray(q.qvalues)).to(dev)
    ds = _dev_f64(q.scale_vec.s)
    out = torch.empty(q.qvalues.shape, dtype=torch.float64, device=dev)
    nv.call("dc_dequantize", dq.data_ptr(), ctypes.c_double(q.w_scale), ds.data_ptr(), q.rows, q.cols,
            out.data_ptr(), nv.stream_ptr())
    return WeightTensor(q.name, out.cpu().numpy())


def simulate_layer(x: np.ndarray, w: WeightTensor, stats: ActivationStats, alpha: float) -> LayerErrorReport:
    """Relative Frobenius errors of the scaled W8A8 path on one layer.

    The INT8 product runs on the tcgen05 W8A8 GEMM (exact int32 accumulation,
    gemm.py); the f64 references are the function's own yardstick."""
    from .gemm import w8a8_matmul_exact

    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 2 or x.shape[1] != w.cols:
        raise DcompError(f"{w.name}: activation shape {x.shape} incompatible with cols {w.cols}")
    sv = compute_scale(stats, alpha)
    dev = nv.require_cuda()
    X = torch.from_numpy(x).to(dev)
    W = torch.from_numpy(w.values).to(dev)
    S = torch.from_numpy(sv.s).to(dev)
    y_ref = X @ W.T
    ref_norm = float(torch.linalg.norm(y_ref))
    if ref_norm == 0.0:
        raise DcompError(f"{w.name}: reference output is identically zero")
    xs = X / S[None, :]
    ws = W * S[None, :]
    fp_err = float(torch.linalg.norm(xs @ ws.T - y_ref)) / ref_norm
    qw, sw = quantize_device(ws, None, w.name)
    qx, sx = quantize_device(xs.contiguous(), None, f"{w.name}.x")
    acc = w8a8_matmul_exact(qx, qw)  # int32 [B, N] = qx @ qw.T
    y_hat = acc.to(torch.float64) * (sx * sw)
    q_err = float(torch.linalg.norm(y_hat - y_ref)) / ref_norm
    return LayerErrorReport(alpha=alpha, fp_identity_error=fp_err, quantized_error=q_err)


# ---- value types of the API (defined after the functions; annotations are strings)

@dataclasses.dataclass(frozen=True)
class ScaleVector:
    alpha: float
    s: np.ndarray  # (cols,) float64, > 0

    def __post_init__(self):
        s = np.asarray(self.s, dtype=np.float64)
        if (s <= 0).any() or not np.isfinite(s).all():
            raise ValueError("scale factors must be positive and finite")
        object.__setattr__(self, "s", s)

    @classmethod
    def identity(cls, cols: int) -> "ScaleVector":
        return cls(0.0, np.ones(cols))


@dataclasses.dataclass(frozen=True)
class QuantizedTensor:
    name: str
    qvalues: np.ndarray  # (rows, cols) int8 in [-127, 127]
    w_scale: float
    scale_vec: ScaleVector

    def __post_init__(self):
        q = np.asarray(self.qvalues, dtype=np.int8)
        if q.ndim != 2:
            raise ValueError(f"{self.name}: expected 2-D qvalues")
        object.__setattr__(self, "qvalues", q)
        if self.w_scale <= 0:
            raise ValueError(f"{self.name}: w_scale must be positive")
        if len(self.scale_vec.s) != q.shape[1]:
            raise ValueError(f"{self.name}: scale_vec length != cols")

    rows = property(lambda self: self.qvalues.shape[0])
    cols = property(lambda self: self.qvalues.shape[1])


@dataclasses.dataclass(frozen=True)
class LayerErrorReport:
    alpha: float
    fp_identity_error: float  # (X/s)(sW) vs XW, no quantization
    quantized_error: float    # full INT8 path vs the f64 reference
