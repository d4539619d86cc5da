"""W8A8 GEMMs on the tcgen05 tensor cores (csrc/gemm_w8a8.cu, csrc/fused_gemm.cu).

``w8a8_matmul_exact(qx, qw)`` returns the exact int32 products qx @ qw.T
(the integer core of the reference's W8A8 numerics, scaling.py:127-152);
callers scale by sx * sw.  Decode-shaped: tokens <= 32 per launch (larger
batches are tiled), weight rows on the UMMA M dimension.
"""

from __future__ import annotations

import torch

from . import native as nv

KB = 128  # K bytes per pipeline stage


def _sm_count() -> int:
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def choose_kslice(n_rows: int, k: int, target_ctas: int | None = None) -> int:
    """Split K so that tiles x splits covers ~2 waves of CTAs."""
    target = target_ctas or 2 * _sm_count()
    tiles = -(-n_rows // 128)
    kb = k // KB
    best = kb
    for splits in range(1, kb + 1):
        if kb % splits:
            continue
        best = kb // splits
        if tiles * splits >= target:
            break
    return best * KB


def w8a8_gemm_into(qx: torch.Tensor, qw: torch.Tensor, acc: torch.Tensor, kslice: int | None = None) -> None:
    """acc[t, n] = sum_k qx[t, k] * qw[n, k] (int32, exact); qx [T<=32, K],
    qw [N, K] int8 CUDA, K % 128 == 0, acc int32 [T, N] (zeroed here when
    K is split)."""
    T, K = qx.shape
    N = qw.shape[0]
    ks = kslice or choose_kslice(N, K)
    if ks < K:
        acc.zero_()
    nv.call("dc_w8a8_gemm", qw.data_ptr(), N, K, qx.data_ptr(), T, acc.data_ptr(), ks, nv.stream_ptr())


def w8a8_matmul_exact(qx: torch.Tensor, qw: torch.Tensor) -> torch.Tensor:
    """int32 [T, N] = qx [T, K] @ qw [N, K]^T for int8 CUDA tensors."""
    nv.require_cuda()
    T, K = qx.shape
    N, K2 = qw.shape
    if K != K2:
        raise ValueError(f"K mismatch {K} != {K2}")
    pad = (-K) % KB
    if pad:  # zero columns change no product
        qx = torch.nn.functional.pad(qx, (0, pad))
        qw = torch.nn.functional.pad(qw, (0, pad))
    qx = qx.contiguous()
    qw = qw.contiguous()
    out = torch.empty((T, N), dtype=torch.int32, device=qx.device)
    for t0 in range(0, T, 32):
        t1 = min(T, t0 + 32)
        part = out[t0:t1] if t0 == 0 and t1 == T else torch.empty((t1 - t0, N), dtype=torch.int32, device=qx.device)
        w8a8_gemm_into(qx[t0:t1].contiguous(), qw, part)
        if part.data_ptr() != out[t0:t1].data_ptr():
            out[t0:t1] = part
    return out
