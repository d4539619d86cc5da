"""Compression-ratio / error sweep over the alpha grid on the GPU (
the reference's ``dcomp sweep`` command, cli.py:201-230, and the paper's
Figure-7 alpha trade-off).

For every alpha: quantize every tensor with the activation-aware scale
(k_absmax / k_quantize), optionally prune (k_colhist ... k_apply), measure the
EXACT standalone blob length of each tensor (``compress_blob``: GPU
histogram -> normalize -> rANS encode; one chunk per tensor, all tensors
encoded concurrently), the near-zero fraction (|q| <= 1, tensors.py:22) and
the mean W8A8 layer error of ``simulate_layer`` on seeded calibration
activations X = N(0,1) * cm (cli.py:205-207).  The CR column is therefore the
reference's number, not an entropy estimate.
"""

from __future__ import annotations

import numpy as np
import torch

from . import native as nv
from .errors import DcompError
from .pruning import prune_device
from .scaling import ALPHA_GRID, compute_scale, quantize_device
from .tensors import ActivationStats, WeightTensor

TAU_NZ = 1
TABLE_BYTES = 384
HEADER_BYTES = 388


def blob_lengths(payloads: list[torch.Tensor], streams: int = 8) -> list[int]:
    """len(compress_blob(p)) for each contiguous uint8 CUDA tensor, exactly
    (the encoder is serial per blob, so blobs run concurrently on ``streams``
    CUDA streams, one warp each)."""
    if not payloads:
        return []
    dev = payloads[0].device
    n = len(payloads)
    hist = torch.empty((n, 256), dtype=torch.int32, device=dev)
    freq = torch.empty((n, 256), dtype=torch.int32, device=dev)
    tb = torch.empty((n, TABLE_BYTES), dtype=torch.uint8, device=dev)
    state = torch.empty(n, dtype=torch.int32, device=dev)
    slen = torch.empty(n, dtype=torch.int64, device=dev)
    todo = torch.ones(n, dtype=torch.uint8, device=dev)
    ss = [torch.cuda.Stream(dev) for _ in range(streams)]
    main = torch.cuda.current_stream(dev)
    keep = []
    for i, p in enumerate(payloads):
        m = p.numel()
        if m == 0:
            raise DcompError("empty input")
        st = ss[i % streams]
        st.wait_stream(main)
        with torch.cuda.stream(st):
            work, wbytes = nv.encode_work(m, m, 1, dev)
            keep.append(work)
            sp = st.cuda_stream
            nv.call("dc_hist_chunks", p.data_ptr(), m, m, 1, hist[i].data_ptr(), sp)
            nv.call("dc_normalize_tables", hist[i].data_ptr(), 1, freq[i].data_ptr(), tb[i].data_ptr(), sp)
            # standalone (bit 0) and lengths only (bit 1): no stream bytes are written
            nv.call("dc_ans_encode_chunks", p.data_ptr(), m, m, 1, todo[i:i + 1].data_ptr(), freq[i].data_ptr(),
                    None, state[i:i + 1].data_ptr(), slen[i:i + 1].data_ptr(), 0, None, None, None, 3,
                    work.data_ptr(), wbytes, sp)
    for st in ss:
        main.wait_stream(st)
    lens = slen.cpu().numpy()
    del keep
    return [HEADER_BYTES + int(x) for x in lens]


def _calib(seed: int, i: int, cols: int, cm: np.ndarray, rows: int) -> np.ndarray:
    rng = np.random.default_rng([seed, i])
    return rng.normal(0.0, 1.0, (rows, cols)) * cm[None, :]


def alpha_sweep(weights: list[WeightTensor], stats: dict[str, ActivationStats], alphas=ALPHA_GRID,
                sparsity: float = 0.0, per_row: bool = False, seed: int = 0, calib_rows: int = 64,
                with_error: bool = True) -> list[dict]:
    """Rows {alpha, cr, near_zero, layer_error} like ``dcomp sweep``."""
    from .scaling import simulate_layer
    dev = nv.require_cuda()
    dw = [torch.from_numpy(np.ascontiguousarray(w.values, dtype=np.float64)).to(dev) for w in weights]
    cms = [np.asarray(stats[w.name].channel_max, dtype=np.float64) for w in weights]
    dcm = [torch.from_numpy(c).to(dev) for c in cms]
    calib = [_calib(seed, i, w.cols, cms[i], calib_rows) for i, w in enumerate(weights)] if with_error else None
    # quantize (+ prune) every (alpha, tensor) first, then encode all of them at
    # once: each standalone blob is one serial chain, so running them side by
    # side makes the whole sweep cost about one (largest) encode
    per_alpha = []
    for alpha in alphas:
        if not 0.0 <= alpha <= 1.0:
            raise DcompError(f"alpha must be in [0, 1], got {alpha}")
        qs = []
        for wt, w, c in zip(weights, dw, dcm):
            s = compute_scale(stats[wt.name], alpha).s  # host numpy, bit-exact with the reference
            q, _ = quantize_device(w, torch.from_numpy(np.ascontiguousarray(s)).to(dev))
            if sparsity > 0:
                q = prune_device(q, c, sparsity, per_row)
            qs.append(q)
        per_alpha.append(qs)
    flat = [q.reshape(-1).view(torch.uint8) for qs in per_alpha for q in qs]
    lens = blob_lengths(flat, streams=min(len(flat), 64))
    rows = []
    for ai, (alpha, qs) in enumerate(zip(alphas, per_alpha)):
        u = sum(q.numel() for q in qs)
        comp = sum(lens[ai * len(qs):(ai + 1) * len(qs)])
        nz = sum(int((q.to(torch.int16).abs() <= TAU_NZ).sum()) for q in qs) / u
        err = None
        if with_error:
            err = float(np.mean([simulate_layer(calib[i], w, stats[w.name], alpha).quantized_error
                                 for i, w in enumerate(weights)]))
        rows.append({"alpha": alpha, "cr": u / comp, "near_zero": nz, "layer_error": err, "raw_bytes": u,
                     "blob_bytes": comp})
    return rows
