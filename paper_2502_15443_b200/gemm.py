"""W8A8 GEMMs on the tcgen05 tensor cores (csrc/gemm_w8a8.cu, csrc/gemm_grouped.cu,
csrc/fused_ring.cu).

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


# ----------------------------------------------------------------- grouped
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

_GT_DTYPE = np.dtype([("x", "<u8"), ("acc", "<u8"), ("t_off", "<i8"), ("n_rows", "<i4"), ("k", "<i4")])


def _equal_kslice(k: int, target: int) -> int:
    """Largest multiple of KB dividing k and <= target (k itself if k <= target)."""
    if k <= target:
        return k
    best = KB
    for ks in range(KB, target + 1, KB):
        if k % ks == 0:
            best = ks
    return best


class _LayerSet:
    """Per-layer activations and int32 accumulators shared by the grouped
    INT8 GEMM and the fused decode GEMM (one launch covers every layer)."""

    def __init__(self, shapes, t_offs, xs, ntok: int):
        assert _GT_DTYPE.itemsize == nv.call("dc_gemm_tensor_bytes")
        self.shapes = [(int(r), int(k)) for r, k in shapes]
        self.ntok = ntok
        self.xs = [x.contiguous() for x in xs]
        dev = self.xs[0].device
        sizes = [ntok * r for r, _ in self.shapes]
        self.acc_flat = torch.zeros(sum(sizes), dtype=torch.int32, device=dev)
        self.accs, pos = [], 0
        for (r, _), n in zip(self.shapes, sizes):
            self.accs.append(self.acc_flat[pos:pos + n].view(ntok, r))
            pos += n
        gt = np.zeros(len(self.shapes), dtype=_GT_DTYPE)
        gt["x"] = [x.data_ptr() for x in self.xs]
        gt["acc"] = [a.data_ptr() for a in self.accs]
        gt["t_off"] = np.asarray(t_offs, dtype=np.int64)
        gt["n_rows"] = [r for r, _ in self.shapes]
        gt["k"] = [k for _, k in self.shapes]
        self.tens = torch.from_numpy(gt.view(np.uint8).copy()).to(dev)

    def units(self, kslice_of) -> torch.Tensor:
        rows = []
        for li, (r, k) in enumerate(self.shapes):
            ks = kslice_of(r, k)
            for m0 in range(0, r, 128):
                for k0 in range(0, k, ks):
                    rows.append((li, m0, k0, ks))
        return torch.tensor(rows, dtype=torch.int32, device=self.xs[0].device)


class GroupedInt8:
    """All linears of a model, uncompressed INT8 weights, one tcgen05 launch."""

    def __init__(self, weights: list[torch.Tensor], xs: list[torch.Tensor], ntok: int):
        if ntok > 16:
            raise ValueError("grouped GEMM handles <= 16 tokens per launch")
        self.layers = _LayerSet([w.shape for w in weights], [0] * len(weights), xs, ntok)
        self.weights = [w.contiguous() for w in weights]
        n = len(weights)
        mb = nv.call("dc_tmap_bytes")
        host = np.zeros(2 * n * mb + 64, dtype=np.uint8)
        off = (-host.ctypes.data) % 64
        maps = host[off:off + 2 * n * mb]
        P = ctypes.c_void_p
        w_ptrs = (P * n)(*[w.data_ptr() for w in self.weights])
        x_ptrs = (P * n)(*[x.data_ptr() for x in self.layers.xs])
        rows = (ctypes.c_int64 * n)(*[w.shape[0] for w in self.weights])
        ks = (ctypes.c_int64 * n)(*[w.shape[1] for w in self.weights])
        nv.lib().dc_w8a8_grouped_maps.argtypes = [P, P, P, P, ctypes.c_int, ctypes.c_int, P]
        rc = nv.lib().dc_w8a8_grouped_maps(w_ptrs, x_ptrs, rows, ks, n, ntok, maps.ctypes.data)
        if rc:
            raise nv.NativeError(f"dc_w8a8_grouped_maps failed ({rc})")
        self.maps = torch.from_numpy(maps.copy()).to(self.weights[0].device)
        self.unit_t = self.layers.units(lambda r, k: k)
        # persistent kernel: round-robin over units, so every unit gets the
        # same K length (split-K with atomics) to keep the SMs balanced
        self.unit_p = self.layers.units(lambda r, k: _equal_kslice(k, 4096))

    @property
    def accs(self):
        return self.layers.accs

    def run(self, max_ctas: int | None = None) -> None:
        """One launch over every layer.  ``max_ctas`` selects the persistent
        kernel (one CTA per SM, grid capped at max_ctas; 0 = every SM)."""
        self.layers.acc_flat.zero_()
        if max_ctas is None:
            nv.call("dc_w8a8_grouped", self.maps.data_ptr(), self.layers.tens.data_ptr(), self.unit_t.data_ptr(),
                    self.unit_t.shape[0], self.layers.ntok, nv.stream_ptr())
        else:
            nv.call("dc_w8a8_grouped_persist", self.maps.data_ptr(), self.layers.tens.data_ptr(),
                    self.unit_p.data_ptr(), self.unit_p.shape[0], self.layers.ntok, int(max_ctas), nv.stream_ptr())


class FusedRing:
    """Fused decode -> TMEM ring -> tcgen05 W8A8 (csrc/fused_ring.cu): one
    persistent 16-warp CTA per SM, 1024 decode chains feeding the tensor core
    every 32 symbols.  Items: 1024 rows x K-slice (<= 2048 bytes).

    ``run()`` trusts the split-point index and reports broken chains through
    ``check()``; ``run_checked()`` verifies and, if any chain broke (stale or
    corrupt index), recomputes the outputs exactly from the container."""

    def __init__(self, image: torch.Tensor, jobs, index, chunk_size: int, shapes, t_offs, xs, ntok: int,
                 scales=None):
        """``scales`` (optional, one float per layer = sx * sw): also emit the
        dequantized fp32 outputs ``ys[i]`` = acc * scale from the same launch
        (fused dequant epilogue; the int32 accumulation stays exact)."""
        if index is None or index.seg_shift != 8:
            raise ValueError("fused path needs a split-point index with 256-symbol segments")
        rows_per = nv.call("dc_fused_item_rows")
        kmax = nv.call("dc_fused_item_k")
        if chunk_size % 256 or any(int(t) % 256 for t in t_offs) or any(k % 256 for _, k in shapes):
            raise ValueError("fused path needs chunk_size, tensor offsets and K multiples of 256")
        for (r, k), t in zip(shapes, t_offs):
            if (rows_per - 1) * k + kmax > chunk_size:
                raise ValueError("chunk too small for the fused path (1024 rows x K must fit in one chunk)")
        self.image, self.jobs, self.index, self.chunk_size = image, jobs, index, chunk_size
        # Consecutive layers that read the same activations and sit back to back
        # in the payload (q/k/v, gate/up) become one taller matrix: its row
        # blocks fill the 1024-row items (a 640-row TP shard alone leaves 3/8
        # of the chains idle).  accs stay per layer (row-slice views).
        shapes = [(int(r), int(k)) for r, k in shapes]
        groups, i = [], 0
        while i < len(shapes):
            j = i + 1
            while (scales is None and j < len(shapes) and shapes[j][1] == shapes[i][1]
                   and int(t_offs[j]) == int(t_offs[j - 1]) + shapes[j - 1][0] * shapes[j - 1][1]
                   and xs[j].data_ptr() == xs[i].data_ptr() and xs[j].shape == xs[i].shape):
                j += 1
            groups.append((i, j))
            i = j
        m_shapes = [(sum(shapes[q][0] for q in range(a, b)), shapes[a][1]) for a, b in groups]
        m_offs = [int(t_offs[a]) for a, _ in groups]
        self.t_offs = m_offs
        self.layers = _LayerSet(m_shapes, m_offs, [xs[a] for a, _ in groups], ntok)
        self._accs = []
        for (a, b), acc in zip(groups, self.layers.accs):
            r0 = 0
            for q in range(a, b):
                self._accs.append(acc[:, r0:r0 + shapes[q][0]])
                r0 += shapes[q][0]
        self.merged_layers = len(shapes) - len(groups)
        shapes, t_offs = m_shapes, m_offs
        items, kss = [], []
        for li, (r, k) in enumerate(self.layers.shapes):
            # a chain's K-slice must never straddle a chunk boundary: use the
            # largest power of two <= kmax dividing K, the layer offset and the chunk size
            ks = kmax
            while ks > 256 and (k % ks or int(t_offs[li]) % ks or chunk_size % ks):
                ks //= 2
            for m0 in range(0, r, rows_per):
                for k0 in range(0, k, ks):
                    items.append((li, m0, k0, min(ks, k - k0)))
            kss.append(ks)
        self.unit_t = torch.tensor(items, dtype=torch.int32, device=image.device)
        self.status = torch.zeros(max(jobs.n, 1), dtype=torch.int32, device=image.device)
        self.ys, self.epi = None, None
        if scales is not None:
            dev = image.device
            self.scales = [float(np.float32(x)) for x in scales]
            self.ys = [torch.zeros((ntok, r), dtype=torch.float32, device=dev) for r, _ in self.layers.shapes]
            nblk = [-(-r // rows_per) for r, _ in self.layers.shapes]
            self.counters = torch.zeros(sum(nblk), dtype=torch.int32, device=dev)
            cnt_off = np.concatenate([[0], np.cumsum(nblk)[:-1]]).astype(np.int64)
            dt = np.dtype([("y", "<u8"), ("cnt", "<u8"), ("scale", "<f4"), ("n_slices", "<i4")])
            assert dt.itemsize == nv.call("dc_fused_epi_bytes")
            e = np.zeros(len(self.layers.shapes), dtype=dt)
            e["y"] = [y.data_ptr() for y in self.ys]
            e["cnt"] = [self.counters.data_ptr() + 4 * int(o) for o in cnt_off]
            e["scale"] = np.asarray(scales, dtype=np.float32)
            e["n_slices"] = [-(-k // ks) for (_, k), ks in zip(self.layers.shapes, kss)]
            self.epi = torch.from_numpy(e.view(np.uint8).copy()).to(dev)

    @property
    def accs(self):
        return self._accs

    def check(self) -> np.ndarray:
        """Per-chunk status after run(); nonzero = chain broken / corrupt."""
        return self.status[: self.jobs.n].cpu().numpy()

    def run(self, max_ctas: int = 0) -> None:
        self.layers.acc_flat.zero_()
        self.status.zero_()
        if self.epi is not None:
            self.counters.zero_()
        j, ix = self.jobs, self.index
        nv.call("dc_fused_ring_gemm", self.image.data_ptr(), j.d_blob_off.data_ptr(), j.d_blob_len.data_ptr(),
                j.d_out_len.data_ptr(), j.d_codec.data_ptr(), self.chunk_size, ix.d_seg_base.data_ptr(),
                ix.d_state.data_ptr(), ix.d_off.data_ptr(), self.layers.tens.data_ptr(), self.unit_t.data_ptr(),
                self.unit_t.shape[0], self.layers.ntok, self.status.data_ptr(),
                self.epi.data_ptr() if self.epi is not None else None, int(max_ctas), nv.stream_ptr())

    def run_checked(self) -> bool:
        """run(), verify every chain (one host sync) and fall back to the exact
        path -- container decode with serial re-decode of broken chunks, then
        the INT8 GEMM -- if any split point did not hold.  Returns True when
        the fused result stood."""
        from . import engine
        from .errors import CorruptStreamError
        self.run()
        if not (self.check() != 0).any():
            return True
        res = engine.decode_jobs(self.image, self.jobs, self.index)
        bad = np.nonzero(res.status != 0)[0]
        if len(bad):
            raise CorruptStreamError(f"corrupt stream (chunk {int(bad[0])})")
        views = [res.out[t:t + r * k].view(torch.int8).view(r, k) for (r, k), t in zip(self.layers.shapes, self.t_offs)]
        gi = GroupedInt8(views, self.layers.xs, self.layers.ntok)
        gi.run()
        self.layers.acc_flat.copy_(gi.layers.acc_flat)
        if self.ys is not None:
            for y, acc, sc in zip(self.ys, self.accs, self.scales):
                y.copy_(acc.to(torch.float32) * sc)
        return False


class MixedStep:
    """A partially compressed model's decode step: the compressed
    layers through the fused decode -> tcgen05 kernel and the plain INT8 layers
    through the grouped tcgen05 GEMM, run CONCURRENTLY on two streams.  The
    fused kernel is ALU-bound and the INT8 GEMM HBM-bound, so they overlap
    well; the persistent fused grid is capped at ``fused_ctas`` SMs (one CTA
    each), leaving the rest to the INT8 GEMM.  ``tune()`` picks the split from
    measured step times -- the reference's latency model assumes exactly this
    overlap (latency.py:144-222: per chunk max(load, decode, compute))."""

    def __init__(self, fused: FusedRing | None, int8: GroupedInt8 | None, fused_ctas: int = 0):
        self.fused, self.int8, self.fused_ctas = fused, int8, fused_ctas
        dev = (fused.layers.acc_flat if fused is not None else int8.layers.acc_flat).device
        self.side = torch.cuda.Stream(dev)

    def run(self) -> None:
        if self.fused is None or self.int8 is None:
            (self.fused.run if self.int8 is None else self.int8.run)()
            return
        main = torch.cuda.current_stream()
        sms = _sm_count()
        fc = self.fused_ctas if 0 < self.fused_ctas < sms else sms
        self.side.wait_stream(main)  # inputs ready / previous step's readers finished
        self.fused.run(fc)           # one CTA per SM on fc SMs ...
        with torch.cuda.stream(self.side):
            self.int8.run(max_ctas=sms - fc if fc < sms else 0)  # ... the persistent GEMM on the others
        main.wait_stream(self.side)

    def tune(self, candidates=None, iters: int = 5) -> dict:
        """Measure the step for each fused-grid size; keep the fastest."""
        from .adaptive import time_ms
        if self.fused is None or self.int8 is None:
            return {}
        sms = _sm_count()
        cands = candidates or sorted(set(range(sms // 4, sms, 8)) | {sms})
        times = {}
        for c in cands:
            self.fused_ctas = c
            times[c] = time_ms(self.run, iters=iters)
        self.fused_ctas = min(times, key=times.get)
        return times
