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

    def __init__(self, shapes, t_offs, xs, ntok: int, accs=None):
        """``accs``: optional caller-owned int32 [ntok, rows] accumulators
        (contiguous; the caller zeroes them) instead of one owned buffer."""
        assert _GT_DTYPE.itemsize == nv.call("dc_gemm_tensor_bytes")
        self.shapes = [(int(r), int(k)) for r, k in shapes]
        self.ntok = ntok
        self.xs = [x.contiguous() for x in xs]
        dev = self.xs[0].device
        sizes = [ntok * r for r, _ in self.shapes]
        if accs is not None:
            assert all(a.is_contiguous() and a.dtype == torch.int32 and tuple(a.shape) == (ntok, r)
                       for a, (r, _) in zip(accs, self.shapes))
            self.acc_flat, self.accs = None, list(accs)
        else:
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

    def __init__(self, weights: list[torch.Tensor], xs: list[torch.Tensor], ntok: int, accs=None):
        if ntok > 16:
            raise ValueError("grouped GEMM handles <= 16 tokens per launch")
        self.layers = _LayerSet([w.shape for w in weights], [0] * len(weights), xs, ntok, accs)
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
        if self.layers.acc_flat is not None:
            self.layers.acc_flat.zero_()
        if max_ctas is None:
            nv.call("dc_w8a8_grouped", self.maps.data_ptr(), self.layers.tens.data_ptr(), self.unit_t.data_ptr(),
                    self.unit_t.shape[0], self.layers.ntok, nv.stream_ptr())
        else:
            nv.call("dc_w8a8_grouped_persist", self.maps.data_ptr(), self.layers.tens.data_ptr(),
                    self.unit_p.data_ptr(), self.unit_p.shape[0], self.layers.ntok, int(max_ctas), nv.stream_ptr())


class _StreamedDecodeGemm:
    """Layers whose 1024-row items the fused ring cannot serve (an item's rows
    spanning more than two chunks -- small chunks -- or a chunk size / layer
    offset / K that is not a multiple of 256): per group of layers, the
    split-point decoder writes ONLY those layers' segments (chunk x segment
    range tasks, so the native layers between them are not decoded twice)
    into an L2-sized scratch slot, and the grouped tcgen05 INT8 GEMM reads
    them back while still L2-resident, accumulating straight into the
    caller's int32 outputs; the slots alternate so group g + 1 decodes on a
    second stream while group g multiplies."""

    SLOT_BYTES = 48 << 20

    def __init__(self, image, jobs, index, layers, ntok: int):
        """``layers``: list of (rows, k, t_off, x, acc view) in payload order."""
        from . import engine
        dev = image.device
        self.image, self.jobs, self.index = image, jobs, index
        K = 1 << index.seg_shift
        out_off = jobs.out_off.astype(np.int64)
        out_len = jobs.out_len.astype(np.int64)
        out_end = out_off + out_len
        self.stored = []  # (slot index, slot byte offset, image byte offset, n) of stored-chunk pieces

        def pieces(t, n):
            """(chunk, first seg, end seg, payload start of first seg, payload end) per chunk of [t, t+n)."""
            c0 = int(np.searchsorted(out_end, t, side="right"))
            c1 = int(np.searchsorted(out_off, t + n, side="left"))
            out = []
            for c in range(c0, c1):
                lo, hi = max(t, int(out_off[c])), min(t + n, int(out_end[c]))
                s_lo, s_hi = (lo - int(out_off[c])) // K, -(-(hi - int(out_off[c])) // K)
                a = int(out_off[c]) + s_lo * K
                b = min(int(out_off[c]) + s_hi * K, int(out_end[c]))
                out.append((c, s_lo, s_hi, a, b, lo, hi))
            return out

        # slot layout per group: each layer's decoded segment span [a, b) at slot
        # position p, chosen so the layer's first weight byte is 16-B aligned
        groups, cur, pos = [], [], 0
        for lay in layers:
            r, k, t, _, _ = lay
            pcs = pieces(t, r * k)
            a0, b1 = pcs[0][3], pcs[-1][4]
            need = (b1 - a0) + 32
            if cur and pos + need > self.SLOT_BYTES:
                groups.append(cur)
                cur, pos = [], 0
            p = pos + ((a0 - t) - pos) % 16  # (p + t - a0) % 16 == 0
            cur.append((lay, pcs, p, a0))
            pos = p + (b1 - a0) + 16
        if cur:
            groups.append(cur)
        self.groups = []
        slot_bytes = 0
        for gi, g in enumerate(groups):
            jc, jo, s_lo, s_hi = [], [], [], []
            for lay, pcs, p, a0 in g:
                for c, sl, sh, a, b, lo, hi in pcs:
                    if jobs.codec[c] == 0:  # stored chunk: plain copy of the layer's bytes
                        self.stored.append((gi, p + lo - a0, int(jobs.blob_off[c]) + lo - int(out_off[c]), hi - lo))
                        continue
                    jc.append(c)
                    jo.append(p + int(out_off[c]) - a0)  # may be negative: the kernel adds it mod 2^64
                    s_lo.append(sl)
                    s_hi.append(sh)
            jc = np.asarray(jc, dtype=np.int64)
            end = max(p + (pcs[-1][4] - a0) for _, pcs, p, a0 in g) + 16
            slot_bytes = max(slot_bytes, end)
            if len(jc):
                lj = engine.JobTable.build(jobs.blob_off[jc], jobs.blob_len[jc],
                                           np.asarray(jo, dtype=np.int64).view(np.uint64), jobs.out_len[jc],
                                           jobs.codec[jc], dev)
                li = engine.SegmentIndex(index.seg_shift, index.seg_base[jc], index.n_segs,
                                         index.d_seg_base[torch.from_numpy(jc).to(dev)].contiguous(),
                                         index.d_state, index.d_off, h_off=index.host_offsets())
                tasks = li.tasks(lj, np.ones(lj.n, bool), seg_range=(np.asarray(s_lo), np.asarray(s_hi)))
            else:
                lj = li = tasks = None
            self.groups.append((lj, li, tasks, jc, g))
        self.slots = [nv.device_bytes(slot_bytes, dev) for _ in range(min(2, len(self.groups)))]
        # one status word per (group, job): chunk ids kept for check()
        n_jobs = [len(jc) for _, _, _, jc, _ in self.groups]
        self.status = torch.zeros(max(sum(n_jobs), 1), dtype=torch.int32, device=dev)
        self.status_chunks = np.concatenate([jc for _, _, _, jc, _ in self.groups]) if sum(n_jobs) else \
            np.zeros(0, np.int64)
        self.status_off = np.concatenate([[0], np.cumsum(n_jobs)[:-1]]).astype(np.int64)
        self.gemms = []
        for gi, (lj, li, tasks, jc, g) in enumerate(self.groups):
            buf = self.slots[gi % len(self.slots)]
            views = [buf[p + t - a0:p + t - a0 + r * k].view(torch.int8).view(r, k) for (r, k, t, _, _), _, p, a0
                     in g]
            self.gemms.append(GroupedInt8(views, [lay[3] for lay, _, _, _ in g], ntok,
                                          accs=[lay[4] for lay, _, _, _ in g]))
        self.side = torch.cuda.Stream(dev)
        self.ev_free = [torch.cuda.Event() for _ in self.slots]

    def chunk_status(self, n_chunks: int) -> np.ndarray:
        """Per-chunk OR of this path's decode statuses."""
        out = np.zeros(n_chunks, dtype=np.int32)
        if len(self.status_chunks):
            st = self.status[: len(self.status_chunks)].cpu().numpy()
            np.maximum.at(out, self.status_chunks, np.abs(st))
        return out

    def run(self) -> None:
        from . import engine
        main = torch.cuda.current_stream()
        self.status.zero_()
        self.side.wait_stream(main)
        n = len(self.slots)
        for gi, ((lj, li, tasks, jc, g), gemm) in enumerate(zip(self.groups, self.gemms)):
            slot = self.slots[gi % n]
            with torch.cuda.stream(self.side):  # decode group gi while group gi - 1 multiplies
                if gi >= n:
                    self.side.wait_event(self.ev_free[gi % n])
                if tasks is not None and tasks.shape[0]:
                    nv.call(engine.segment_kernel(lj), self.image.data_ptr(), lj.d_blob_off.data_ptr(),
                            lj.d_blob_len.data_ptr(), lj.d_out_off.data_ptr(), lj.d_out_len.data_ptr(),
                            li.seg_shift, li.d_seg_base.data_ptr(), li.d_state.data_ptr(), li.d_off.data_ptr(),
                            tasks.data_ptr(), tasks.shape[0], slot.data_ptr(),
                            self.status.data_ptr() + 4 * int(self.status_off[gi]), self.side.cuda_stream)
                for sgi, so, io, nb in self.stored:
                    if sgi == gi:
                        slot[so:so + nb].copy_(self.image[io:io + nb])
                ev = torch.cuda.Event()
                ev.record(self.side)
            main.wait_event(ev)
            gemm.run()
            self.ev_free[gi % n].record(main)


def _row_slices(li: int, r: int, k: int, t: int, chunk_size: int, rows_per: int) -> list:
    """Items (layer, m0, 0, k): each row block's whole rows as one K-slice.
    A chain must never cross a chunk boundary inside its slice, so a row block
    where some row straddles one is cut there (a multiple of 256 from the row
    start: the layer offset, K and the chunk size are)."""
    out = []
    for m0 in range(0, r, rows_per):
        rows = np.arange(m0, min(m0 + rows_per, r), dtype=np.int64)
        st = t + rows * k
        ca, cb = st // chunk_size, (st + k - 1) // chunk_size
        bad = np.nonzero(ca != cb)[0]
        edges = [0] + sorted({int(cb[i] * chunk_size - st[i]) for i in bad}) + [k]
        out += [(li, m0, a, b - a) for a, b in zip(edges, edges[1:])]
    return out


class FusedRing:
    """Fused decode -> TMEM ring -> tcgen05 W8A8 (csrc/fused_ring.cu): one
    persistent 16-warp CTA per SM, 1024 decode chains feeding the tensor core
    every 32 symbols.  Items: 1024 rows x K-slice (<= 2048 bytes).

    Any chunk size: a layer whose items would span more than two chunks (its
    1024 rows x K exceed a chunk), or whose chunk size / offset / K is not a
    multiple of 256, goes through ``_StreamedDecodeGemm`` (decode into an
    L2-sized scratch slot, then the grouped INT8 GEMM) inside the same run().

    ``run()`` trusts the split-point index and reports broken chains through
    ``check()``; ``run_checked()`` verifies and, if any chain broke (stale or
    corrupt index), recomputes the outputs exactly from the container."""

    def __init__(self, image: torch.Tensor, jobs, index, chunk_size: int, shapes, t_offs, xs, ntok: int,
                 scales=None, act_scales=None):
        """``scales`` (optional, one float per layer = sx * sw) or
        ``act_scales`` (one (device f64 sx tensor, float sw) per layer, e.g.
        from dc_act_quant): also emit the dequantized fp32 outputs ``ys[i]``
        = acc * scale from the same launch (fused dequant epilogue; the int32
        accumulation stays exact)."""
        if index is None or index.seg_shift != 8:
            raise ValueError("fused path needs a split-point index with 256-symbol segments")
        rows_per = nv.call("dc_fused_item_rows")
        kmax = nv.call("dc_fused_item_k")
        self.image, self.jobs, self.index, self.chunk_size = image, jobs, index, chunk_size
        epilogue = scales is not None or act_scales is not None
        # Consecutive layers that read the same activations and sit back to back
        # in the payload (q/k/v, gate/up) become one taller matrix: its row
        # blocks fill the 1024-row items (a 640-row TP shard alone leaves 3/8
        # of the chains idle).  accs stay per layer (row-slice views).
        shapes = [(int(r), int(k)) for r, k in shapes]
        groups, i = [], 0
        while i < len(shapes):
            j = i + 1
            while (not epilogue and j < len(shapes) and shapes[j][1] == shapes[i][1]
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
        items, kss, fallback = [], [], []
        for li, (r, k) in enumerate(self.layers.shapes):
            t = m_offs[li]
            native = chunk_size % 256 == 0 and t % 256 == 0 and k % 256 == 0
            # a chain's K-slice must never straddle a chunk boundary: the largest
            # power of two <= kmax dividing K, the layer offset and the chunk size
            ks = kmax
            while ks > 256 and (k % ks or t % ks or chunk_size % ks):
                ks //= 2
            if native and not epilogue and ks < k <= kmax:
                # a whole row fits one slice (e.g. a TP shard's K = 768 or 1792):
                # one K-slice per row block instead of K/ks small ones
                mine = _row_slices(li, r, k, t, chunk_size, rows_per)
            else:
                mine = [(li, m0, k0, min(ks, k - k0)) for m0 in range(0, r, rows_per) for k0 in range(0, k, ks)]
            if native and mine:  # every item's rows must touch at most two chunks (two table slots)
                it = np.asarray(mine, dtype=np.int64)
                first = t + it[:, 1] * k + it[:, 2]
                last = t + (np.minimum(it[:, 1] + rows_per, r) - 1) * k + it[:, 2] + it[:, 3] - 1
                native = bool(((last // chunk_size) - (first // chunk_size) <= 1).all())
            if native:
                items += mine
            else:
                fallback.append(li)
            kss.append(ks)
        self.native_layers = len(self.layers.shapes) - len(fallback)
        self.unit_t = (torch.tensor(items, dtype=torch.int32, device=image.device) if items
                       else torch.zeros((0, 4), dtype=torch.int32, device=image.device))
        self.status = torch.zeros(max(jobs.n, 1), dtype=torch.int32, device=image.device)
        self._fb = None
        if fallback:
            self._fb = _StreamedDecodeGemm(
                image, jobs, index, [(*self.layers.shapes[li], m_offs[li], self.layers.xs[li], self.layers.accs[li])
                                     for li in fallback], ntok)
        self._fb_layers = fallback
        self.ys, self.epi = None, None
        if epilogue:
            dev = image.device
            n_l = len(self.layers.shapes)
            self.scales = [float(np.float32(x)) for x in scales] if scales is not None else None
            self.act_scales = act_scales
            self.ys = [torch.zeros((ntok, r), dtype=torch.float32, device=dev) for r, _ in self.layers.shapes]
            nblk = [-(-r // rows_per) for r, _ in self.layers.shapes]
            self.counters = torch.zeros(sum(nblk), dtype=torch.int32, device=dev)
            cnt_off = np.concatenate([[0], np.cumsum(nblk)[:-1]]).astype(np.int64)
            dt = np.dtype([("y", "<u8"), ("cnt", "<u8"), ("scale", "<f4"), ("n_slices", "<i4"), ("sx", "<u8"),
                           ("sw", "<f8")])
            assert dt.itemsize == nv.call("dc_fused_epi_bytes")
            e = np.zeros(n_l, dtype=dt)
            e["y"] = [y.data_ptr() for y in self.ys]
            e["cnt"] = [self.counters.data_ptr() + 4 * int(o) for o in cnt_off]
            if scales is not None:
                e["scale"] = np.asarray(scales, dtype=np.float32)
            else:
                e["sx"] = [sx.data_ptr() for sx, _ in act_scales]
                e["sw"] = [float(sw) for _, sw in act_scales]
            e["n_slices"] = [-(-k // ks) for (_, k), ks in zip(self.layers.shapes, kss)]
            self.epi = torch.from_numpy(e.view(np.uint8).copy()).to(dev)

    @property
    def accs(self):
        return self._accs

    def check(self) -> np.ndarray:
        """Per-chunk status after run(); nonzero = chain broken / corrupt."""
        st = self.status[: self.jobs.n].cpu().numpy()
        if self._fb is not None:
            st = np.where(st != 0, st, self._fb.chunk_status(self.jobs.n))
        return st

    def _fallback_epilogue(self) -> None:
        for li in self._fb_layers:
            acc = self.layers.accs[li]
            if self.scales is not None:
                self.ys[li].copy_(acc.to(torch.float32) * self.scales[li])
            else:
                sx, sw = self.act_scales[li]
                self.ys[li].copy_(acc.to(torch.float32) * (sx * sw).to(torch.float32))

    def run(self, max_ctas: int = 0) -> None:
        self.layers.acc_flat.zero_()
        self.status.zero_()
        if self.epi is not None:
            self.counters.zero_()
        j, ix = self.jobs, self.index
        if self.unit_t.shape[0]:
            nv.call("dc_fused_ring_gemm", self.image.data_ptr(), j.d_blob_off.data_ptr(), j.d_blob_len.data_ptr(),
                    j.d_out_len.data_ptr(), j.d_codec.data_ptr(), self.chunk_size, ix.d_seg_base.data_ptr(),
                    ix.d_state.data_ptr(), ix.d_off.data_ptr(), self.layers.tens.data_ptr(), self.unit_t.data_ptr(),
                    self.unit_t.shape[0], self.layers.ntok, self.status.data_ptr(),
                    self.epi.data_ptr() if self.epi is not None else None, int(max_ctas), nv.stream_ptr())
        if self._fb is not None:
            self._fb.run()
            if self.ys is not None:
                self._fallback_epilogue()

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
            for li, y in enumerate(self.ys):
                acc = self.layers.accs[li]
                if self.scales is not None:
                    y.copy_(acc.to(torch.float32) * self.scales[li])
                else:
                    sx, sw = self.act_scales[li]
                    y.copy_(acc.to(torch.float32) * (sx * sw).to(torch.float32))
        return False


class CompressedLinears:
    """Every linear of a compressed model from floating-point activations in
    one call (W8A8 numerics of scaling.py:127-152 on a decode step):

      1. prologue (dc_act_quant, one CTA per input): X' = X / s (IEEE f64,
         per input channel), sx = max|X'| / 127, qx = round-half-away(X'/sx)
         -- exactly the reference's quantize of X / s;
      2. FusedRing with the device-side dequant epilogue: decode -> TMEM ->
         tcgen05 int8 MMA, exact int32 accumulation, y = acc * (sx * sw) in
         fp32 (any chunk size, see FusedRing).

    ``w_scales[i]`` / ``s_vecs[i]`` (host f64 arrays) are the layers'
    quantization scale and channel scale vector (QuantizedTensor.w_scale /
    scale_vec.s).  ``run(xs)`` takes [ntok, K] fp32 / bf16 / fp16 / f64
    CUDA tensors and returns the fp32 outputs [ntok, rows] per layer."""

    _DT = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2, torch.float16: 3}

    def __init__(self, image, jobs, index, chunk_size: int, shapes, t_offs, w_scales, s_vecs, ntok: int,
                 dtype=torch.float32):
        dev = image.device
        self.ntok, self.dtype, self.shapes = ntok, dtype, [(int(r), int(k)) for r, k in shapes]
        self.x_in = [torch.zeros((ntok, k), dtype=dtype, device=dev) for _, k in self.shapes]
        self.qx = [torch.zeros((ntok, k), dtype=torch.int8, device=dev) for _, k in self.shapes]
        self.sx = torch.zeros(len(self.shapes), dtype=torch.float64, device=dev)
        self.s = [None if s is None else torch.from_numpy(np.ascontiguousarray(s, dtype=np.float64)).to(dev)
                  for s in s_vecs]
        self.act_status = torch.zeros(max(len(self.shapes), 1), dtype=torch.int32, device=dev)
        self.xp = [torch.empty((ntok, k), dtype=torch.float64, device=dev) for _, k in self.shapes]
        self.mbits = torch.zeros(max(len(self.shapes), 1), dtype=torch.int64, device=dev)
        dt = np.dtype([("x", "<u8"), ("s", "<u8"), ("q", "<u8"), ("sx", "<u8"), ("xp", "<u8"), ("mbits", "<u8"),
                       ("k", "<i8")])
        assert dt.itemsize == nv.call("dc_act_quant_bytes")
        t = np.zeros(len(self.shapes), dtype=dt)
        t["x"] = [x.data_ptr() for x in self.x_in]
        t["s"] = [0 if s is None else s.data_ptr() for s in self.s]
        t["q"] = [q.data_ptr() for q in self.qx]
        t["sx"] = [self.sx.data_ptr() + 8 * i for i in range(len(self.shapes))]
        t["xp"] = [x.data_ptr() for x in self.xp]
        t["mbits"] = [self.mbits.data_ptr() + 8 * i for i in range(len(self.shapes))]
        t["k"] = [k for _, k in self.shapes]
        self.table = torch.from_numpy(t.view(np.uint8).copy()).to(dev)
        self.ring = FusedRing(image, jobs, index, chunk_size, self.shapes, t_offs, self.qx, ntok,
                              act_scales=[(self.sx[i:i + 1], float(w)) for i, w in enumerate(w_scales)])

    def prologue(self) -> None:
        self.act_status.zero_()
        self.mbits.zero_()
        nv.call("dc_act_quant", self.table.data_ptr(), len(self.shapes), self._DT[self.dtype], self.ntok,
                max(k for _, k in self.shapes), self.act_status.data_ptr(), nv.stream_ptr())

    def run(self, xs=None, max_ctas: int = 0) -> list[torch.Tensor]:
        """(Copies ``xs`` into the static input buffers, then) prologue + fused
        ring in two launches; returns the fp32 outputs (views of ys)."""
        if xs is not None:
            for buf, x in zip(self.x_in, xs):
                buf.copy_(x)
        self.prologue()
        self.ring.run(max_ctas)
        return self.ring.ys

    def check(self) -> np.ndarray:
        return self.ring.check()


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
