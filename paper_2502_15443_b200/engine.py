"""Device-side engine: chunk job tables, the split-point index, and the
decode / encode pipelines over the C-ABI kernels.

Data layout in HBM:
  * ``base``      uint8: the chunk payloads exactly as in the DCC1 file
                  (the whole file image, or any buffer holding blobs), with
                  READ_SLACK readable bytes past the end.
  * job table     five device arrays (blob_off, blob_len, out_off, out_len,
                  codec), one entry per chunk.
  * SegmentIndex  per ANS chunk ceil(len / 2^shift) split points
                  (state u32, stream offset u32): 8 bytes per segment.  It
                  lives OUTSIDE the DCC1 bytes (which stay bit-exact) and is
                  only an accelerator: the kernels never form an address from
                  a split point outside its chunk's stream span, a wrong one
                  is caught by the chain checks and the chunk is re-decoded
                  exactly, and a sidecar whose body CRC fails is not trusted
                  (every ANS chunk goes to the exact decoder).
"""

from __future__ import annotations

import dataclasses
import math
import os
import struct
import zlib

import numpy as np
import torch

from . import native as nv

HEADER_BYTES = 388
DEFAULT_SEG_SHIFT = 8          # 256-symbol segments: 8 B of index per 256 B of weights
STAGE_SLOP = 16  # staged span = stream bytes + up to 15 B of 16-B alignment


def _dev():
    return nv.require_cuda()


def _t(a: np.ndarray, dtype, device) -> torch.Tensor:
    return torch.from_numpy(np.array(a, copy=True)).to(device=device, dtype=dtype)


@dataclasses.dataclass
class JobTable:
    """Chunk jobs inside one device byte buffer."""

    n: int
    blob_off: np.ndarray   # u64 host copies
    blob_len: np.ndarray
    out_off: np.ndarray
    out_len: np.ndarray
    codec: np.ndarray      # u8
    d_blob_off: torch.Tensor
    d_blob_len: torch.Tensor
    d_out_off: torch.Tensor
    d_out_len: torch.Tensor
    d_codec: torch.Tensor

    @classmethod
    def build(cls, blob_off, blob_len, out_off, out_len, codec, device=None) -> "JobTable":
        dev = device or _dev()
        # np.array copies: a 1-element strided field view counts as "contiguous"
        # for numpy but keeps its 29-byte stride, which torch rejects
        arrs = [np.array(a, dtype=np.uint64) for a in (blob_off, blob_len, out_off, out_len)]
        cod = np.ascontiguousarray(codec, dtype=np.uint8)
        d = [_t(a.view(np.int64), torch.int64, dev) for a in arrs]
        return cls(len(cod), *arrs, cod, *d, _t(cod, torch.uint8, dev))

    @property
    def total_out(self) -> int:
        return int(self.out_off[-1] + self.out_len[-1]) if self.n else 0


@dataclasses.dataclass
class SegmentIndex:
    """Split points of every ANS chunk (device arrays + host copies)."""

    seg_shift: int
    seg_base: np.ndarray       # i64 per chunk (first segment), host
    n_segs: int
    d_seg_base: torch.Tensor   # int64 [n_chunks]
    d_state: torch.Tensor      # int32 storage of u32 [n_segs]
    d_off: torch.Tensor        # int32 storage of u32 [n_segs]
    h_off: np.ndarray | None = None  # host copy of the offsets when already on the host
    # lazy sidecar: pinned host bytes of (state, off) not yet copied; PipelinedDecode
    # uploads each chunk group's split points just ahead of that group's stream bytes
    pending: torch.Tensor | None = None
    # sidecar body CRC still to be checked on the device (pinned sidecars): the
    # device copy of the body (8 * n_segs bytes) and the CRC32 stored after it
    raw: torch.Tensor | None = None
    crc_expected: int | None = None

    @staticmethod
    def layout(out_len: np.ndarray, codec: np.ndarray, seg_shift: int) -> tuple[np.ndarray, int]:
        K = 1 << seg_shift
        nseg = np.where(codec == 1, (out_len.astype(np.int64) + K - 1) // K, 0)
        base = np.zeros(len(nseg), dtype=np.int64)
        if len(nseg):
            base[1:] = np.cumsum(nseg)[:-1]
        return base, int(nseg.sum())

    @classmethod
    def empty(cls, jobs: JobTable, seg_shift: int = DEFAULT_SEG_SHIFT, device=None) -> "SegmentIndex":
        dev = device or _dev()
        base, n = cls.layout(jobs.out_len, jobs.codec, seg_shift)
        return cls(seg_shift, base, n, _t(base, torch.int64, dev),
                   torch.zeros(max(n, 1), dtype=torch.int32, device=dev),
                   torch.zeros(max(n, 1), dtype=torch.int32, device=dev))

    @property
    def nbytes(self) -> int:
        return 8 * self.n_segs

    def upload_segments(self, s0: int, s1: int) -> None:
        """Copy split points [s0, s1) of a lazy index on the current stream."""
        if self.pending is None or s1 <= s0:
            return
        n = self.n_segs
        self.d_state.view(torch.uint8)[4 * s0:4 * s1].copy_(self.pending[4 * s0:4 * s1], non_blocking=True)
        self.d_off.view(torch.uint8)[4 * s0:4 * s1].copy_(self.pending[4 * n + 4 * s0:4 * n + 4 * s1],
                                                          non_blocking=True)

    def ensure_uploaded(self) -> None:
        if self.pending is not None:
            self.upload_segments(0, self.n_segs)
            self.pending = None

    def host_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        self.ensure_uploaded()
        return (self.d_state[: self.n_segs].cpu().numpy().view(np.uint32),
                self.d_off[: self.n_segs].cpu().numpy().view(np.uint32))

    def host_offsets(self) -> np.ndarray:
        if self.h_off is None:
            self.h_off = self.d_off[: self.n_segs].cpu().numpy().view(np.uint32)
        return self.h_off

    # ---- sidecar (".dcidx") -------------------------------------------------
    MAGIC = b"DCIX"

    def to_bytes(self, binding: int) -> bytes:
        st, off = self.host_arrays()
        head = self.MAGIC + struct.pack("<HIIQ", 1, self.seg_shift, binding, self.n_segs)
        body = st.tobytes() + off.tobytes()
        return head + body + struct.pack("<I", zlib.crc32(body))

    @classmethod
    def from_bytes(cls, buf, jobs: JobTable, binding: int, device=None, lazy: bool = False) -> "SegmentIndex | None":
        """Load a sidecar (bytes-like, or a pinned CPU uint8 tensor that is
        copied to the device directly); None if it does not belong to this
        container.  ``lazy`` (pinned tensor only): leave the copy to the
        consumer (PipelinedDecode uploads it group by group)."""
        src = None
        if isinstance(buf, torch.Tensor):
            src, buf = buf, buf.numpy()
        if len(buf) < 26 or bytes(buf[:4]) != cls.MAGIC:
            return None
        ver, shift, bind, n = struct.unpack_from("<HIIQ", buf, 4)
        if ver != 1 or bind != binding or not 6 <= shift <= 10:
            return None
        base, want = cls.layout(jobs.out_len, jobs.codec, shift)
        if n != want or len(buf) != 22 + 8 * n + 4:
            return None
        (crc,) = struct.unpack_from("<I", buf, 22 + 8 * n)
        dev = device or _dev()
        pending = None
        if src is not None and src.is_pinned():
            # the body CRC is checked on the device after the upload
            # (PipelinedDecode.finish, or right here when not lazy)
            d = nv.device_bytes(8 * n, dev)
            if lazy:
                pending = src[22:22 + 8 * n]
            else:
                d[:8 * n].copy_(src[22:22 + 8 * n], non_blocking=True)
                if n and not _device_crc_ok(d, 8 * n, crc):
                    return None
        else:
            if zlib.crc32(memoryview(np.frombuffer(buf, np.uint8, 8 * n, 22))) != crc:
                return None  # damaged sidecar: not trusted (index-less decode)
            d = nv.to_device_bytes(np.frombuffer(buf, np.uint8, 8 * n, 22), dev)  # pinned, pipelined upload
        off = np.frombuffer(buf, np.uint32, n, 22 + 4 * n)
        idx = cls(shift, base, n, _t(base, torch.int64, dev), d[:4 * n].view(torch.int32),
                  d[4 * n:8 * n].view(torch.int32), h_off=off, pending=pending)
        if lazy and pending is not None and n:
            idx.raw, idx.crc_expected = d, crc
        return idx

    def body_crc_ok(self) -> bool:
        """Device check of a lazily uploaded sidecar's body CRC (True when
        there is nothing to check); call after the upload was issued."""
        if self.crc_expected is None:
            return True
        ok = _device_crc_ok(self.raw, 8 * self.n_segs, self.crc_expected)
        self.crc_expected, self.raw = None, None
        return ok

    # ---- work decomposition -------------------------------------------------
    def tasks(self, jobs: JobTable, ok: np.ndarray, max_segs: int | None = None,
              seg_range: tuple[np.ndarray, np.ndarray] | None = None) -> torch.Tensor:
        """int32 [n_tasks, 4] = (chunk, first segment, count, 0): at most
        ``max_segs`` segments and at most the kernel's staging capacity of stream bytes each.
        ``seg_range`` = (first, end) segment per job limits each chunk to that
        segment range (decoding part of a chunk)."""
        mode = decode_mode(jobs)
        max_segs = max_segs or nv.call({"small": "dc_decode_small_segments", "narrow": "dc_decode_narrow_segments",
                                        "wide": "dc_decode_task_segments"}[mode])
        stage_cap = nv.call("dc_decode_stage_cap", 1 if mode == "narrow" else 0) - STAGE_SLOP
        K = 1 << self.seg_shift
        sel = np.nonzero((jobs.codec == 1) & ok & (jobs.out_len > 0))[0]
        nseg = (jobs.out_len[sel].astype(np.int64) + K - 1) // K
        if seg_range is None:
            lo_s, hi_s = np.zeros_like(nseg), nseg
        else:
            lo_s = np.asarray(seg_range[0], dtype=np.int64)[sel]
            hi_s = np.minimum(np.asarray(seg_range[1], dtype=np.int64)[sel], nseg)
            keep = hi_s > lo_s
            sel, nseg, lo_s, hi_s = sel[keep], nseg[keep], lo_s[keep], hi_s[keep]
        ntask = (hi_s - lo_s + max_segs - 1) // max_segs
        chunk = np.repeat(sel, ntask)
        first_task = np.repeat(np.cumsum(ntask) - ntask, ntask)
        s0 = np.repeat(lo_s, ntask) + (np.arange(int(ntask.sum())) - first_task) * max_segs
        nsg = np.repeat(nseg, ntask)
        cnt = np.minimum(max_segs, np.repeat(hi_s, ntask) - s0)
        # stream byte span per task: split the (rare) ones that overflow staging
        off = self.host_offsets()
        base = self.seg_base[chunk]
        plen = jobs.blob_len[chunk].astype(np.int64) - HEADER_BYTES
        lo = off[base + s0].astype(np.int64)
        end = s0 + cnt
        hi = np.where(end < nsg, off[np.minimum(base + end, max(self.n_segs - 1, 0))].astype(np.int64), plen)
        # tasks whose staged stream bytes overflow shared memory are halved
        # (vectorized, level by level) until every task fits
        nmax = max(self.n_segs - 1, 0)
        split = False
        for _ in range(32):
            big = (hi - lo + 15 > stage_cap) & (cnt > 1)
            if not big.any():
                break
            split = True
            h = cnt[big] // 2
            k_chunk, k_s0, k_cnt, k_nsg, k_base, k_plen = (chunk[big], s0[big], cnt[big], nsg[big], base[big],
                                                           plen[big])
            keep = ~big
            chunk = np.concatenate([chunk[keep], k_chunk, k_chunk])
            s0 = np.concatenate([s0[keep], k_s0, k_s0 + h])
            cnt = np.concatenate([cnt[keep], h, k_cnt - h])
            nsg = np.concatenate([nsg[keep], k_nsg, k_nsg])
            base = np.concatenate([base[keep], k_base, k_base])
            plen = np.concatenate([plen[keep], k_plen, k_plen])
            lo = off[base + s0].astype(np.int64)
            end = s0 + cnt
            hi = np.where(end < nsg, off[np.minimum(base + end, nmax)].astype(np.int64), plen)
        if split:  # back to (chunk, first segment) order
            order = np.lexsort((s0, chunk))
            chunk, s0, cnt = chunk[order], s0[order], cnt[order]
        # pinned + async: a pageable copy would block the host behind any
        # large H2D already queued on the copy engine
        pin = torch.zeros((len(chunk), 4), dtype=torch.int32, pin_memory=True)
        out = pin.numpy()
        out[:, 0], out[:, 1], out[:, 2] = chunk, s0, cnt
        self.last_tasks_host = out
        return pin.to(_dev(), non_blocking=True)


def _device_crc_ok(buf: torch.Tensor, nbytes: int, want: int) -> bool:
    off = torch.zeros(1, dtype=torch.int64, device=buf.device)
    ln = torch.full((1,), nbytes, dtype=torch.int64, device=buf.device)
    got = crc32_ranges(buf, off, ln, nbytes)
    return int(got.item()) & 0xFFFFFFFF == want


# ------------------------------------------------------------------ decode
def validate(base: torch.Tensor, jobs: JobTable, status: torch.Tensor) -> None:
    nv.call("dc_ans_validate", base.data_ptr(), jobs.d_blob_off.data_ptr(), jobs.d_blob_len.data_ptr(),
            jobs.d_out_len.data_ptr(), jobs.d_codec.data_ptr(), jobs.n, status.data_ptr(), nv.stream_ptr())


def decode_serial(base, jobs: JobTable, ids: np.ndarray, out: torch.Tensor, status: torch.Tensor,
                  index: SegmentIndex | None = None) -> None:
    if len(ids) == 0:
        return
    d_ids = torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int32)).to(out.device)
    nv.call("dc_ans_decode_serial", base.data_ptr(), jobs.d_blob_off.data_ptr(), jobs.d_blob_len.data_ptr(),
            jobs.d_out_off.data_ptr(), jobs.d_out_len.data_ptr(), d_ids.data_ptr(), len(ids), out.data_ptr(),
            index.seg_shift if index else 0, index.d_seg_base.data_ptr() if index else None,
            index.d_state.data_ptr() if index else None, index.d_off.data_ptr() if index else None,
            status.data_ptr(), nv.stream_ptr())


def small_mode(jobs: JobTable) -> bool:
    """Every chunk small enough for the warp-task decoder (k_decode_small):
    its tasks are warp-sized, so SegmentIndex.tasks and the kernel choice
    both follow this one predicate."""
    lim = int(os.environ.get("DCOMP_SMALL_MAX_CHUNK", "0")) or nv.call("dc_decode_small_max_chunk")
    return jobs.n > 0 and int(jobs.out_len.max()) <= lim


def segment_kernel(jobs: JobTable) -> str:
    return {"small": "dc_ans_decode_small", "narrow": "dc_ans_decode_segments_narrow",
            "wide": "dc_ans_decode_segments"}[decode_mode(jobs)]


def decode_mode(jobs: JobTable) -> str:
    """Which split-point decoder the chunk sizes call for (one predicate shared
    by SegmentIndex.tasks and segment_kernel): "small" (warp tasks, chunks <=
    32 KiB), "narrow" (4-warp CTAs, 256-segment tasks, chunks <= 64 KiB by
    default, DCOMP_NARROW_MAX_CHUNK overrides) or "wide" (8-warp CTAs)."""
    if small_mode(jobs):
        return "small"
    lim = int(os.environ.get("DCOMP_NARROW_MAX_CHUNK", str(NARROW_MAX_CHUNK)))
    return "narrow" if jobs.n > 0 and int(jobs.out_len.max()) <= lim else "wide"


NARROW_MAX_CHUNK = 64 << 10


def decode_segments(base, jobs: JobTable, index: SegmentIndex, tasks: torch.Tensor, out: torch.Tensor,
                    status: torch.Tensor) -> None:
    if tasks.shape[0] == 0:
        return
    nv.call(segment_kernel(jobs), base.data_ptr(), jobs.d_blob_off.data_ptr(), jobs.d_blob_len.data_ptr(),
            jobs.d_out_off.data_ptr(), jobs.d_out_len.data_ptr(), index.seg_shift, index.d_seg_base.data_ptr(),
            index.d_state.data_ptr(), index.d_off.data_ptr(), tasks.data_ptr(), tasks.shape[0], out.data_ptr(),
            status.data_ptr(), nv.stream_ptr())


def store_copy(base, jobs: JobTable, out: torch.Tensor) -> None:
    if not (jobs.codec == 0).any():
        return
    nv.call("dc_store_copy", base.data_ptr(), jobs.d_blob_off.data_ptr(), jobs.d_out_off.data_ptr(),
            jobs.d_out_len.data_ptr(), jobs.d_codec.data_ptr(), jobs.n, out.data_ptr(), nv.stream_ptr())


def crc32_ranges(data: torch.Tensor, d_off: torch.Tensor, d_len: torch.Tensor, max_len: int) -> torch.Tensor:
    n = d_off.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.int32, device=data.device)
    if n:
        nv.call("dc_crc32_ranges", data.data_ptr(), data.numel() * data.element_size(), d_off.data_ptr(),
                d_len.data_ptr(), n, int(max_len),
                out.data_ptr(), nv.stream_ptr())
    return out[:n]


@dataclasses.dataclass
class DecodeResult:
    out: torch.Tensor          # uint8 [total]
    status: np.ndarray         # int32 per chunk (DC_CHUNK_*)
    index: SegmentIndex | None


def decode_jobs(base: torch.Tensor, jobs: JobTable, index: SegmentIndex | None = None,
                build_index: bool = False, seg_shift: int = DEFAULT_SEG_SHIFT,
                tasks: torch.Tensor | None = None, out: torch.Tensor | None = None) -> DecodeResult:
    """Decode every job into one device buffer.  With an index: segment-
    parallel kernel (+ exact serial re-run of chunks whose chain breaks).
    Without: exact serial kernel per chunk (optionally recording an index)."""
    dev = base.device
    if out is None:
        out = nv.device_bytes(jobs.total_out, dev)
    status = torch.zeros(max(jobs.n, 1), dtype=torch.int32, device=dev)
    validate(base, jobs, status)
    st = status[: jobs.n].cpu().numpy()
    ok = st == nv.CHUNK_OK
    ans_ids = np.nonzero((jobs.codec == 1) & ok & (jobs.out_len > 0))[0]
    if index is None and build_index:
        index = SegmentIndex.empty(jobs, seg_shift, dev)
        decode_serial(base, jobs, ans_ids, out, status, index)
    elif index is None:
        decode_serial(base, jobs, ans_ids, out, status, None)
    else:
        if tasks is None:
            tasks = index.tasks(jobs, ok)
        decode_segments(base, jobs, index, tasks, out, status)
        st = status[: jobs.n].cpu().numpy()
        redo = np.nonzero(st == nv.CHUNK_CHAIN)[0]
        if len(redo):
            decode_serial(base, jobs, redo, out, status, None)
    store_copy(base, jobs, out)
    return DecodeResult(out, status[: jobs.n].cpu().numpy(), index)


# ------------------------------------------------------------------ encode
@dataclasses.dataclass
class EncodeResult:
    n: int
    chunk_size: int
    total: int
    codec: np.ndarray          # u8: 1 = ANS blob, 0 = stored
    comp_len: np.ndarray       # u64 per chunk
    crc: np.ndarray            # u32 per chunk (uncompressed bytes)
    freq: torch.Tensor         # int32 [n, 256]
    d_tables: torch.Tensor     # uint8 [n, 384]
    d_state: torch.Tensor      # int32 [n] (u32)
    d_stream_len: torch.Tensor  # int64 [n]
    scratch: torch.Tensor      # uint8 [total] encoder output slots
    index: SegmentIndex | None


def encode_payload(payload: torch.Tensor, chunk_size: int, mask: np.ndarray | None,
                   seg_shift: int | None = DEFAULT_SEG_SHIFT) -> EncodeResult:
    """Histogram -> normalize -> reverse encode every chunk selected by
    ``mask`` (None = all); decide codec per chunk like container.pack."""
    dev = payload.device
    total = int(payload.numel())
    n = math.ceil(total / chunk_size) if total else 0
    sp = nv.stream_ptr()
    mask = np.ones(n, bool) if mask is None else np.asarray(mask, bool)
    lens = np.minimum(chunk_size, total - np.arange(n, dtype=np.int64) * chunk_size).astype(np.uint64)
    hist = torch.empty((max(n, 1), 256), dtype=torch.int32, device=dev)
    freq = torch.empty((max(n, 1), 256), dtype=torch.int32, device=dev)
    tables = torch.empty((max(n, 1), 384), dtype=torch.uint8, device=dev)
    state = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    slen = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    scratch = nv.device_bytes(total, dev)
    index = None
    if n:
        nv.call("dc_hist_chunks", payload.data_ptr(), total, chunk_size, n, hist.data_ptr(), sp)
        nv.call("dc_normalize_tables", hist.data_ptr(), n, freq.data_ptr(), tables.data_ptr(), sp)
        todo = torch.from_numpy(mask.astype(np.uint8)).to(dev)
        if seg_shift is not None:
            base_np, nseg = SegmentIndex.layout(lens, np.where(mask, 1, 0).astype(np.uint8), seg_shift)
            index = SegmentIndex(seg_shift, base_np, nseg, _t(base_np, torch.int64, dev),
                                 torch.zeros(max(nseg, 1), dtype=torch.int32, device=dev),
                                 torch.zeros(max(nseg, 1), dtype=torch.int32, device=dev))
        work, wbytes = nv.encode_work(total, chunk_size, n, dev)
        nv.call("dc_ans_encode_chunks", payload.data_ptr(), total, chunk_size, n, todo.data_ptr(),
                freq.data_ptr(), scratch.data_ptr(), state.data_ptr(), slen.data_ptr(),
                seg_shift if index else 0, index.d_seg_base.data_ptr() if index else None,
                index.d_state.data_ptr() if index else None, index.d_off.data_ptr() if index else None, 0,
                work.data_ptr(), wbytes, sp)
        del work  # stream-ordered reuse by the caching allocator
    d_off = torch.from_numpy((np.arange(n, dtype=np.int64) * chunk_size)).to(dev)
    d_len = torch.from_numpy(lens.view(np.int64)).to(dev)
    crc = crc32_ranges(payload, d_off, d_len, min(chunk_size, total)).cpu().numpy().view(np.uint32)
    sl = slen[:n].cpu().numpy().view(np.uint64)
    is_ans = mask & (sl != np.uint64(0xFFFFFFFFFFFFFFFF))
    comp = np.where(is_ans, sl + HEADER_BYTES, lens).astype(np.uint64)
    codec = is_ans.astype(np.uint8)
    if index is not None:
        # encoder recorded (state, bytes emitted so far); decoder offset = total - emitted
        d_codec = torch.from_numpy(codec).to(dev)
        seg_chunk = torch.repeat_interleave(
            torch.arange(n, device=dev),
            torch.from_numpy(np.where(mask, (lens.astype(np.int64) + (1 << seg_shift) - 1) >> seg_shift, 0)).to(dev))
        if index.n_segs:
            sl_t = slen[:n]
            emitted = index.d_off[: index.n_segs].to(torch.int64) & 0xFFFFFFFF
            offs = sl_t[seg_chunk] - emitted
            index.d_off[: index.n_segs] = offs.to(torch.int32)
        # chunks that ended up stored carry no segments: rebuild a compact index
        if not is_ans.all() and index.n_segs:
            keep_seg = d_codec[seg_chunk].bool()
            base_np, nseg = SegmentIndex.layout(lens, codec, seg_shift)
            index = SegmentIndex(seg_shift, base_np, nseg, _t(base_np, torch.int64, dev),
                                 index.d_state[: index.n_segs][keep_seg].contiguous(),
                                 index.d_off[: index.n_segs][keep_seg].contiguous())
            if nseg == 0:
                index.d_state = torch.zeros(1, dtype=torch.int32, device=dev)
                index.d_off = torch.zeros(1, dtype=torch.int32, device=dev)
    return EncodeResult(n, chunk_size, total, codec, comp, crc, freq, tables, state, slen, scratch, index)


def assemble(payload: torch.Tensor, enc: EncodeResult, file_off: np.ndarray, dst: torch.Tensor) -> None:
    if enc.n == 0:
        return
    dev = payload.device
    d_codec = torch.from_numpy(enc.codec).to(dev)
    d_foff = torch.from_numpy(np.ascontiguousarray(file_off, dtype=np.uint64).view(np.int64)).to(dev)
    nv.call("dc_assemble_payloads", payload.data_ptr(), enc.total, enc.chunk_size, enc.n, d_codec.data_ptr(),
            enc.d_tables.data_ptr(), enc.d_state.data_ptr(), enc.d_stream_len.data_ptr(), enc.scratch.data_ptr(),
            d_foff.data_ptr(), dst.data_ptr(), nv.stream_ptr())


# --------------------------------------------------------- pipelined decode
_SIDE_STREAMS: dict = {}


def _streams(dev):
    if dev not in _SIDE_STREAMS:
        _SIDE_STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _SIDE_STREAMS[dev]


_TIMELINE = os.environ.get("DCOMP_TIMELINE") == "1"


class PipelinedDecode:
    """Host container bytes -> host decoded bytes: H2D of chunk group g+1,
    validate + split-point decode + CRC of group g and D2H of group g-1
    overlapped on three streams.  ``src`` is the file as a uint8 numpy array
    (pageable: staged through pinned buffers) or a pinned CPU uint8 tensor
    (copied directly).  The constructor only enqueues work; ``host_out`` may
    be wrapped (views) before ``finish()``, which waits, re-decodes chunks
    whose split-point chain broke (exact serial kernel) and returns
    (decoded host bytes, per-chunk status, per-chunk CRC32)."""

    LOOKAHEAD = int(os.environ.get("DCOMP_H2D_LOOKAHEAD", "2"))

    GROUPS = int(os.environ.get("DCOMP_E2E_GROUPS", "16"))

    D2H_SPLIT = int(os.environ.get("DCOMP_D2H_SPLIT", "2"))  # measured: 45.5 -> 47.2 GB/s e2e (OPT-6.7B)

    def __init__(self, src, jobs: JobTable, index: SegmentIndex, groups: int | None = None):
        groups = groups or self.GROUPS
        dev = jobs.d_blob_off.device
        self.dev, self.jobs = dev, jobs
        s_copy, s_out, s_out2 = _streams(dev)
        s_comp = torch.cuda.current_stream(dev)
        self.s_comp = s_comp
        n = jobs.n
        pinned = isinstance(src, torch.Tensor)
        size = src.numel() if pinned else src.size
        self.image = image = nv.device_bytes(size, dev)
        self.out = out = nv.device_bytes(jobs.total_out, dev)
        self.host_out = host_out = torch.empty(jobs.total_out, dtype=torch.uint8, pin_memory=True)
        self.status = status = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.crc = crc = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self.marks = marks = [] if _TIMELINE else None
        self._mark("init", s_comp)
        # contiguous chunk groups: a short ramp (1/128, 1/32, 1/16 of the file)
        # so the first D2H starts early, then ~equal file bytes
        ends = jobs.blob_off + jobs.blob_len
        fr = np.array([1 / 128, 1 / 32, 1 / 16]) if groups >= 8 else np.zeros(0)
        fr = np.concatenate([fr, np.full(groups - len(fr), (1 - fr.sum()) / (groups - len(fr)))])
        cuts = np.searchsorted(np.cumsum(jobs.blob_len.astype(np.float64)),
                               np.cumsum(fr)[:-1] * float(jobs.blob_len.sum())).tolist()
        bounds = sorted(set([0] + [min(max(c + 1, 1), n) for c in cuts] + [n]))
        grp = list(zip(bounds, bounds[1:]))
        lazy = index.pending is not None
        seg_end = np.append(index.seg_base, index.n_segs)
        ev_h2d, ev_d2h = {}, {}

        def issue_h2d(i):
            # H2D runs at most LOOKAHEAD groups ahead of the D2H: the link is
            # shared by both directions and the (larger) D2H is the long pole
            g0, g1 = grp[i]
            f0, f1 = int(jobs.blob_off[g0]), int(ends[g1 - 1])
            if pinned:
                stage = src[f0:f1]
            else:
                stage = torch.empty(f1 - f0, dtype=torch.uint8, pin_memory=True)
                nv._parallel_copy(stage.numpy(), src[f0:f1], piece=8 << 20)
            with torch.cuda.stream(s_copy):
                if i - self.LOOKAHEAD in ev_d2h:
                    s_copy.wait_event(ev_d2h[i - self.LOOKAHEAD])
                self._mark(f"h2d{g0}", s_copy)
                if lazy:
                    index.upload_segments(int(seg_end[g0]), int(seg_end[g1]))
                image[f0:f1].copy_(stage, non_blocking=True)
                ev_h2d[i] = torch.cuda.Event()
                ev_h2d[i].record(s_copy)
                self._mark(f"h2d{g0}_end", s_copy)

        for i in range(min(self.LOOKAHEAD, len(grp))):
            issue_h2d(i)
        sp_comp = s_comp.cuda_stream
        self.max_len = max_len = int(jobs.out_len.max()) if n else 0
        self._keep = []
        for i, (g0, g1) in enumerate(grp):
            sel = np.zeros(n, bool)
            sel[g0:g1] = True
            tasks = index.tasks(jobs, sel)  # per group: the first decode issues early
            self._keep.append(tasks)
            s_comp.wait_event(ev_h2d[i])
            k = g1 - g0
            off8 = lambda t: t.data_ptr() + 8 * g0  # noqa: E731
            nv.call("dc_ans_validate", image.data_ptr(), off8(jobs.d_blob_off), off8(jobs.d_blob_len),
                    off8(jobs.d_out_len), jobs.d_codec.data_ptr() + g0, k, status.data_ptr() + 4 * g0, sp_comp)
            if tasks.shape[0]:
                nv.call(segment_kernel(jobs), image.data_ptr(), jobs.d_blob_off.data_ptr(),
                        jobs.d_blob_len.data_ptr(), jobs.d_out_off.data_ptr(), jobs.d_out_len.data_ptr(),
                        index.seg_shift, index.d_seg_base.data_ptr(), index.d_state.data_ptr(),
                        index.d_off.data_ptr(), tasks.data_ptr(), tasks.shape[0], out.data_ptr(),
                        status.data_ptr(), sp_comp)
            nv.call("dc_store_copy", image.data_ptr(), off8(jobs.d_blob_off), off8(jobs.d_out_off),
                    off8(jobs.d_out_len), jobs.d_codec.data_ptr() + g0, k, out.data_ptr(), sp_comp)
            nv.call("dc_crc32_ranges", out.data_ptr(), out.numel(), off8(jobs.d_out_off), off8(jobs.d_out_len), k,
                    max_len,
                    crc.data_ptr() + 4 * g0, sp_comp)
            ev_dec = torch.cuda.Event()
            ev_dec.record(s_comp)
            s_out.wait_event(ev_dec)
            o0 = int(jobs.out_off[g0])
            o1 = int(jobs.out_off[g1 - 1] + jobs.out_len[g1 - 1])
            self._mark(f"dec{g0}_end", s_comp)
            with torch.cuda.stream(s_out):
                self._mark(f"d2h{g0}", s_out)
                if self.D2H_SPLIT > 1 and o1 - o0 >= (8 << 20):
                    # two copies in flight (two copy engines) for the larger direction
                    mid = o0 + (((o1 - o0) // 2) & ~4095)
                    s_out2.wait_event(ev_dec)
                    with torch.cuda.stream(s_out2):
                        host_out[mid:o1].copy_(out[mid:o1], non_blocking=True)
                        ev2 = torch.cuda.Event()
                        ev2.record(s_out2)
                    host_out[o0:mid].copy_(out[o0:mid], non_blocking=True)
                    s_out.wait_event(ev2)
                else:
                    host_out[o0:o1].copy_(out[o0:o1], non_blocking=True)
                ev_d2h[i] = torch.cuda.Event()
                ev_d2h[i].record(s_out)
                self._mark(f"d2h{g0}_end", s_out)
            if i + self.LOOKAHEAD < len(grp):
                issue_h2d(i + self.LOOKAHEAD)
        if lazy:  # every group's split points are in flight on s_copy
            index.pending = None
            s_comp.wait_stream(s_copy)
        self.index = index
        self._mark("issued", None)

    def _mark(self, name, stream):
        """DCOMP_TIMELINE=1: device events (and host issue times) per pipeline stage."""
        if self.marks is None:
            return
        import time
        ev = None
        if stream is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
        self.marks.append((name, time.perf_counter(), ev))

    def timeline(self) -> list[tuple[str, float, float]]:
        """(stage, host issue ms, device ms) relative to construction; after finish()."""
        if not self.marks:
            return []
        h0, e0 = self.marks[0][1], self.marks[0][2]
        return [(nm, (h - h0) * 1e3, e0.elapsed_time(ev) if ev is not None else float("nan"))
                for nm, h, ev in self.marks]

    def finish(self):
        jobs, n, out, host_out = self.jobs, self.jobs.n, self.out, self.host_out
        torch.cuda.synchronize(self.dev)
        st = self.status[:n].cpu().numpy()
        redo = np.nonzero(st == nv.CHUNK_CHAIN)[0]
        if not self.index.body_crc_ok():  # damaged sidecar: every ANS chunk by the exact decoder
            redo = np.nonzero((st == nv.CHUNK_OK) | (st == nv.CHUNK_CHAIN))[0]
            redo = redo[(jobs.codec[redo] == 1) & (jobs.out_len[redo] > 0)]
        if len(redo):  # broken split points: exact serial decode, then refresh CRC + host bytes
            decode_serial(self.image, jobs, redo, out, self.status, None)
            nv.call("dc_crc32_ranges", out.data_ptr(), out.numel(), jobs.d_out_off.data_ptr(), jobs.d_out_len.data_ptr(), n,
                    self.max_len, self.crc.data_ptr(), self.s_comp.cuda_stream)
            torch.cuda.synchronize(self.dev)
            for c in redo:
                a, b = int(jobs.out_off[c]), int(jobs.out_off[c] + jobs.out_len[c])
                host_out[a:b].copy_(out[a:b])
            st = self.status[:n].cpu().numpy()
        return host_out.numpy(), st, self.crc[:n].cpu().numpy().view(np.uint32)


def decode_file_pipelined(data, jobs: JobTable, index: SegmentIndex, groups: int | None = None):
    """One-shot PipelinedDecode (see there)."""
    return PipelinedDecode(data, jobs, index, groups).finish()
