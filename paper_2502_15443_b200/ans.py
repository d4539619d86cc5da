"""Static-table rANS over bytes -- the reference's ans.py API, B200 kernels.

Same wire form as the reference (ans.py:1-12):

    blob = packed table (256 x u12 = 384 B) | start state (u32 LE) | stream

and the same names, signatures, errors and messages.  Entropy coding runs on
the GPU: ``AnsTable.for_data`` (histogram + exact normalization),
``ans_compress``/``compress_blob`` (reverse encoder) and every decoder
(``decompress_into``, ``ans_decompress``, ``decompress_blob``,
``decode_blobs_into``).  The 384-byte table packing / parsing helpers are
host-side format code.
"""

from __future__ import annotations

import dataclasses
import struct

import numpy as np
import torch

from . import engine
from . import native as nv
from .errors import CorruptStreamError, DcompError, TruncatedError

PROB_BITS = 12
PROB_SCALE = 1 << PROB_BITS
STATE_LOWER = 1 << 20
STATE_UPPER = 1 << 28
TABLE_BYTES = 384
HEADER_BYTES = TABLE_BYTES + 4


def _as_u8(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        if data.dtype == np.int8:
            data = data.view(np.uint8)
        elif data.dtype != np.uint8:
            raise TypeError(f"expected byte data, got dtype {data.dtype}")
        return np.ascontiguousarray(data.reshape(-1))
    return np.frombuffer(bytes(data), dtype=np.uint8)


def _pack_u12(freq: np.ndarray) -> bytes:
    f = np.minimum(np.asarray(freq, dtype=np.uint32), PROB_SCALE - 1)
    lo, hi = f[0::2], f[1::2]
    out = np.empty(TABLE_BYTES, dtype=np.uint8)
    out[0::3] = lo & 0xFF
    out[1::3] = ((lo >> 8) & 0x0F) | ((hi & 0x0F) << 4)
    out[2::3] = hi >> 4
    return out.tobytes()


def _unpack_u12(buf) -> np.ndarray:
    raw = np.frombuffer(bytes(buf), dtype=np.uint8).astype(np.uint32)
    f = np.empty(256, dtype=np.uint32)
    f[0::2] = raw[0::3] | ((raw[1::3] & 0x0F) << 8)
    f[1::2] = (raw[1::3] >> 4) | (raw[2::3] << 4)
    return f


@dataclasses.dataclass(frozen=True)
class AnsTable:
    frequencies: np.ndarray  # (256,) uint32, sums to 4096

    def __post_init__(self):
        f = np.ascontiguousarray(self.frequencies, dtype=np.uint32)
        if f.shape != (256,):
            raise ValueError("frequency table must have 256 entries")
        if int(f.sum()) != PROB_SCALE:
            raise ValueError(f"frequencies sum to {int(f.sum())}, expected {PROB_SCALE}")
        object.__setattr__(self, "frequencies", f)

    @classmethod
    def for_data(cls, data) -> "AnsTable":
        """GPU histogram + exact largest-remainder normalization."""
        u8 = _as_u8(data)
        if u8.size == 0:
            raise DcompError("empty input")
        dev = nv.require_cuda()
        d = nv.to_device_bytes(u8, dev)
        hist = torch.empty((1, 256), dtype=torch.int32, device=dev)
        freq = torch.empty((1, 256), dtype=torch.int32, device=dev)
        tb = torch.empty((1, TABLE_BYTES), dtype=torch.uint8, device=dev)
        sp = nv.stream_ptr()
        nv.call("dc_hist_chunks", d.data_ptr(), u8.size, u8.size, 1, hist.data_ptr(), sp)
        nv.call("dc_normalize_tables", hist.data_ptr(), 1, freq.data_ptr(), tb.data_ptr(), sp)
        return cls(freq[0].cpu().numpy().view(np.uint32))

    def to_bytes(self) -> bytes:
        return _pack_u12(self.frequencies)

    @classmethod
    def from_bytes(cls, buf) -> "AnsTable":
        if len(buf) != TABLE_BYTES:
            raise CorruptStreamError("corrupt stream: bad table size")
        f = _unpack_u12(buf)
        total = int(f.sum())
        if total == PROB_SCALE - 1 and np.count_nonzero(f) == 1:
            f = f.copy()
            f[int(np.argmax(f))] = PROB_SCALE  # single-symbol stream
        elif total != PROB_SCALE:
            raise CorruptStreamError("corrupt stream: invalid frequency table")
        return cls(f)

    def cumulative(self) -> np.ndarray:
        c = np.zeros(256, dtype=np.uint32)
        c[1:] = np.cumsum(self.frequencies)[:-1]
        return c

    def decode_table(self) -> np.ndarray:
        """Slot table (API compatibility): freq | offset << 16 | symbol << 32."""
        f = self.frequencies.astype(np.uint64)
        counts = self.frequencies
        sym = np.repeat(np.arange(256, dtype=np.uint64), counts)
        off = np.arange(PROB_SCALE, dtype=np.uint64) - np.repeat(self.cumulative().astype(np.uint64), counts)
        return np.repeat(f, counts) | (off << np.uint64(16)) | (sym << np.uint64(32))


# ------------------------------------------------------------------ encode
def _encode_one(u8: np.ndarray) -> tuple[np.ndarray, bytes, int]:
    """GPU encode of one standalone blob: (freq, stream in decoder order, state)."""
    dev = nv.require_cuda()
    n = u8.size
    d = nv.to_device_bytes(u8, dev)
    hist = torch.empty((1, 256), dtype=torch.int32, device=dev)
    freq = torch.empty((1, 256), dtype=torch.int32, device=dev)
    tb = torch.empty((1, TABLE_BYTES), dtype=torch.uint8, device=dev)
    state = torch.empty(1, dtype=torch.int32, device=dev)
    slen = torch.empty(1, dtype=torch.int64, device=dev)
    todo = torch.ones(1, dtype=torch.uint8, device=dev)
    room = 2 * n + 8                     # worst case: 2 bytes per symbol (+ slop)
    scratch = nv.device_bytes(room, dev)
    slot = scratch.data_ptr() + room - n  # slot [slot, slot + n) ends at scratch end
    sp = nv.stream_ptr()
    nv.call("dc_hist_chunks", d.data_ptr(), n, n, 1, hist.data_ptr(), sp)
    nv.call("dc_normalize_tables", hist.data_ptr(), 1, freq.data_ptr(), tb.data_ptr(), sp)
    work, wbytes = nv.encode_work(n, n, 1, dev)
    nv.call("dc_ans_encode_chunks", d.data_ptr(), n, n, 1, todo.data_ptr(), freq.data_ptr(), slot,
            state.data_ptr(), slen.data_ptr(), 0, None, None, None, 1, work.data_ptr(), wbytes, sp)
    sl = int(slen.item())
    stream = scratch[room - sl:room].cpu().numpy().tobytes() if sl else b""
    return freq[0].cpu().numpy().view(np.uint32), stream, int(state.item()) & 0xFFFFFFFF


def compress_blobs(pieces: list[np.ndarray], streams: int = 16) -> list[bytes]:
    """compress_blob() of many byte arrays at once: every blob's serial encode
    chain runs concurrently (one warp each, side CUDA streams), so the batch
    costs about one (largest) blob instead of their sum."""
    dev = nv.require_cuda()
    n = len(pieces)
    if n == 0:
        return []
    sizes = [int(p.size) for p in pieces]
    if min(sizes) == 0:
        raise DcompError("empty input")
    src = nv.to_device_bytes(np.concatenate([np.asarray(p, dtype=np.uint8).reshape(-1) for p in pieces]), dev)
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    hist = torch.empty((n, 256), dtype=torch.int32, device=dev)
    freq = torch.empty((n, 256), dtype=torch.int32, device=dev)
    tb = torch.empty((n, TABLE_BYTES), dtype=torch.uint8, device=dev)
    state = torch.empty(n, dtype=torch.int32, device=dev)
    slen = torch.empty(n, dtype=torch.int64, device=dev)
    todo = torch.ones(n, dtype=torch.uint8, device=dev)
    main = torch.cuda.current_stream(dev)
    ss = [torch.cuda.Stream(dev) for _ in range(min(streams, n))]
    keep = []
    for i, (m, o) in enumerate(zip(sizes, offs)):
        st = ss[i % len(ss)]
        st.wait_stream(main)
        with torch.cuda.stream(st):
            room = 2 * m + 8  # worst case: 2 bytes per symbol (+ slop)
            scratch = nv.device_bytes(room, dev)
            work, wbytes = nv.encode_work(m, m, 1, dev)
            keep.append((scratch, work, room))
            p = src.data_ptr() + int(o)
            sp = st.cuda_stream
            nv.call("dc_hist_chunks", p, m, m, 1, hist[i].data_ptr(), sp)
            nv.call("dc_normalize_tables", hist[i].data_ptr(), 1, freq[i].data_ptr(), tb[i].data_ptr(), sp)
            nv.call("dc_ans_encode_chunks", p, m, m, 1, todo[i:i + 1].data_ptr(), freq[i].data_ptr(),
                    scratch.data_ptr() + room - m, state[i:i + 1].data_ptr(), slen[i:i + 1].data_ptr(), 0, None,
                    None, None, 1, work.data_ptr(), wbytes, sp)
    for st in ss:
        main.wait_stream(st)
    sl = slen.cpu().numpy()
    x0 = state.cpu().numpy().view(np.uint32)
    tables = tb.cpu().numpy()
    out = []
    for i, (scratch, _, room) in enumerate(keep):
        k = int(sl[i])
        stream = scratch[room - k:room].cpu().numpy().tobytes() if k else b""
        out.append(tables[i].tobytes() + struct.pack("<I", int(x0[i])) + stream)
    return out


def ans_compress(data) -> tuple[AnsTable, bytes]:
    """Compress bytes; returns (table, payload = state u32 LE + stream)."""
    u8 = _as_u8(data)
    if u8.size == 0:
        raise DcompError("empty input")
    freq, stream, state = _encode_one(u8)
    return AnsTable(freq), struct.pack("<I", state) + stream


def compress_blob(data) -> bytes:
    table, payload = ans_compress(data)
    return table.to_bytes() + payload


# ------------------------------------------------------------------ decode
def split_blob(blob) -> tuple[AnsTable, bytes]:
    if len(blob) < HEADER_BYTES:
        raise TruncatedError("truncated stream: missing table header")
    return AnsTable.from_bytes(blob[:TABLE_BYTES]), blob[TABLE_BYTES:]


_PROLOGUE = {
    nv.CHUNK_TRUNC_TABLE: (TruncatedError, "truncated stream: missing table header"),
    nv.CHUNK_BAD_TABLE: (CorruptStreamError, "corrupt stream: invalid frequency table"),
    nv.CHUNK_STATE_RANGE: (CorruptStreamError, "corrupt stream: final state out of range"),
    nv.CHUNK_EMPTY_BAD: (CorruptStreamError, "corrupt stream"),
}


def _stage_blobs(blobs: list[bytes], out_lens: list[int]):
    """Concatenate blobs into one device buffer; outputs at 16-byte aligned offsets."""
    dev = nv.require_cuda()
    lens = np.array([len(b) for b in blobs], dtype=np.uint64)
    boff = np.zeros(len(blobs), dtype=np.uint64)
    if len(blobs):
        boff[1:] = np.cumsum(lens)[:-1]
    olen = np.array(out_lens, dtype=np.uint64)
    ooff = np.zeros(len(blobs), dtype=np.uint64)
    if len(blobs):
        aligned = (olen + np.uint64(15)) & ~np.uint64(15)
        ooff[1:] = np.cumsum(aligned)[:-1]
    base = nv.to_device_bytes(b"".join(blobs), dev)
    codec = np.ones(len(blobs), dtype=np.uint8)
    jobs = engine.JobTable.build(boff, lens, ooff, olen, codec, dev)
    return base, jobs


def _decode_many(blobs: list[bytes], out_lens: list[int]):
    base, jobs = _stage_blobs(blobs, out_lens)
    res = engine.decode_jobs(base, jobs)
    return res, jobs


def decompress_into(table: AnsTable, payload, out: np.ndarray) -> None:
    """Decode a payload (state + stream) into a preallocated uint8 array."""
    if len(payload) < 4:
        raise TruncatedError("truncated stream: missing final state")
    (state,) = struct.unpack_from("<I", payload)
    if not STATE_LOWER <= state < STATE_UPPER:
        raise CorruptStreamError("corrupt stream: final state out of range")
    if out.size == 0:
        if len(payload) != 4 or state != STATE_LOWER:
            raise CorruptStreamError("corrupt stream")
        return
    res, jobs = _decode_many([table.to_bytes() + bytes(payload)], [out.size])
    if res.status[0] != nv.CHUNK_OK:
        raise CorruptStreamError("corrupt stream")
    out.reshape(-1).view(np.uint8)[:] = res.out[: out.size].cpu().numpy()


def ans_decompress(table: AnsTable, payload, out_len: int) -> bytes:
    out = np.empty(out_len, dtype=np.uint8)
    decompress_into(table, payload, out)
    return out.tobytes()


def decompress_blob(blob, out_len: int) -> bytes:
    table, payload = split_blob(blob)
    return ans_decompress(table, payload, out_len)


def decode_blobs_into(jobs: list[tuple[bytes, np.ndarray]], labels=None) -> None:
    """Decode many independent blobs into their preallocated outputs in one
    GPU pass.  Error order follows the reference (ans.py:375-430): the first
    prologue error in job order, else the first failing chunk in the
    reference's processing order (outputs grouped by length)."""
    if not jobs:
        return
    blobs = [bytes(b) for b, _ in jobs]
    outs = [o for _, o in jobs]
    res, jt = _decode_many(blobs, [o.size for o in outs])
    st = res.status
    for i, s in enumerate(st):
        if s in _PROLOGUE:
            label = labels[i] if labels is not None else i
            cls, msg = _PROLOGUE[s]
            if s == nv.CHUNK_EMPTY_BAD:
                raise CorruptStreamError(f"corrupt stream (chunk {label})")
            raise cls(f"{msg} (chunk {label})")
    bad = np.nonzero(st == nv.CHUNK_CORRUPT)[0]
    if len(bad):
        # reference processing order: groups keyed by output length in order of
        # first appearance, jobs in order within a group
        order: dict[int, list[int]] = {}
        for i, o in enumerate(outs):
            if o.size:
                order.setdefault(o.size, []).append(i)
        badset = set(int(b) for b in bad)
        first = next(i for g in order.values() for i in g if i in badset)
        label = labels[first] if labels is not None else first
        raise CorruptStreamError(f"corrupt stream (chunk {label})")
    host = res.out.cpu().numpy()
    for i, o in enumerate(outs):
        if o.size:
            off = int(jt.out_off[i])
            o.reshape(-1).view(np.uint8)[:] = host[off:off + o.size]


def warm_kernels() -> None:
    """Load the library and run every codec kernel once on a tiny input."""
    data = np.array([1, 2, 3, 1], dtype=np.uint8)
    blob = compress_blob(data)
    decompress_blob(blob, 4)
    outs = [np.empty(4, dtype=np.uint8) for _ in range(6)]
    decode_blobs_into([(blob, o) for o in outs])
