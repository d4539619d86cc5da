"""DCC1 container -- the reference's container.py API over B200 kernels.

Byte layout (normative, reference container.py:1-18, little-endian):

    "DCC1" | u16 version | u32 header_len | header (body | u32 crc32(body))
    | u32 chunk_count | chunk_count x <B Q Q Q I> | chunk payloads

    body  = u32 chunk_size, u32 tensor_count, then per tensor
            u16 name_len | name | u32 rows | u32 cols | f64 w_scale | f64 alpha
            | f32[cols] scale vector | f32[cols] channel maxima
    entry = codec (0 store / 1 ans) | file_offset | comp_len | uncomp_len
            | crc32 of the uncompressed chunk

Tensors are concatenated row-major and cut every ``chunk_size`` bytes.

What runs where:
  * GPU: per-chunk histograms, normalization, rANS encode, payload assembly,
    rANS decode (split-point parallel when an index is available, else the
    exact per-chunk walk), CRC32 of every chunk.
  * host: the header / chunk-table bytes (format code, O(tensors + chunks)).

``pack``/``unpack`` return exactly what the reference returns (bytes /
ModelBundle); ``pack_indexed``, ``unpack(..., index=)``, the ``.dcidx``
sidecar and ``pack_device`` (a payload already on the GPU) are B200
extensions.

Memory note: ``unpack`` decodes into ONE pinned host buffer and the returned
tensors' ``qvalues`` are views into it (the D2H runs at PCIe speed straight
into them); the buffer lives as long as any of those arrays.  Pass
``copy=True`` for the reference's independent per-tensor (pageable) copies.
"""

from __future__ import annotations

import dataclasses
import math
import os
import struct
import zlib

import numpy as np
import torch

from . import engine
from . import native as nv
from .errors import (
    BadMagicError,
    ChecksumError,
    CorruptStreamError,
    DataFormatError,
    DcompError,
    TruncatedError,
    UnsupportedVersionError,
)
from .scaling import QuantizedTensor, ScaleVector
from .tensors import ActivationStats

MAGIC = b"DCC1"
VERSION = 1
MIN_CHUNK_SIZE = 4096
DEFAULT_CHUNK_SIZE = 16 * 2**20
CODEC_STORE = 0
CODEC_ANS = 1

_ENTRY = struct.Struct("<BQQQI")
ENTRY_DTYPE = np.dtype([("codec", "u1"), ("file_offset", "<u8"), ("comp_len", "<u8"),
                        ("uncomp_len", "<u8"), ("crc32", "<u4")])
assert ENTRY_DTYPE.itemsize == _ENTRY.size == 29
SIDECAR_SUFFIX = ".dcidx"


def thread_count() -> int:
    """DCOMP_THREADS semantics of the reference (container.py:58-65); the
    GPU path does not use host threads, the CPU baseline does."""
    env = os.environ.get("DCOMP_THREADS")
    if env is not None:
        try:
            return max(1, int(env))
        except ValueError:
            raise DcompError(f"DCOMP_THREADS must be an integer, got {env!r}") from None
    return os.cpu_count() or 1


@dataclasses.dataclass(frozen=True)
class ModelBundle:
    tensors: list[QuantizedTensor]
    stats: dict[str, ActivationStats]
    chunk_size: int = DEFAULT_CHUNK_SIZE


@dataclasses.dataclass(frozen=True)
class ChunkEntry:
    codec: int
    file_offset: int
    comp_len: int
    uncomp_len: int
    crc32: int


@dataclasses.dataclass(frozen=True)
class ContainerInfo:
    chunk_size: int
    directory: list[tuple[str, int, int, float, float]]  # name, rows, cols, w_scale, alpha
    chunks: list[ChunkEntry]
    file_size: int

    @property
    def total_uncompressed(self) -> int:
        return sum(c.uncomp_len for c in self.chunks)


# ------------------------------------------------------------------ writer
def _stats_map(stats) -> dict[str, ActivationStats]:
    return stats if isinstance(stats, dict) else {s.name: s for s in stats}


def _header(tensors, stats: dict, chunk_size: int) -> bytes:
    parts = [struct.pack("<II", chunk_size, len(tensors))]
    for t in tensors:
        st = stats.get(t.name)
        if st is None:
            raise DcompError(f"missing activation stats for tensor {t.name!r}")
        if len(st.channel_max) != t.cols:
            raise DcompError(f"stats length {len(st.channel_max)} != cols {t.cols} for tensor {t.name!r}")
        raw_name = t.name.encode("utf-8")
        parts += [struct.pack("<H", len(raw_name)), raw_name,
                  struct.pack("<IIdd", t.rows, t.cols, t.w_scale, t.scale_vec.alpha),
                  t.scale_vec.s.astype("<f4").tobytes(), st.channel_max.astype("<f4").tobytes()]
    body = b"".join(parts)
    return body + struct.pack("<I", zlib.crc32(body))


def _mask_of(plan, n_chunks: int) -> np.ndarray:
    if plan is None:
        return np.ones(n_chunks, dtype=bool)
    mask = np.asarray(getattr(plan, "compressed_mask", plan), dtype=bool)
    if mask.shape != (n_chunks,):
        raise DcompError(f"plan covers {mask.size} chunks, container has {n_chunks}")
    return mask


def _device_payload(tensors) -> torch.Tensor:
    """Concatenated int8 payload on the GPU: the tensors are gathered into one
    pinned staging buffer by parallel host copies, then one async H2D."""
    dev = nv.require_cuda()
    total = sum(t.qvalues.size for t in tensors)
    out = nv.device_bytes(total, dev)
    if total == 0:
        return out
    stage = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    sv = stage.numpy()
    from concurrent.futures import ThreadPoolExecutor
    jobs, pos = [], 0
    for t in tensors:
        n = t.qvalues.size
        if n:
            jobs.append((sv[pos:pos + n], np.ascontiguousarray(t.qvalues).reshape(-1).view(np.uint8)))
        pos += n
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(lambda j: np.copyto(j[0], j[1]), jobs))
    out[:total].copy_(stage, non_blocking=True)
    return out


def pack_device(payload: torch.Tensor, header: bytes, chunk_size: int, plan=None,
                seg_shift: int | None = engine.DEFAULT_SEG_SHIFT):
    """Encode a device-resident payload into a DCC1 image.

    Returns (device file image uint8, EncodeResult, entries ndarray).  The
    image holds the whole file; its payload region is assembled on the GPU.
    """
    total = int(payload.numel())
    n = math.ceil(total / chunk_size) if total else 0
    mask = _mask_of(plan, n)
    enc = engine.encode_payload(payload, chunk_size, mask, seg_shift)
    first = len(MAGIC) + 2 + 4 + len(header) + 4 + n * _ENTRY.size
    offs = np.zeros(n, dtype=np.uint64)
    if n:
        offs[1:] = np.cumsum(enc.comp_len)[:-1]
    file_off = offs + np.uint64(first)
    entries = np.zeros(n, dtype=ENTRY_DTYPE)
    entries["codec"] = enc.codec
    entries["file_offset"] = file_off
    entries["comp_len"] = enc.comp_len
    entries["uncomp_len"] = np.minimum(chunk_size, total - np.arange(n, dtype=np.uint64) * np.uint64(chunk_size))
    entries["crc32"] = enc.crc
    size = first + int(enc.comp_len.sum())
    image = nv.device_bytes(size, payload.device)
    prefix = MAGIC + struct.pack("<HI", VERSION, len(header)) + header + struct.pack("<I", n) + entries.tobytes()
    image[:first].copy_(torch.frombuffer(bytearray(prefix), dtype=torch.uint8))
    engine.assemble(payload, enc, file_off, image)
    return image, enc, entries


def _pack_impl(tensors, stats, chunk_size, plan, seg_shift):
    if chunk_size < MIN_CHUNK_SIZE:
        raise DcompError(f"chunk_size must be >= {MIN_CHUNK_SIZE}, got {chunk_size}")
    names = [t.name for t in tensors]
    if len(set(names)) != len(names):
        raise DcompError("duplicate tensor names")
    header = _header(tensors, _stats_map(stats), chunk_size)
    total = sum(t.qvalues.size for t in tensors)
    _mask_of(plan, math.ceil(total / chunk_size))  # reference checks the plan before encoding
    if total == 0:
        data = MAGIC + struct.pack("<HI", VERSION, len(header)) + header + struct.pack("<I", 0)
        return data, None
    payload = _device_payload(tensors)
    image, enc, _ = pack_device(payload, header, chunk_size, plan, seg_shift)
    return nv.to_bytes(image), enc.index  # pinned D2H, then the one (parallel) copy `bytes` needs


def pack(tensors, stats, chunk_size: int = DEFAULT_CHUNK_SIZE, plan=None) -> bytes:
    """Serialize quantized tensors into DCC1 bytes (bit-identical to the
    reference's pack).  ``plan`` selects per-chunk codecs (None = all ANS);
    chunks whose blob would not shrink are stored raw."""
    return _pack_impl(tensors, stats, chunk_size, plan, None)[0]


def pack_indexed(tensors, stats, chunk_size: int = DEFAULT_CHUNK_SIZE, plan=None,
                 seg_shift: int = engine.DEFAULT_SEG_SHIFT):
    """``pack`` plus the split-point index the GPU encoder records for free."""
    return _pack_impl(tensors, stats, chunk_size, plan, seg_shift)


def write_container(path, tensors, stats, chunk_size: int = DEFAULT_CHUNK_SIZE, plan=None,
                    sidecar: bool = False) -> None:
    data, index = _pack_impl(tensors, stats, chunk_size, plan, engine.DEFAULT_SEG_SHIFT if sidecar else None)
    with open(path, "wb") as f:
        f.write(data)
    if sidecar and index is not None:
        with open(str(path) + SIDECAR_SUFFIX, "wb") as f:
            f.write(index.to_bytes(binding_of(data)))


# ------------------------------------------------------------------ reader
class _Cursor:
    def __init__(self, buf: bytes, pos: int = 0):
        self.buf = buf
        self.pos = pos

    def take(self, n: int) -> bytes:
        if self.pos + n > len(self.buf):
            raise TruncatedError(f"truncated file at offset {self.pos}")
        out = self.buf[self.pos:self.pos + n]
        self.pos += n
        return out

    def fmt(self, f: str):
        return struct.unpack(f, self.take(struct.calcsize(f)))


def _check_stats(names, sv, cv, lens, upto: int) -> None:
    """Reference order (container.py:216-229): for tensor i < upto, first a
    bad scale vector, then bad channel maxima; raise the earliest."""
    if upto == 0:
        return
    n = int(lens[:upto].sum())
    s_bad = (sv[:n] <= 0) | ~np.isfinite(sv[:n])
    c_bad = (cv[:n] < 0) | ~np.isfinite(cv[:n])
    if not (s_bad.any() or c_bad.any()):
        return
    ends = np.cumsum(lens[:upto])
    first = lambda m: int(np.searchsorted(ends, int(np.argmax(m)), side="right")) if m.any() else upto  # noqa: E731
    i_s, i_c = first(s_bad), first(c_bad)
    if i_s <= i_c:
        raise DataFormatError(f"{names[i_s]}: scale vector not positive finite")
    raise DataFormatError(f"{names[i_c]}: channel maxima not finite non-negative")


def _parse_header(header: bytes):
    """Reference container.py:201-235.  One walk over the entries (no copies:
    memoryview slices), then the per-channel checks of every s / cm vector in
    one vectorized pass; errors keep the reference's order.  s / cm come back
    as f32 views (the file's values); ScaleVector / ActivationStats widen them
    to f64 exactly when the bundle is built (overlapped with the GPU in
    unpack)."""
    if len(header) < 4:
        raise DataFormatError("header too small to hold its checksum")
    mv = memoryview(header)
    body = mv[:-4]
    if zlib.crc32(body) != struct.unpack_from("<I", mv, len(mv) - 4)[0]:
        raise ChecksumError(-1, "header checksum mismatch")
    cur = _Cursor(body)
    chunk_size, count = cur.fmt("<II")
    if chunk_size < 1:
        raise DataFormatError("invalid chunk size 0")
    meta, s_parts, c_parts = [], [], []

    def stats():
        names = [m[0] for m in meta]
        lens = np.array([m[2] for m in meta], dtype=np.int64)
        sv = np.concatenate(s_parts) if s_parts else np.empty(0, np.float32)
        cv = np.concatenate(c_parts) if c_parts else np.empty(0, np.float32)
        return names, sv, cv, lens

    try:
        for _ in range(count):
            (nl,) = cur.fmt("<H")
            try:
                name = bytes(cur.take(nl)).decode("utf-8")
            except UnicodeDecodeError as e:
                raise DataFormatError(f"tensor name is not valid UTF-8: {e}") from None
            rows, cols, w_scale, alpha = cur.fmt("<IIdd")
            if rows < 1 or cols < 1:
                raise DataFormatError(f"{name}: invalid dims {rows}x{cols}")
            if not (np.isfinite(w_scale) and w_scale > 0):
                raise DataFormatError(f"{name}: invalid w_scale {w_scale}")
            s_parts.append(np.frombuffer(cur.take(4 * cols), dtype="<f4"))
            c_parts.append(np.frombuffer(cur.take(4 * cols), dtype="<f4"))
            meta.append((name, rows, cols, w_scale, alpha))
    except (DataFormatError, TruncatedError):
        # an earlier tensor's stats error comes first in the reference's walk
        names, sv, cv, lens = stats()
        _check_stats(names, sv, cv, lens, len(meta))
        raise
    names, sv, cv, lens = stats()
    _check_stats(names, sv, cv, lens, len(meta))
    if cur.pos != len(body):
        raise DataFormatError(f"{len(body) - cur.pos} stray bytes in header")
    if len(set(names)) != len(names):
        raise DataFormatError("duplicate tensor names in header")
    directory, pos = [], 0
    for name, rows, cols, w_scale, alpha in meta:
        directory.append((name, rows, cols, w_scale, alpha, sv[pos:pos + cols], cv[pos:pos + cols]))
        pos += cols
    return chunk_size, directory


def _parse(data: bytes, total: int | None = None):
    """Structure + chunk table validation (reference container.py:238-274),
    vectorized over chunks with the reference's first-error order.  ``data``
    may be just the file's prefix through the chunk table when ``total`` (the
    file length) is given."""
    total = len(data) if total is None else total
    cur = _Cursor(data)
    if cur.take(4) != MAGIC:
        raise BadMagicError("not a DCC1 container")
    (version,) = cur.fmt("<H")
    if version != VERSION:
        raise UnsupportedVersionError(f"unsupported container version {version}")
    (hlen,) = cur.fmt("<I")
    chunk_size, directory = _parse_header(cur.take(hlen))
    ent, start = _parse_table(data, cur, chunk_size, total)
    _check_total(ent, directory)
    return chunk_size, directory, ent, start


def _check_total(ent, directory) -> None:
    total = int(ent["uncomp_len"].sum(dtype=np.uint64)) if len(ent) else 0
    want = sum(r * c for _, r, c, *_ in directory)
    if total != want:
        raise DataFormatError(f"chunks carry {total} bytes, directory declares {want}")


def _parse_table_first(data: bytes, total: int):
    """Chunk table of a container whose header body is parsed later (unpack
    overlaps the header walk with the GPU pipeline): the same table checks as
    _parse with chunk_size read from the raw header.  Any error here, or later
    in the header, is re-raised by a full _parse so the reference's first-error
    order holds.  Returns (chunk_size, ent, start, header bytes)."""
    try:
        if len(data) < 14 or data[:4] != MAGIC or struct.unpack_from("<H", data, 4)[0] != VERSION:
            raise DataFormatError("prefix")
        (hlen,) = struct.unpack_from("<I", data, 6)
        if hlen < 12 or 10 + hlen > len(data):
            raise DataFormatError("header")
        (chunk_size,) = struct.unpack_from("<I", data, 10)
        if chunk_size < 1:
            raise DataFormatError("chunk size")
        ent, start = _parse_table(data, _Cursor(data, 10 + hlen), chunk_size, total)
        return chunk_size, ent, start, data[10:10 + hlen]
    except DataFormatError:
        _parse(data, total)  # raises the reference's first error
        raise


def _parse_table(data: bytes, cur: "_Cursor", chunk_size: int, total: int):
    (count,) = cur.fmt("<I")
    avail = (total - cur.pos) // _ENTRY.size
    if avail < count:
        raise TruncatedError(f"truncated file at offset {cur.pos + avail * _ENTRY.size}")
    ent = np.frombuffer(data, dtype=ENTRY_DTYPE, count=count, offset=cur.pos)
    cur.pos += count * _ENTRY.size
    start = cur.pos
    if count:
        codec = ent["codec"]
        off = ent["file_offset"]
        clen = ent["comp_len"]
        ulen = ent["uncomp_len"]
        huge = bool((clen > np.uint64(1 << 50)).any())
        if huge:  # exact big-int accumulation, as the reference does
            exp = [start]
            for c in clen[:-1]:
                exp.append(exp[-1] + int(c))
            expected = np.array(exp, dtype=object)
            off_cmp = np.array([int(o) for o in off], dtype=object) != expected
        else:
            expected = np.empty(count, dtype=np.uint64)
            expected[0] = start
            expected[1:] = np.uint64(start) + np.cumsum(clen[:-1], dtype=np.uint64)
            off_cmp = off != expected
        last = np.zeros(count, bool)
        last[-1] = True
        conds = [
            ((codec != CODEC_STORE) & (codec != CODEC_ANS), lambda i: f"chunk {i}: unknown codec {ent['codec'][i]}"),
            (off_cmp, lambda i: f"chunk {i}: offset {int(off[i])}, expected {int(expected[i])}"),
            ((codec == CODEC_STORE) & (clen != ulen), lambda i: f"chunk {i}: store codec with comp_len != uncomp_len"),
            (ulen == 0, lambda i: f"chunk {i}: empty chunk"),
            ((~last & (ulen != np.uint64(chunk_size))) | (ulen > np.uint64(chunk_size)),
             lambda i: f"chunk {i}: uncompressed length {int(ulen[i])} breaks chunking"),
        ]
        first_bad = [int(np.argmax(c)) if c.any() else count for c, _ in conds]
        i = min(first_bad)
        if i < count:
            k = first_bad.index(i)
            raise DataFormatError(conds[k][1](i))
        end = int(expected[-1]) + int(clen[-1])
    else:
        end = start
    if end > total:
        raise TruncatedError(f"chunk payloads extend past end of file ({end} > {total})")
    if end < total:
        raise DataFormatError(f"{total - end} trailing bytes after last chunk")
    return ent, start


def binding_of(data: bytes) -> int:
    """Ties a sidecar index to its container: CRC32 of the file prefix fields,
    the header's own stored CRC32 (which fingerprints the whole header) and
    the chunk table (offsets, lengths and per-chunk CRC32s) -- a few KB."""
    (hlen,) = struct.unpack_from("<I", data, 6)
    (count,) = struct.unpack_from("<I", data, 10 + hlen)
    mv = memoryview(data)
    return zlib.crc32(mv[6 + hlen: 14 + hlen + count * _ENTRY.size], zlib.crc32(mv[:10]))


def _file_bytes(data) -> bytes:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return bytes(data)
    with open(data, "rb") as f:
        return f.read()


def inspect(data) -> ContainerInfo:
    """Validate the structure (no payload decode) and describe the container."""
    data = _file_bytes(data)
    chunk_size, directory, ent, _ = _parse(data)
    chunks = [ChunkEntry(int(e["codec"]), int(e["file_offset"]), int(e["comp_len"]), int(e["uncomp_len"]),
                         int(e["crc32"])) for e in ent]
    return ContainerInfo(chunk_size, [(n, r, c, ws, a) for n, r, c, ws, a, _, _ in directory], chunks, len(data))


def jobs_for(ent: np.ndarray, device=None) -> engine.JobTable:
    n = len(ent)
    ulen = ent["uncomp_len"].astype(np.uint64)
    ooff = np.zeros(n, dtype=np.uint64)
    if n:
        ooff[1:] = np.cumsum(ulen)[:-1]
    return engine.JobTable.build(ent["file_offset"], ent["comp_len"], ooff, ulen, ent["codec"], device)


def raise_decode_errors(status: np.ndarray) -> None:
    """First prologue error (chunk order), then the first corrupt chunk --
    the order the reference's decode_blobs_into reports them in."""
    pro = np.nonzero((status >= nv.CHUNK_TRUNC_TABLE) & (status <= nv.CHUNK_EMPTY_BAD))[0]
    if len(pro):
        i = int(pro[0])
        s = int(status[i])
        if s == nv.CHUNK_TRUNC_TABLE:
            raise TruncatedError(f"truncated stream: missing table header (chunk {i})")
        if s == nv.CHUNK_BAD_TABLE:
            raise CorruptStreamError(f"corrupt stream: invalid frequency table (chunk {i})")
        if s == nv.CHUNK_STATE_RANGE:
            raise CorruptStreamError(f"corrupt stream: final state out of range (chunk {i})")
        raise CorruptStreamError(f"corrupt stream (chunk {i})")
    bad = np.nonzero(status != nv.CHUNK_OK)[0]
    if len(bad):
        raise CorruptStreamError(f"corrupt stream (chunk {int(bad[0])})")


def decode_and_verify(base: torch.Tensor, ent: np.ndarray, index=None, build_index: bool = False,
                      tasks=None) -> engine.DecodeResult:
    """GPU decode of every chunk + reference error semantics + CRC check."""
    jobs = jobs_for(ent, base.device)
    res = engine.decode_jobs(base, jobs, index=index, build_index=build_index, tasks=tasks)
    raise_decode_errors(res.status)
    if jobs.n:
        crc = engine.crc32_ranges(res.out, jobs.d_out_off, jobs.d_out_len, int(jobs.out_len.max()))
        got = crc.cpu().numpy().view(np.uint32)
        bad = np.nonzero(got != ent["crc32"])[0]
        if len(bad):
            raise ChecksumError(int(bad[0]))
    return res


def _bundle(directory, host: np.ndarray, chunk_size: int) -> ModelBundle:
    tensors, stats = [], {}
    pos = 0
    for name, rows, cols, w_scale, alpha, s, cm in directory:
        n = rows * cols
        q = host[pos:pos + n].view(np.int8).reshape(rows, cols)
        pos += n
        tensors.append(QuantizedTensor(name, q, w_scale, ScaleVector(alpha, s)))
        stats[name] = ActivationStats(name, cm)
    return ModelBundle(tensors=tensors, stats=stats, chunk_size=chunk_size)


def _prefix(view: np.ndarray) -> memoryview:
    """The file's bytes through the end of the chunk table (header + table),
    for parsing a container that lives in a pinned tensor: a zero-copy view
    (the header of a large model is ~10 MB; copying it delayed the first H2D)."""
    mv = memoryview(view).cast("B")
    if view.size < 14:
        return mv
    (hlen,) = struct.unpack_from("<I", view, 6)
    if 14 + hlen > view.size:
        return mv
    (count,) = struct.unpack_from("<I", view, 10 + hlen)
    return mv[: min(view.size, 14 + hlen + count * _ENTRY.size)]


def _copied(b: ModelBundle) -> ModelBundle:
    ts = [QuantizedTensor(t.name, np.array(t.qvalues, copy=True), t.w_scale, t.scale_vec) for t in b.tensors]
    return ModelBundle(tensors=ts, stats=b.stats, chunk_size=b.chunk_size)


def unpack(data, index=None, copy: bool = False) -> ModelBundle:
    """Decode and verify a container (inverse of pack).  ``index`` (a
    SegmentIndex or sidecar bytes) enables the split-point parallel decoder;
    without it each ANS chunk is decoded by one exact sequential walk.
    ``data`` (and a sidecar ``index``) may also be pinned CPU uint8 tensors:
    the container is then copied to the GPU straight from that memory.
    ``copy=True``: per-tensor pageable copies instead of views of the pinned
    output buffer (see the module docstring)."""
    import time
    clock = [time.perf_counter()]

    def lap(name):  # host-side phase times; DCOMP_PHASE_SYNC=1 serializes them against the GPU
        if _PHASE_SYNC:
            torch.cuda.synchronize()
        now = time.perf_counter()
        LAST_UNPACK_MS[name] = (now - clock[0]) * 1e3
        clock[0] = now

    src = None
    if isinstance(data, torch.Tensor):
        if data.dtype != torch.uint8 or data.is_cuda or data.dim() != 1:
            raise DcompError("container tensor must be a 1-D uint8 CPU tensor")
        src = data if data.is_pinned() else None
        view = data.numpy()
        head, total = _prefix(view), view.size
        data = view
    else:
        data = _file_bytes(data)
        head, total = data, len(data)
    LAST_UNPACK_MS.clear()
    binding = None
    if index is None and _INDEX_CACHE_SIZE > 0:  # split points recorded by an earlier index-less unpack
        try:
            binding = binding_of(head)
            index = _INDEX_CACHE.get((torch.cuda.current_device(), binding))
        except struct.error:
            binding = None
    if index is not None:  # split-point path: H2D / decode / D2H pipelined per chunk group
        # chunk table first: the GPU pipeline starts before the header body
        # (names, stats, header CRC) is walked on the host
        chunk_size, ent, _, hdr = _parse_table_first(head, total)
        lap("table")
        jobs = jobs_for(ent)
        if len(ent) and isinstance(index, (bytes, bytearray, memoryview, torch.Tensor)):
            index = engine.SegmentIndex.from_bytes(index, jobs, binding_of(head), lazy=True)
        lap("index")
        if len(ent) and index is not None:
            pd = engine.PipelinedDecode(src if src is not None else np.frombuffer(data, np.uint8), jobs, index)
            lap("launch")
            try:
                _, directory = _parse_header(hdr)
                _check_total(ent, directory)
            except DataFormatError:
                pd.finish()
                _parse(head, total)  # the reference's first error
                raise
            lap("header")
            out = _bundle(directory, pd.host_out.numpy(), chunk_size)  # views; filled by the pipeline
            lap("bundle")
            _, status, crc = pd.finish()
            lap("pipeline")
            if pd.marks is not None:
                LAST_UNPACK_TIMELINE[:] = [("host:" + k, v, float("nan")) for k, v in LAST_UNPACK_MS.items()]
                LAST_UNPACK_TIMELINE.extend(pd.timeline())
            raise_decode_errors(status)
            bad = np.nonzero(crc != ent["crc32"])[0]
            if len(bad):
                raise ChecksumError(int(bad[0]))
            return _copied(out) if copy else out
    chunk_size, directory, ent, _ = _parse(head, total)
    if len(ent) == 0:
        return _bundle(directory, np.empty(0, np.uint8), chunk_size)
    lap("parse")
    base = nv.to_device_bytes(data)
    lap("h2d")
    record = binding is not None and index is None
    res = decode_and_verify(base, ent, index=index, build_index=record)
    lap("decode_crc")
    if record and res.index is not None and res.index.n_segs:  # verified: keep for the next unpack
        _INDEX_CACHE[(torch.cuda.current_device(), binding)] = res.index
        while len(_INDEX_CACHE) > _INDEX_CACHE_SIZE:
            _INDEX_CACHE.pop(next(iter(_INDEX_CACHE)))
    host = nv.to_host(res.out)
    lap("d2h")
    out = _bundle(directory, host, chunk_size)
    lap("bundle")
    return _copied(out) if copy else out


# Split-point indexes recorded by index-less unpacks (the serial pass records
# them for free), keyed by the container's binding: a later unpack of the same
# container takes the parallel path.  Device memory: 8 B per 256 B of weights
# per entry, keyed by (device, binding) so an index is only used on the device
# that holds it; DCOMP_INDEX_CACHE=0 disables, clear_index_cache() frees.
_INDEX_CACHE: dict = {}
_INDEX_CACHE_SIZE = int(os.environ.get("DCOMP_INDEX_CACHE", "2"))


def clear_index_cache() -> None:
    _INDEX_CACHE.clear()


LAST_UNPACK_MS: dict[str, float] = {}  # phase timings of the last unpack() (diagnostics)
LAST_UNPACK_TIMELINE: list = []  # DCOMP_TIMELINE=1: per-stage (name, host ms, device ms)
_PHASE_SYNC = os.environ.get("DCOMP_PHASE_SYNC") == "1"


def read_container(path) -> ModelBundle:
    side = str(path) + SIDECAR_SUFFIX
    index = None
    if os.path.exists(side):
        with open(side, "rb") as f:
            index = f.read()
    return unpack(path, index=index)


# --------------------------------------------------------- benchmark helpers
def chunked_compress(data, chunk_size: int = DEFAULT_CHUNK_SIZE) -> list[bytes]:
    """Split raw bytes into chunk-sized ANS blobs (every chunk encoded, no store
    fallback; reference container.py:349-354), all chunks encoded concurrently."""
    from .ans import compress_blobs
    u8 = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data.reshape(-1).view(np.uint8)
    return compress_blobs([u8[i:i + chunk_size] for i in range(0, u8.size, chunk_size)])


def chunked_decompress(blobs: list[bytes], lengths: list[int]) -> np.ndarray:
    from .ans import decode_blobs_into
    out = np.empty(int(sum(lengths)), dtype=np.uint8)
    jobs, pos = [], 0
    for blob, n in zip(blobs, lengths):
        jobs.append((blob, out[pos:pos + n]))
        pos += n
    decode_blobs_into(jobs)
    return out
