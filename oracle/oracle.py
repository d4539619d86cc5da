"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

A restatement of the CPU reference (arXiv 2502.15443 `dcomp`, see
/root/reference/pkg/src/dcomp) used to check the CUDA product path.  Only
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import it; the product package never does.

The byte/integer kernels live in ``dcomp_oracle.c`` (built by
``oracle/Makefile`` into ``oracle/liboracle.so``); this module restates the
Python glue around them (container layout, decode grouping, planner
arithmetic).  Each function cites the reference file:line it follows.
Parity of the restatement is pinned by tests/test_oracle_golden.py against
golden vectors that tests/golden/make_golden.py produced by running the
reference itself.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
import subprocess
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

PROB_SCALE = 4096
STATE_LOWER = 1 << 20
STATE_UPPER = 1 << 28
TABLE_BYTES = 384
HEADER_BYTES = 388
MAGIC = b"DCC1"
ENTRY = struct.Struct("<BQQQI")


class OracleError(Exception):
    """Oracle-side verdict.  ``kind`` names the reference exception class."""

    def __init__(self, kind: str, msg: str, chunk: int | None = None):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg
        self.chunk = chunk


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.or_normalize.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.or_pack_u12.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.or_unpack_table.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.or_unpack_table.restype = ctypes.c_int
        L.or_compress_blob.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        L.or_compress_blob.restype = ctypes.c_uint64
        L.or_decode.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_uint64]
        L.or_decode.restype = ctypes.c_int
        L.or_decode4.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_uint64]
        L.or_decode4.restype = ctypes.c_int
        L.or_crc32.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32]
        L.or_crc32.restype = ctypes.c_uint32
        L.or_quantize.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_void_p]
        L.or_quantize.restype = ctypes.c_int
        L.or_prune.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                               ctypes.c_double, ctypes.c_int, ctypes.c_void_p]
        L.or_prune.restype = ctypes.c_int
        L.or_gen_weights.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.or_gen_quantize.argtypes = [ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_void_p]
        L.or_gen_quantize.restype = ctypes.c_int
        del u8p
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _u8(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data.reshape(-1).view(np.uint8))
    return np.frombuffer(bytes(data), dtype=np.uint8)


# ---------------------------------------------------------------- codec
def normalize(hist) -> np.ndarray:
    """ans.py:213-243."""
    h = np.ascontiguousarray(hist, dtype=np.uint64)
    f = np.zeros(256, dtype=np.uint32)
    lib().or_normalize(_ptr(h), _ptr(f))
    return f


def pack_u12(freq) -> bytes:
    """ans.py:246-253."""
    f = np.ascontiguousarray(freq, dtype=np.uint32)
    out = np.zeros(TABLE_BYTES, dtype=np.uint8)
    lib().or_pack_u12(_ptr(f), _ptr(out))
    return out.tobytes()


def unpack_table(buf) -> np.ndarray:
    """ans.py:284-299.  Raises OracleError('CorruptStreamError')."""
    if len(buf) != TABLE_BYTES:
        raise OracleError("CorruptStreamError", "corrupt stream: bad table size")
    b = np.frombuffer(bytes(buf), dtype=np.uint8).copy()
    f = np.zeros(256, dtype=np.uint32)
    if lib().or_unpack_table(_ptr(b), _ptr(f)) != 0:
        raise OracleError("CorruptStreamError", "corrupt stream: invalid frequency table")
    return f


def table_for(data) -> np.ndarray:
    """ans.py:277-282 (AnsTable.for_data)."""
    u8 = _u8(data)
    if u8.size == 0:
        raise OracleError("DcompError", "empty input")
    return normalize(np.bincount(u8, minlength=256))


def compress_blob(data) -> bytes:
    """ans.py:316-330."""
    u8 = _u8(data)
    if u8.size == 0:
        raise OracleError("DcompError", "empty input")
    out = np.empty(HEADER_BYTES + 2 * u8.size + 8, dtype=np.uint8)
    scratch = np.empty(2 * u8.size + 8, dtype=np.uint8)
    n = lib().or_compress_blob(_ptr(u8), u8.size, _ptr(out), _ptr(scratch))
    return out[:n].tobytes()


def _split(blob):
    """ans.py:333-343 + 364-367.  Returns (freq, stream array, state)."""
    if len(blob) < HEADER_BYTES:
        raise OracleError("TruncatedError", "truncated stream: missing table header")
    freq = unpack_table(blob[:TABLE_BYTES])
    (state,) = struct.unpack_from("<I", blob, TABLE_BYTES)
    if not STATE_LOWER <= state < STATE_UPPER:
        raise OracleError("CorruptStreamError", "corrupt stream: final state out of range")
    stream = np.frombuffer(bytes(blob[HEADER_BYTES:]), dtype=np.uint8)
    return freq, stream, state


def decompress_blob(blob, out_len: int) -> bytes:
    """ans.py:346-372."""
    freq, stream, state = _split(blob)
    out = np.empty(out_len, dtype=np.uint8)
    if out_len == 0:
        if stream.size != 0 or state != STATE_LOWER:
            raise OracleError("CorruptStreamError", "corrupt stream")
        return b""
    st = np.ascontiguousarray(stream) if stream.size else np.zeros(1, np.uint8)
    if lib().or_decode(_ptr(st), stream.size, state, _ptr(freq), _ptr(out), out_len) != 0:
        raise OracleError("CorruptStreamError", "corrupt stream")
    return out.tobytes()


def decode_blobs_into(jobs, labels=None) -> None:
    """ans.py:375-430: prepare in job order, group by output length, quads,
    then a pair, then singles; a failing multi-lane pass is re-run singly."""
    prepared = []
    for idx, (blob, out) in enumerate(jobs):
        label = labels[idx] if labels is not None else idx
        try:
            freq, stream, state = _split(blob)
        except OracleError as e:
            raise OracleError(e.kind, f"{e.msg} (chunk {label})", label) from None
        if out.size == 0:
            if stream.size != 0 or state != STATE_LOWER:
                raise OracleError("CorruptStreamError", f"corrupt stream (chunk {label})", label)
            continue
        st = np.ascontiguousarray(stream) if stream.size else np.zeros(1, np.uint8)
        prepared.append((out.size, st, stream.size, state, freq, out, label))
    groups: dict[int, list] = {}
    for item in prepared:
        groups.setdefault(item[0], []).append(item)
    L = lib()

    def single(item):
        if L.or_decode(_ptr(item[1]), item[2], item[3], _ptr(item[4]), _ptr(item[5]), item[0]) != 0:
            raise OracleError("CorruptStreamError", f"corrupt stream (chunk {item[6]})", item[6])

    for group in groups.values():
        while len(group) >= 4:
            quad, group[:] = group[:4], group[4:]
            arr = lambda k, t: (t * 4)(*[it[k] for it in quad])  # noqa: E731
            streams = (ctypes.c_void_p * 4)(*[_ptr(it[1]) for it in quad])
            plens = (ctypes.c_uint64 * 4)(*[it[2] for it in quad])
            x0s = (ctypes.c_uint32 * 4)(*[it[3] for it in quad])
            freqs = (ctypes.c_void_p * 4)(*[_ptr(it[4]) for it in quad])
            outs = (ctypes.c_void_p * 4)(*[_ptr(it[5]) for it in quad])
            del arr
            bad = L.or_decode4(streams, plens, x0s, freqs, outs, quad[0][0])
            for bit, item in enumerate(quad):
                if bad & (1 << bit):
                    single(item)
        for item in group:
            single(item)


def crc32(data, crc: int = 0) -> int:
    u8 = _u8(data)
    return int(lib().or_crc32(_ptr(u8) if u8.size else 0, u8.size, crc))


# ---------------------------------------------------------------- transforms
def quantize(w: np.ndarray, s: np.ndarray | None = None) -> tuple[np.ndarray, float]:
    """scaling.py:78-105 (scale_weights + quantize).  Returns (q, w_scale)."""
    w = np.ascontiguousarray(w, dtype=np.float64)
    rows, cols = w.shape
    s = np.ones(cols) if s is None else np.ascontiguousarray(s, dtype=np.float64)
    q = np.empty((rows, cols), dtype=np.int8)
    ws = ctypes.c_double(0.0)
    rc = lib().or_quantize(_ptr(w), _ptr(s), rows, cols, _ptr(q), ctypes.addressof(ws))
    if rc == 1:
        raise OracleError("DcompError", "empty input")
    if rc == 2:
        raise OracleError("DcompError", "zero dynamic range")
    return q, ws.value


def gen_weights(key: int, n: int, start: int = 0) -> np.ndarray:
    """bench.py's hash weights (dcomp_oracle.c or_gen_weights), flat f64."""
    out = np.empty(n, dtype=np.float64)
    if n:
        lib().or_gen_weights(key & 0xFFFFFFFF, start, n, _ptr(out))
    return out


def gen_quantize(key: int, rows: int, cols: int, s: np.ndarray) -> tuple[np.ndarray, float]:
    """Hash weights -> scale_weights + quantize (scaling.py:78-105), fused so
    no f64 tensor is materialized.  Releases the GIL (ctypes)."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    q = np.empty((rows, cols), dtype=np.int8)
    ws = ctypes.c_double(0.0)
    rc = lib().or_gen_quantize(key & 0xFFFFFFFF, _ptr(s), rows, cols, _ptr(q), ctypes.addressof(ws))
    if rc:
        raise OracleError("DcompError", "empty input" if rc == 1 else "zero dynamic range")
    return q, ws.value


def compute_scale(cm: np.ndarray, alpha: float) -> np.ndarray:
    """scaling.py:68-75."""
    if alpha == 0.0:
        return np.ones(len(cm))
    return np.maximum(np.asarray(cm, dtype=np.float64), 1e-8) ** alpha


def prune(q: np.ndarray, cm: np.ndarray, sparsity: float, per_row: bool = False) -> np.ndarray:
    """pruning.py:37-64."""
    q = np.ascontiguousarray(q, dtype=np.int8)
    cm = np.ascontiguousarray(cm, dtype=np.float64)
    out = np.empty_like(q)
    lib().or_prune(_ptr(q), _ptr(cm), q.shape[0], q.shape[1], float(sparsity), int(per_row), _ptr(out))
    return out


# ---------------------------------------------------------------- container
def _header(entries, chunk_size: int) -> bytes:
    """container.py:102-117.  entries: (name, q, w_scale, alpha, s, cm)."""
    parts = [struct.pack("<II", chunk_size, len(entries))]
    for name, q, w_scale, alpha, s, cm in entries:
        nb = name.encode("utf-8")
        parts += [struct.pack("<H", len(nb)), nb, struct.pack("<IIdd", q.shape[0], q.shape[1], w_scale, alpha),
                  np.asarray(s).astype("<f4").tobytes(), np.asarray(cm).astype("<f4").tobytes()]
    body = b"".join(parts)
    return body + struct.pack("<I", zlib.crc32(body))


def pack(entries, chunk_size: int, mask=None, threads: int = 1) -> bytes:
    """container.py:135-177."""
    header = _header(entries, chunk_size)
    payload = (np.concatenate([np.ascontiguousarray(e[1]).reshape(-1).view(np.uint8) for e in entries])
               if entries else np.empty(0, np.uint8))
    n = math.ceil(payload.size / chunk_size)
    mask = np.ones(n, bool) if mask is None else np.asarray(mask, bool)
    raws = [payload[i * chunk_size:(i + 1) * chunk_size] for i in range(n)]
    todo = [i for i in range(n) if mask[i]]
    if threads > 1 and len(todo) > 1:
        with ThreadPoolExecutor(max_workers=min(threads, len(todo))) as pool:
            blobs = dict(zip(todo, pool.map(compress_blob, (raws[i] for i in todo))))
    else:
        blobs = {i: compress_blob(raws[i]) for i in todo}
    entries_b, payloads = [], []
    offset = 4 + 2 + 4 + len(header) + 4 + n * ENTRY.size
    for i, raw in enumerate(raws):
        blob = blobs.get(i)
        if blob is not None and len(blob) < raw.size:
            codec, data = 1, blob
        else:
            codec, data = 0, raw.tobytes()
        entries_b.append(ENTRY.pack(codec, offset, len(data), raw.size, zlib.crc32(raw)))
        payloads.append(data)
        offset += len(data)
    return b"".join([MAGIC, struct.pack("<HI", 1, len(header)), header, struct.pack("<I", n)]
                    + entries_b + payloads)


def parse(data: bytes):
    """container.py:201-274 (happy path + the structural checks).
    Returns (chunk_size, directory, entries)."""
    if data[:4] != MAGIC:
        raise OracleError("BadMagicError", "not a DCC1 container")
    version, hlen = struct.unpack_from("<HI", data, 4)
    if version != 1:
        raise OracleError("UnsupportedVersionError", f"unsupported container version {version}")
    header = data[10:10 + hlen]
    if len(header) < hlen:
        raise OracleError("TruncatedError", "truncated file")
    body = header[:-4]
    if zlib.crc32(body) != struct.unpack("<I", header[-4:])[0]:
        raise OracleError("ChecksumError", "header checksum mismatch", -1)
    chunk_size, count = struct.unpack_from("<II", body, 0)
    pos = 8
    directory = []
    for _ in range(count):
        (nl,) = struct.unpack_from("<H", body, pos)
        pos += 2
        name = body[pos:pos + nl].decode("utf-8")
        pos += nl
        rows, cols, w_scale, alpha = struct.unpack_from("<IIdd", body, pos)
        pos += 24
        s = np.frombuffer(body, "<f4", cols, pos).astype(np.float64)
        pos += 4 * cols
        cm = np.frombuffer(body, "<f4", cols, pos).astype(np.float64)
        pos += 4 * cols
        directory.append((name, rows, cols, w_scale, alpha, s, cm))
    pos = 10 + hlen
    (n,) = struct.unpack_from("<I", data, pos)
    pos += 4
    entries = [ENTRY.unpack_from(data, pos + i * ENTRY.size) for i in range(n)]
    return chunk_size, directory, entries


def unpack(data: bytes, threads: int = 1):
    """container.py:296-346.  Returns list of (name, q, w_scale, alpha, s, cm)."""
    chunk_size, directory, entries = parse(data)
    total = sum(e[3] for e in entries)
    out = np.empty(total, dtype=np.uint8)
    jobs, labels = [], []
    pos = 0
    for i, (codec, off, clen, ulen, _crc) in enumerate(entries):
        dest = out[pos:pos + ulen]
        if codec == 0:
            dest[:] = np.frombuffer(data, np.uint8, clen, off)
        else:
            jobs.append((data[off:off + clen], dest))
            labels.append(i)
        pos += ulen
    if jobs:
        workers = min(threads, math.ceil(len(jobs) / 4))
        if workers > 1:
            per = math.ceil(len(jobs) / workers / 4) * 4
            slices = [(jobs[i:i + per], labels[i:i + per]) for i in range(0, len(jobs), per)]
            with ThreadPoolExecutor(max_workers=workers) as pool:
                list(pool.map(lambda s: decode_blobs_into(s[0], s[1]), slices))
        else:
            decode_blobs_into(jobs, labels)
    pos = 0
    for i, e in enumerate(entries):
        if zlib.crc32(out[pos:pos + e[3]]) != e[4]:
            raise OracleError("ChecksumError", f"checksum mismatch in chunk {i}", i)
        pos += e[3]
    res = []
    pos = 0
    for name, rows, cols, w_scale, alpha, s, cm in directory:
        q = out[pos:pos + rows * cols].view(np.int8).reshape(rows, cols).copy()
        pos += rows * cols
        res.append((name, q, w_scale, alpha, s, cm))
    return res


# ---------------------------------------------------------------- planner
def block_mask(n_chunks: int, block_size: int) -> np.ndarray:
    """latency.py:104-113."""
    mask = np.zeros(n_chunks, bool)
    if block_size > 0:
        mask[block_size - 1::block_size] = True
        mask[(n_chunks // block_size) * block_size:] = False
    return mask


def latency_seconds(B_load: float, D_max: float, c_sat: float, I_gpu: float, chunk_size: int,
                    mask: np.ndarray, cr) -> float:
    """latency.py:183-200 (rates in GB/s, GB = 1e9)."""
    cr = np.broadcast_to(np.asarray(cr, np.float64), mask.shape)
    S = float(chunk_size)
    D = D_max * min(1.0, chunk_size / c_sat) * 1e9
    load = np.where(mask, S / cr, S) / (B_load * 1e9)
    dec = np.where(mask, S / D, 0.0)
    comp = np.full(mask.size, S / (I_gpu * 1e9))
    return float(np.sum(np.maximum(np.maximum(load, dec), comp)))
