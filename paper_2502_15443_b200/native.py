"""ctypes binding of the C-ABI library (include/dcomp_b200.h).

The library is built in-tree (``python -m paper_2502_15443_b200._build``) as
``libdcomp_b200.so``.  There is no CPU fallback: if the library or a CUDA
device is missing, every GPU entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DCOMP_LIB") or os.path.join(HERE, "libdcomp_b200.so")  # DCOMP_LIB: A/B builds

READ_SLACK = 16384  # DC_READ_SLACK

# per-chunk status codes (DC_CHUNK_*)
CHUNK_OK = 0
CHUNK_TRUNC_TABLE = 1
CHUNK_BAD_TABLE = 2
CHUNK_STATE_RANGE = 3
CHUNK_EMPTY_BAD = 4
CHUNK_CORRUPT = 5
CHUNK_CHAIN = 6


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is not available (no CPU fallback exists)."""


class NativeError(RuntimeError):
    """A C-ABI call returned an argument or CUDA error."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I32 = ctypes.c_int32

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "dc_version": [],
    "dc_last_error": [],
    "dc_device_sm_count": [ctypes.c_int],
    "dc_ans_validate": [_P, _P, _P, _P, _P, _I64, _P, _P],
    "dc_ans_decode_serial": [_P, _P, _P, _P, _P, _P, _I64, _P, _U32, _P, _P, _P, _P, _P],
    "dc_decode_task_segments": [],
    "dc_ans_decode_segments": [_P, _P, _P, _P, _P, _U32, _P, _P, _P, _P, _I64, _P, _P, _P],
    "dc_ans_decode_segments_narrow": [_P, _P, _P, _P, _P, _U32, _P, _P, _P, _P, _I64, _P, _P, _P],
    "dc_decode_narrow_segments": [],
    "dc_decode_stage_cap": [ctypes.c_int],
    "dc_decode_small_segments": [],
    "dc_decode_small_max_chunk": [],
    "dc_ans_decode_small": [_P, _P, _P, _P, _P, _U32, _P, _P, _P, _P, _I64, _P, _P, _P],
    "dc_store_copy": [_P, _P, _P, _P, _P, _I64, _P, _P],
    "dc_crc32_ranges": [_P, _U64, _P, _P, _I64, _U64, _P, _P],
    "dc_channel_absmax": [_P, ctypes.c_int, _I64, _I64, _P, _P],
    "dc_act_quant_bytes": [],
    "dc_act_quant": [_P, ctypes.c_int, ctypes.c_int, _I64, _I64, _P, _P],
    "dc_hist_chunks": [_P, _U64, _U64, _I64, _P, _P],
    "dc_normalize_tables": [_P, _I64, _P, _P, _P],
    "dc_ans_encode_chunks": [_P, _U64, _U64, _I64, _P, _P, _P, _P, _P, _U32, _P, _P, _P, _U32, _P, _U64, _P],
    "dc_ans_encode_work_bytes": [_U64, _U64, _I64, _P],
    "dc_assemble_payloads": [_P, _U64, _U64, _I64, _P, _P, _P, _P, _P, _P, _P, _P],
    "dc_quant_absmax": [_P, ctypes.c_int, _P, _I64, _I64, _P, _P, _P],
    "dc_quantize": [_P, ctypes.c_int, _P, _I64, _I64, ctypes.c_double, _P, _P],
    "dc_dequantize": [_P, ctypes.c_double, _P, _I64, _I64, _P, _P],
    "dc_scale_weights": [_P, _P, _I64, _I64, _P, _P],
    "dc_prune_scratch_bytes": [_I64, _I64, _P],
    "dc_prune_scores": [_P, _P, _I64, _I64, _P, _P],
    "dc_prune_tensor": [_P, _P, _I64, _I64, _I64, _P, _P, _P],
    "dc_prune_rows": [_P, _P, _I64, _I64, _I64, _P, _P],
    "dc_w8a8_gemm": [_P, _I64, _I64, _P, _I64, _P, _I64, _P],
    "dc_gemm_tensor_bytes": [],
    "dc_tmap_bytes": [],
    "dc_w8a8_grouped_maps": [_P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P],
    "dc_w8a8_grouped": [_P, _P, _P, _I64, ctypes.c_int, _P],
    "dc_w8a8_grouped_persist": [_P, _P, _P, _I64, ctypes.c_int, ctypes.c_int, _P],
    "dc_fused_item_rows": [],
    "dc_fused_item_k": [],
    "dc_fused_ring_gemm": [_P, _P, _P, _P, _P, _U64, _P, _P, _P, _P, _P, _I64, ctypes.c_int, _P, _P, ctypes.c_int,
                           _P],
    "dc_fused_epi_bytes": [],
}
_RESTYPES = {"dc_last_error": ctypes.c_char_p}

_lib = None


def lib():
    """Load the library (fails loudly: there is no CPU path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is missing; build it with `python -m paper_2502_15443_b200._build`")
    L = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = L
    return L


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the dcomp B200 path has no CPU fallback")
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def call(name: str, *args) -> int:
    rc = getattr(lib(), name)(*args)
    if rc < 0:
        msg = lib().dc_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")
    return rc


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def device_bytes(nbytes: int, device=None) -> torch.Tensor:
    """uint8 device buffer of ``nbytes`` with READ_SLACK readable bytes past
    its end (returned view excludes the slack)."""
    dev = device if device is not None else require_cuda()
    raw = torch.empty(int(nbytes) + READ_SLACK, dtype=torch.uint8, device=dev)
    return raw[: int(nbytes)]


_COPY_POOL = None


def _parallel_copy(dst: "np.ndarray", src: "np.ndarray", piece: int = 32 << 20) -> None:
    """Host memcpy in parallel slices (numpy releases the GIL on large copies)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    global _COPY_POOL
    n = src.size
    if n <= piece:
        np.copyto(dst, src)
        return
    if _COPY_POOL is None:
        _COPY_POOL = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1))
    futs = [_COPY_POOL.submit(np.copyto, dst[i:i + piece], src[i:i + piece]) for i in range(0, n, piece)]
    for f in futs:
        f.result()


def to_device_bytes(data, device=None, pinned: bool = True) -> torch.Tensor:
    """Host bytes-like / uint8 ndarray -> device buffer with read slack.
    Large inputs stream through two pinned staging buffers: the host copy of
    piece i+1 (parallel memcpy) overlaps the H2D DMA of piece i."""
    import numpy as np

    arr = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data.reshape(-1).view(np.uint8)
    out = device_bytes(arr.size, device)
    n = arr.size
    if n == 0:
        return out
    if not pinned or n < (4 << 20):
        out.copy_(torch.from_numpy(arr.copy()))
        return out
    piece = 64 << 20
    stream = torch.cuda.current_stream()
    bufs = [torch.empty(min(piece, n), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    for i, off in enumerate(range(0, n, piece)):
        b = i & 1
        if done[b] is not None:
            done[b].synchronize()  # the DMA out of this staging buffer finished
        ln = min(piece, n - off)
        _parallel_copy(bufs[b].numpy()[:ln], arr[off:off + ln], piece=8 << 20)
        out[off:off + ln].copy_(bufs[b][:ln], non_blocking=True)
        done[b] = torch.cuda.Event()
        done[b].record(stream)
    return out


def to_host(t: torch.Tensor) -> "np.ndarray":
    """Device tensor -> numpy array backed by pinned host memory (one DMA, no
    extra host copy); the array keeps the pinned buffer alive."""
    host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    host.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy()


# `bytes` results (pack returns bytes, as the reference does) are filled in
# place: a fresh bytes object of the right size, written by parallel slice
# copies from the pinned D2H buffer -- a single-threaded .tobytes() of a few
# hundred MB is bound by first-touch page faults (~2 GB/s), the threads fault
# their pages concurrently.  CPython-only: the payload offset of a bytes
# object is checked once; anything unexpected falls back to .tobytes().
_PyBytes_New = ctypes.pythonapi.PyBytes_FromStringAndSize
_PyBytes_New.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
_PyBytes_New.restype = ctypes.py_object


def _bytes_offset() -> int | None:
    import sys
    off = sys.getsizeof(b"") - 1  # header size: the payload follows it
    probe = _PyBytes_New(None, 8)
    ctypes.memmove(id(probe) + off, b"dcomp-ok", 8)
    return off if probe == b"dcomp-ok" else None


try:
    _BYTES_OFF = _bytes_offset()
except Exception:  # noqa: BLE001 - any surprise: plain copies
    _BYTES_OFF = None


def host_to_bytes(src: "np.ndarray") -> bytes:
    """uint8 host array -> bytes, copied by parallel slices into the new object."""
    import numpy as np
    n = int(src.size)
    if _BYTES_OFF is None or n < (64 << 20):
        return src.tobytes()
    out = _PyBytes_New(None, n)
    dst = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(id(out) + _BYTES_OFF))
    _parallel_copy(dst, src.reshape(-1).view(np.uint8), piece=8 << 20)
    return out


def to_bytes(t: torch.Tensor) -> bytes:
    """Device uint8 tensor -> bytes (pinned D2H, then parallel host copies)."""
    return host_to_bytes(to_host(t))


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def encode_work(total: int, chunk_size: int, n_chunks: int, device=None):
    """Device work buffer for dc_ans_encode_chunks (uint8 tensor, size)."""
    import torch
    need = ctypes.c_uint64(0)
    call("dc_ans_encode_work_bytes", int(total), int(chunk_size), int(n_chunks), ctypes.byref(need))
    buf = torch.empty(int(need.value), dtype=torch.uint8, device=device or require_cuda())
    return buf, int(need.value)
