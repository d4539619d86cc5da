"""DCWT weights files + stats JSON (the reference's ``dcomp.dcwt``,
/root/reference/pkg/src/dcomp/dcwt.py:1-108) and the B200 ingest path.

Wire format (little-endian, dcwt.py:1-11):

    "DCW1" | u16 version = 1 | u32 tensor_count
    per tensor: u16 name_len | UTF-8 name | u8 dtype | u32 rows | u32 cols
                | rows x cols raw values, row-major

dtype tags 0 = f32, 1 = f64, 2 = i8.  The stats file is a JSON object
{tensor name: [per-input-channel activation max, ...]}.

``read_weights`` / ``write_weights`` / ``read_stats`` / ``write_stats`` are
the reference's functions (same results and exceptions).  B200 additions:

  * ``read_weights_device`` -- the file is read once into pinned host memory
    and each tensor is copied to the GPU in its stored dtype (f32 stays f32:
    the quantize kernels widen to f64 in registers, exactly), so ingest
    moves the file's bytes, not the f64 widening of them;
  * ``quantize_file`` -- DCWT + stats -> compression-aware INT8 on the GPU
    (the reference's ``dcomp quantize`` input path, cli.py:58-78);
  * ``collect_activation_stats`` / ``export_weights`` -- the exporter's
    calibration hooks (exporter export.py:63-123) with the per-channel
    max|x| reduced on the device by ``dc_channel_absmax`` (no host copy of
    activations, one sync at the end).
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from .errors import BadMagicError, DataFormatError, TruncatedError, UnsupportedVersionError
from .tensors import ActivationStats, WeightTensor

MAGIC = b"DCW1"
VERSION = 1

_DTYPES = {0: np.dtype("<f4"), 1: np.dtype("<f8"), 2: np.dtype("i1")}
_TAGS = {np.dtype("float32"): 0, np.dtype("float64"): 1, np.dtype("int8"): 2}
_TORCH = {0: torch.float32, 1: torch.float64, 2: torch.int8}


# ------------------------------------------------------------- writing
def write_weights(path, tensors, dtype=np.float64) -> None:
    """Write WeightTensors (or (name, 2-D array) pairs) as one DCWT file."""
    dt = np.dtype(dtype)
    tag = _TAGS[dt]
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<HI", VERSION, len(tensors)))
        for t in tensors:
            name, values = (t.name, t.values) if isinstance(t, WeightTensor) else t
            nb = name.encode("utf-8")
            if len(nb) > 0xFFFF:
                raise ValueError(f"tensor name too long: {name!r}")
            rows, cols = values.shape
            f.write(struct.pack("<H", len(nb)) + nb + struct.pack("<BII", tag, rows, cols))
            f.write(np.ascontiguousarray(values, dtype=dt.newbyteorder("<")).tobytes())


def write_stats(path, stats) -> None:
    """ActivationStats (or (name, array) pairs) -> the stats JSON."""
    doc = {}
    for st in stats:
        name, cm = (st.name, st.channel_max) if isinstance(st, ActivationStats) else st
        doc[name] = np.asarray(cm, dtype=np.float64).tolist()
    with open(path, "w", encoding="utf-8") as f:
        json.dump(doc, f)


# ------------------------------------------------------------- reading
def _directory(buf) -> list[tuple[str, int, int, int, int]]:
    """(name, tag, rows, cols, data offset) per tensor, with the reference
    reader's checks and messages (dcwt.py:48-87)."""
    pos = 0

    def take(n: int):
        nonlocal pos
        if pos + n > len(buf):
            raise TruncatedError(f"truncated file at offset {pos}")
        out = buf[pos:pos + n]
        pos += n
        return out

    if bytes(take(4)) != MAGIC:
        raise BadMagicError("not a DCWT file")
    version, count = struct.unpack("<HI", take(6))
    if version != VERSION:
        raise UnsupportedVersionError(f"unsupported DCWT version {version}")
    out = []
    for _ in range(count):
        (nl,) = struct.unpack("<H", take(2))
        name = bytes(take(nl)).decode("utf-8")
        tag, rows, cols = struct.unpack("<BII", take(9))
        if tag not in _DTYPES:
            raise DataFormatError(f"{name}: unknown dtype tag {tag}")
        at = pos
        take(rows * cols * _DTYPES[tag].itemsize)
        out.append((name, tag, rows, cols, at))
    if pos != len(buf):
        raise DataFormatError(f"{len(buf) - pos} trailing bytes after tensor data")
    return out


def read_weights(path) -> list[WeightTensor]:
    """DCWT file -> WeightTensors, values widened to float64 (dcwt.py:65-87)."""
    with open(path, "rb") as f:
        buf = f.read()
    return [WeightTensor(name, np.frombuffer(buf, _DTYPES[tag], rows * cols, at).reshape(rows, cols)
                         .astype(np.float64))
            for name, tag, rows, cols, at in _directory(buf)]


def read_stats(path) -> dict[str, ActivationStats]:
    """Stats JSON -> {name: ActivationStats} (dcwt.py:100-108)."""
    with open(path, encoding="utf-8") as f:
        try:
            doc = json.load(f)
        except json.JSONDecodeError as e:
            raise DataFormatError(f"stats file is not valid JSON: {e}") from e
    if not isinstance(doc, dict):
        raise DataFormatError("stats file must be a JSON object")
    return {name: ActivationStats(name, np.asarray(v, dtype=np.float64)) for name, v in doc.items()}


# --------------------------------------------------------- B200 ingest
def read_weights_device(path, device=None) -> list[tuple[str, torch.Tensor]]:
    """DCWT file -> [(name, device tensor in the stored dtype)]: one read
    into pinned host memory, then one H2D copy per tensor (same checks and
    exceptions as ``read_weights``)."""
    from . import native as nv
    dev = device or nv.require_cuda()
    with open(path, "rb") as f:
        f.seek(0, 2)
        size = f.tell()
        f.seek(0)
        pin = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        view = pin.numpy()
        got = f.readinto(memoryview(view))
    directory = _directory(view[:got])
    out = []
    for name, tag, rows, cols, at in directory:
        nbytes = rows * cols * _DTYPES[tag].itemsize
        d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        d.copy_(pin[at:at + nbytes], non_blocking=True)
        out.append((name, d.view(_TORCH[tag]).view(rows, cols)))
    torch.cuda.current_stream(dev).synchronize()  # the pinned staging buffer is released here
    return out


def quantize_file(weights_path, stats_path, alpha: float, device=None):
    """DCWT + stats -> [QuantizedTensor] and {name: ActivationStats} with the
    compression-aware quantization on the GPU straight from the stored dtype
    (the reference reads, widens to f64 and quantizes on the host:
    cli.py:58-78 -> scaling.py:108-111)."""
    from .errors import DcompError
    from .scaling import QuantizedTensor, compute_scale, quantize_device
    stats = read_stats(stats_path)
    out = []
    for name, w in read_weights_device(weights_path, device):
        if name not in stats:
            raise DcompError(f"no activation stats for tensor {name!r}")
        if w.dtype == torch.int8:
            w = w.to(torch.float32)  # exact: the kernels widen f32 to f64
        sv = compute_scale(stats[name], alpha)
        if len(sv.s) != w.shape[1]:
            raise DcompError(f"{name}: scale length {len(sv.s)} != cols {w.shape[1]}")
        q, ws = quantize_device(w, torch.from_numpy(sv.s), name)
        out.append(QuantizedTensor(name, q.cpu().numpy(), ws, sv))
    return out, stats


# ------------------------------------------------------ exporter hooks
_DTYPE_CODE = {torch.float64: 0, torch.float32: 1, torch.bfloat16: 2, torch.float16: 3}


def collect_activation_stats(model: torch.nn.Module, calibration, out_path=None) -> dict[str, np.ndarray]:
    """Per-input-channel max|x| entering every nn.Linear over the calibration
    samples (the exporter's collect_activation_stats, export.py:77-123):
    a forward pre-hook per linear feeds its input to dc_channel_absmax, which
    folds it into a device-resident running max; one host sync at the end."""
    from . import native as nv
    acc: dict[str, torch.Tensor] = {}
    hooks = []

    def make_hook(name):
        def hook(_mod, inputs):
            x = inputs[0].detach()
            if x.dtype not in _DTYPE_CODE:
                x = x.to(torch.float32)
            x = x.reshape(-1, x.shape[-1]).contiguous()
            if not x.is_cuda:
                raise nv.NativeUnavailable("collect_activation_stats runs the model on a CUDA device")
            a = acc.get(name)
            if a is None:
                a = acc[name] = torch.zeros(x.shape[1], dtype=torch.int64, device=x.device)
            nv.call("dc_channel_absmax", x.data_ptr(), _DTYPE_CODE[x.dtype], x.shape[0], x.shape[1], a.data_ptr(),
                    nv.stream_ptr())
        return hook

    for name, mod in model.named_modules():
        if isinstance(mod, torch.nn.Linear):
            hooks.append(mod.register_forward_pre_hook(make_hook(name)))
    if not hooks:
        raise ValueError("model contains no linear layers")
    model.eval()
    n = 0
    try:
        with torch.no_grad():
            for sample in calibration:
                if isinstance(sample, dict):
                    model(**sample)
                elif isinstance(sample, (tuple, list)):
                    model(*sample)
                else:
                    model(sample)
                n += 1
    finally:
        for h in hooks:
            h.remove()
    if n == 0:
        raise ValueError("need at least one calibration sample")
    stats = {name: a.cpu().numpy().view(np.float64).copy() for name, a in acc.items()}
    if out_path is not None:
        write_stats(out_path, list(stats.items()))
    return stats


def export_weights(model: torch.nn.Module, out_path) -> list[dict]:
    """Every nn.Linear's weight (rows = out channels, cols = in channels) to a
    float32 DCWT file (export.py:63-75); returns [{"name", "rows", "cols"}]."""
    pairs = [(name, mod.weight.detach().float().cpu().numpy()) for name, mod in model.named_modules()
             if isinstance(mod, torch.nn.Linear)]
    if not pairs:
        raise ValueError("checkpoint contains no 2-D weight matrices")
    write_weights(out_path, pairs, dtype=np.float32)
    return [{"name": n, "rows": int(v.shape[0]), "cols": int(v.shape[1])} for n, v in pairs]
