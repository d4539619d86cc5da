"""``dcomp`` command line on the B200 (the reference's cli.py:301-393 surface).

    python -m paper_2502_15443_b200 <command> [flags]      (or .cli)

Same commands, flags, printed text and exit codes as the reference's
``dcomp`` console script -- 0 success, 2 usage, 3 data / format / argument
error, 4 internal error -- but every heavy step runs through this package's
GPU API:

  synth     host generator (the reference's exact PCG64 draws, tensors.py:134-200)
  quantize  DCWT read into pinned memory, weights to the GPU in their stored
            dtype, compression-aware quantize kernels, all-store DCC1 writer
  prune     GPU unpack -> prune kernels (histogram radix select) -> writer
  pack      GPU unpack -> GPU histogram / normalize / rANS encode -> DCC1
  unpack    GPU unpack (validate, decode, CRC) -> all-store DCC1
  analyze   GPU unpack + per-tensor k_hist reports (analyze_quantized) and
            exact standalone blob lengths from the GPU encoder, all tensors
            encoded side by side (DCWT input: host analyze_float, GPU lengths)
  sweep     the alpha sweep on the GPU (sweep.alpha_sweep)
  bench     bench_codecs on a quantized synthetic tensor
  simulate  the latency model / partial-compression planner (host, exact)
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys

import numpy as np

from . import container, dcwt
from .errors import DataFormatError, DcompError, InternalError
from .latency import (
    REFERENCE_PROFILE,
    Architecture,
    CompressionPlan,
    HardwareProfile,
    choose_architecture,
    latency,
    memory_footprint,
    plan_partial,
)
from .pruning import PruneConfig, PruneScope, prune
from .tensors import DEFAULT_SEED, SynthSpec, analyze_float, analyze_quantized, compression_ratio, default_ensemble, \
    synth_ensemble

EXIT_OK, EXIT_USAGE, EXIT_DATA, EXIT_INTERNAL = 0, 2, 3, 4


def _chunks(tensors, chunk_size: int) -> int:
    return -(-sum(t.qvalues.size for t in tensors) // chunk_size)


def _store_plan(tensors, chunk_size: int) -> CompressionPlan:
    return CompressionPlan.block_plan(chunk_size, _chunks(tensors, chunk_size), 0)


def _rewrite_stored(path, bundle_or_tensors, stats, chunk_size: int) -> None:
    container.write_container(path, bundle_or_tensors, stats, chunk_size=chunk_size,
                              plan=_store_plan(bundle_or_tensors, chunk_size))


# --------------------------------------------------------------- pipeline
def cmd_synth(a) -> int:
    pairs = (default_ensemble(a.seed) if a.preset == "default"
             else [synth_ensemble(SynthSpec(rows=a.rows, cols=a.cols, name=a.name), a.seed)])
    dcwt.write_weights(a.out_weights, [w for w, _ in pairs])
    dcwt.write_stats(a.out_stats, [s for _, s in pairs])
    for w, _ in pairs:
        print(f"{w.name}: {w.rows}x{w.cols}")
    print(f"wrote {len(pairs)} tensors to {a.out_weights}, stats to {a.out_stats}")
    return EXIT_OK


def _device_inputs(a):
    """(name, device weights in the stored dtype) + stats, with the
    reference's checks in its order (cli.py:58-64)."""
    weights = dcwt.read_weights_device(a.weights)
    stats = dcwt.read_stats(a.stats)
    for name, _ in weights:
        if name not in stats:
            raise DataFormatError(f"missing activation stats for tensor {name!r}")
    return weights, stats


def _quantize_all(weights, stats, alpha: float):
    import torch

    from .scaling import QuantizedTensor, compute_scale, quantize_device
    out = []
    for name, w in weights:
        sv = compute_scale(stats[name], alpha)
        if len(sv.s) != w.shape[1]:
            raise DcompError(f"{name}: scale length {len(sv.s)} != cols {w.shape[1]}")
        q, ws = quantize_device(w.float() if w.dtype == torch.int8 else w, torch.from_numpy(sv.s), name)
        out.append(QuantizedTensor(name, q.cpu().numpy(), ws, sv))
    return out


def cmd_quantize(a) -> int:
    weights, stats = _device_inputs(a)
    tensors = _quantize_all(weights, stats, a.alpha)
    _rewrite_stored(a.out, tensors, stats, a.chunk_size)
    print(f"quantized {len(tensors)} tensors at alpha={a.alpha} -> {a.out}")
    return EXIT_OK


def cmd_prune(a) -> int:
    b = container.unpack(a.infile)
    cfg = PruneConfig(a.sparsity, PruneScope(a.scope))
    pruned = [prune(t, b.stats[t.name], cfg) for t in b.tensors]
    _rewrite_stored(a.out, pruned, b.stats, b.chunk_size)
    print(f"pruned at sparsity={a.sparsity} scope={a.scope} -> {a.out}")
    return EXIT_OK


def cmd_pack(a) -> int:
    b = container.unpack(a.infile)
    chunk_size = a.chunk_size or b.chunk_size
    n = _chunks(b.tensors, chunk_size)
    block_size = {"store": 0, "ans": 1}.get(a.codec, a.block_size if a.block_size is not None else 1)
    blob = container.pack(b.tensors, b.stats, chunk_size=chunk_size,
                          plan=CompressionPlan.block_plan(chunk_size, n, block_size))
    with open(a.out, "wb") as f:
        f.write(blob)
    total = sum(t.qvalues.size for t in b.tensors)
    print(f"packed {n} chunks (block_size={block_size}) -> {a.out}")
    print(f"payload {total} bytes, file {len(blob)} bytes, CR {compression_ratio(total, len(blob)):.4f}")
    return EXIT_OK


def cmd_unpack(a) -> int:
    b = container.unpack(a.infile)
    _rewrite_stored(a.out, b.tensors, b.stats, b.chunk_size)
    print(f"verified and unpacked {len(b.tensors)} tensors -> {a.out}")
    return EXIT_OK


# -------------------------------------------------------------- reporting
def _blob_lengths(arrays: list[np.ndarray]) -> list[int]:
    """Exact len(compress_blob(x)) for every array, all encoded on the GPU
    side by side (sweep.blob_lengths)."""
    import torch

    from . import native as nv
    from .sweep import blob_lengths
    dev = nv.require_cuda()
    return blob_lengths([torch.from_numpy(np.ascontiguousarray(x).reshape(-1).view(np.uint8)).to(dev)
                         for x in arrays], streams=max(1, min(len(arrays), 64)))


def _layer_row(name, rows, cols, rep, nbytes, ans_bytes) -> dict:
    return {"name": name, "rows": rows, "cols": cols, "near_zero_fraction": rep.near_zero_fraction,
            "byte_entropy": rep.byte_entropy, "uncompressed_bytes": int(nbytes), "ans_bytes": int(ans_bytes)}


def analyze_report(path) -> dict:
    """The reference's analyze document (cli.py:123-184) from GPU passes."""
    with open(path, "rb") as f:
        magic = f.read(4)
    if magic == container.MAGIC:
        b = container.unpack(path)
        info = container.inspect(path)
        lens = _blob_lengths([t.qvalues for t in b.tensors])
        layers = [_layer_row(t.name, t.rows, t.cols, analyze_quantized(t), t.qvalues.size, n)
                  for t, n in zip(b.tensors, lens)]
        extra = {"file_size": info.file_size,
                 "container_cr": (compression_ratio(info.total_uncompressed, info.file_size)
                                  if info.total_uncompressed else 1.0)}
        fmt = "dcc1"
    elif magic == dcwt.MAGIC:
        ws = dcwt.read_weights(path)
        lens = _blob_lengths([w.values for w in ws])
        layers = [_layer_row(w.name, w.rows, w.cols, analyze_float(w), w.values.nbytes, n) for w, n in zip(ws, lens)]
        extra, fmt = {}, "dcwt"
    else:
        raise DataFormatError(f"{path}: neither a DCWT nor a DCC1 file")
    for r in layers:
        r["cr"] = compression_ratio(r["uncompressed_bytes"], r["ans_bytes"])
    elems = sum(r["rows"] * r["cols"] for r in layers)
    u = sum(r["uncompressed_bytes"] for r in layers)
    c = sum(r["ans_bytes"] for r in layers)
    totals = {"uncompressed_bytes": u, "ans_bytes": c, "cr": compression_ratio(u, c) if u else 1.0,
              "near_zero_fraction": (sum(r["near_zero_fraction"] * r["rows"] * r["cols"] for r in layers) / elems
                                     if elems else 0.0)}
    totals.update(extra)
    return {"format": fmt, "layers": layers, "totals": totals}


def cmd_analyze(a) -> int:
    rep = analyze_report(a.infile)
    if a.json:
        print(json.dumps(rep, indent=2))
        return EXIT_OK
    print(f"format: {rep['format']}")
    print(f"{'layer':<12} {'shape':>11} {'near-zero':>9} {'entropy':>8} {'cr':>8}")
    for r in rep["layers"]:
        print(f"{r['name']:<12} {r['rows']:>5}x{r['cols']:<5} {r['near_zero_fraction']:>9.4f} "
              f"{r['byte_entropy']:>8.4f} {r['cr']:>8.4f}")
    t = rep["totals"]
    print(f"{'TOTAL':<12} {'':>11} {t['near_zero_fraction']:>9.4f} {'':>8} {t['cr']:>8.4f}")
    if "container_cr" in t:
        print(f"container: file CR {t['container_cr']:.4f}")
    return EXIT_OK


def cmd_sweep(a) -> int:
    from .sweep import alpha_sweep
    weights = dcwt.read_weights(a.weights)
    stats = dcwt.read_stats(a.stats)
    for w in weights:
        if w.name not in stats:
            raise DataFormatError(f"missing activation stats for tensor {w.name!r}")
    rows = alpha_sweep(weights, stats, sparsity=a.sparsity, per_row=a.scope == PruneScope.PER_ROW.value,
                       seed=a.seed)
    buf = io.StringIO()
    wr = csv.writer(buf)
    wr.writerow(["alpha", "cr", "near_zero", "layer_error"])
    for r in rows:
        wr.writerow([r["alpha"], f"{r['cr']:.6f}", f"{r['near_zero']:.6f}", f"{r['layer_error']:.6f}"])
    if a.out:
        with open(a.out, "w", encoding="utf-8") as f:
            f.write(buf.getvalue())
        print(f"wrote {a.out}")
    else:
        sys.stdout.write(buf.getvalue())
    return EXIT_OK


def cmd_bench(a) -> int:
    from .codec_bench import bench_codecs
    from .scaling import quantize_scaled
    w, st = synth_ensemble(SynthSpec(rows=a.size_mib * 2**20 // 8192, cols=8192, name="bench"), a.seed)
    q = quantize_scaled(w, st, 0.5)
    rows = bench_codecs(q.qvalues.reshape(-1).view(np.uint8), repetitions=a.repetitions)
    if a.json:
        print(json.dumps({"bytes": int(q.qvalues.size), "rows": [r.to_dict() for r in rows]}, indent=2))
        return EXIT_OK
    print(f"{'codec':<7} {'cr':>8} {'compress MB/s':>14} {'decompress MB/s':>16}")
    for r in rows:
        print(f"{r.codec:<7} {r.cr:>8.4f} {r.compress_mbps:>14.1f} {r.decompress_mbps:>16.1f}")
    return EXIT_OK


def _read_json(path, cls):
    with open(path, encoding="utf-8") as f:
        return cls.from_json(f.read())


def cmd_simulate(a) -> int:
    prof = _read_json(a.profile, HardwareProfile) if a.profile else REFERENCE_PROFILE
    if a.plan:
        plan = _read_json(a.plan, CompressionPlan)
    elif a.n_chunks is not None:
        plan = CompressionPlan.block_plan(a.chunk_size, a.n_chunks, a.block_size)
    elif a.budget is None:
        raise DcompError("need --plan or --n-chunks (or --budget with --n-chunks)")
    else:
        plan = None
    if a.budget is not None:
        if a.n_chunks is None:
            raise DcompError("--budget needs --n-chunks and --chunk-size")
        arch = Architecture.GPU_BUFFER if a.arch == "auto" else Architecture(a.arch)
        res = plan_partial(prof, a.n_chunks, a.chunk_size, a.cr, a.budget, arch)
        if a.json:
            doc = json.loads(res.report.to_json())
            doc.update(block_size=res.plan.block_size, feasible=res.feasible)
            print(json.dumps(doc, indent=2))
            return EXIT_OK
        print(f"block_size: {res.plan.block_size}")
        print(f"compressed fraction: {res.plan.compressed_fraction:.4f}")
        print(f"latency: {res.report.per_sample_latency:.6e} s")
        if not res.feasible:
            print("warning: budget infeasible even with all chunks stored", file=sys.stderr)
        return EXIT_OK
    cr = np.where(plan.compressed_mask, a.cr, 1.0)
    arch = (choose_architecture(prof, memory_footprint(plan, cr, buffer_chunks=0), plan.chunk_size)
            if a.arch == "auto" else Architecture(a.arch))
    rep = latency(prof, plan, arch, cr)
    if a.json:
        print(rep.to_json())
        return EXIT_OK
    s = rep.stage_seconds
    print(f"architecture: {rep.architecture.value}")
    print(f"per-sample latency: {rep.per_sample_latency:.6e} s")
    print(f"bottleneck: {rep.bottleneck.value}")
    print(f"stage seconds: loading={s['loading']:.6e} decompression={s['decompression']:.6e} "
          f"compute={s['compute']:.6e}")
    print(f"memory: gpu={rep.memory_used_gpu:.3e} cpu={rep.memory_used_cpu:.3e}")
    return EXIT_OK


# ----------------------------------------------------------------- parser
_SCOPES = [s.value for s in PruneScope]
_COMMANDS = [  # (name, help, handler, [(flags, kwargs)])
    ("synth", "generate a synthetic weights + stats pair", cmd_synth, [
        (("--out-weights",), dict(required=True)), (("--out-stats",), dict(required=True)),
        (("--seed",), dict(type=int, default=DEFAULT_SEED)),
        (("--preset",), dict(choices=["default", "single"], default="default")),
        (("--rows",), dict(type=int, default=512)), (("--cols",), dict(type=int, default=512)),
        (("--name",), dict(default="synth"))]),
    ("quantize", "scale + quantize DCWT weights into a container", cmd_quantize, [
        (("--weights",), dict(required=True)), (("--stats",), dict(required=True)),
        (("--out",), dict(required=True)), (("--alpha",), dict(type=float, default=0.5)),
        (("--chunk-size",), dict(type=int, default=container.DEFAULT_CHUNK_SIZE))]),
    ("prune", "zero the lowest-scoring weight fraction", cmd_prune, [
        (("--in",), dict(dest="infile", required=True)), (("--out",), dict(required=True)),
        (("--sparsity",), dict(type=float, required=True)),
        (("--scope",), dict(choices=_SCOPES, default="per_tensor"))]),
    ("pack", "re-chunk and entropy-code a container", cmd_pack, [
        (("--in",), dict(dest="infile", required=True)), (("--out",), dict(required=True)),
        (("--block-size",), dict(type=int, default=None)), (("--codec",), dict(choices=["ans", "store"], default=None)),
        (("--chunk-size",), dict(type=int, default=None))]),
    ("unpack", "verify a container and rewrite it uncompressed", cmd_unpack, [
        (("--in",), dict(dest="infile", required=True)), (("--out",), dict(required=True))]),
    ("analyze", "distribution and compressibility report", cmd_analyze, [
        (("--in",), dict(dest="infile", required=True)), (("--json",), dict(action="store_true"))]),
    ("sweep", "CR/error sweep over the alpha grid (CSV)", cmd_sweep, [
        (("--weights",), dict(required=True)), (("--stats",), dict(required=True)),
        (("--out",), dict(default=None)), (("--sparsity",), dict(type=float, default=0.0)),
        (("--scope",), dict(choices=_SCOPES, default="per_tensor")),
        (("--seed",), dict(type=int, default=DEFAULT_SEED))]),
    ("bench", "codec throughput benchmark on synthetic weights", cmd_bench, [
        (("--size-mib",), dict(type=int, default=64)), (("--seed",), dict(type=int, default=7)),
        (("--repetitions",), dict(type=int, default=3)), (("--json",), dict(action="store_true"))]),
    ("simulate", "latency model / partial-compression planner", cmd_simulate, [
        (("--profile",), dict(default=None)), (("--plan",), dict(default=None)),
        (("--n-chunks",), dict(type=int, default=None)),
        (("--chunk-size",), dict(type=int, default=container.DEFAULT_CHUNK_SIZE)),
        (("--block-size",), dict(type=int, default=1)), (("--cr",), dict(type=float, default=2.0)),
        (("--arch",), dict(choices=[x.value for x in Architecture] + ["auto"], default="auto")),
        (("--budget",), dict(type=float, default=None)), (("--json",), dict(action="store_true"))]),
]


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="dcomp", description=__doc__)
    sub = p.add_subparsers(dest="command", required=True)
    for name, help_, fn, flags in _COMMANDS:
        sp = sub.add_parser(name, help=help_)
        for f, kw in flags:
            sp.add_argument(*f, **kw)
        sp.set_defaults(func=fn)
    return p


def main(argv=None) -> int:
    """Run one command; argparse usage errors exit 2 (SystemExit), data and
    argument errors return 3, internal errors 4 (cli.py:378-393)."""
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except InternalError as e:
        print(f"internal error: {e}", file=sys.stderr)
        return EXIT_INTERNAL
    except (DcompError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_DATA
    except Exception as e:  # noqa: BLE001 -- the exit-code contract covers everything else
        print(f"internal error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
