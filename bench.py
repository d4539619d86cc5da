#!/usr/bin/env python
"""Benchmark driver (contract: one JSON line on rank 0).

Workload: the north star's target configuration (BASELINE.json north_star,
config C4's shape): OPT-6.7B-shaped W8A8 weights from a deterministic
integer-hash generator (~N(0, 0.2); channel maxima as SynthSpec),
compression-aware quantized (alpha 0.5) and packed FULLY compressed into
DCC1 at the reference's default 16 MiB chunks by the GPU encoder.  One step
= the reference's unpack work on the container resident in HBM: validate
every chunk, split-point parallel rANS decode, raw copy of stored chunks,
CRC32 of every decoded chunk checked against the chunk table
(container.py:296-331).

  value     decompressed GB/s of that step (container resident in HBM)
  e2e       same metric through the public API ``container.unpack`` from
            pinned HOST bytes (H2D, decode, CRC verify, D2H of every weight);
            ``e2e.index_less`` = the reference's exact call (no sidecar)
  roofline  dominant kernel (k_decode_segments): algorithmic bytes
            N * (1 + 1/CR) per launch / its CUDA-event time vs measured HBM
  decode_step_tokens  fused decode -> tcgen05 W8A8 vs INT8 at B = 1, 16
  extra     the same measurements on OPT-1.3B (config C2)
  cpu_baseline  the C oracle (a restatement of the reference's numba
            kernels) decoding a bounded sample on this box's host cores

``--impl reference`` times the reference's unpack (the oracle port, all host
threads) on whole-layer samples of the SAME container (identical bytes; both
lines carry the digest of its header + chunk table); under torchrun only
rank 0 runs it.  Multi-GPU: one process per GPU, each decodes its own copy
(weak scaling, no collective on the data path); time = max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode GB/s (decompressed INT8) vs HBM peak; tokens/s compressed vs INT8; CR"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--model", default="opt-6.7b")
    p.add_argument("--extra-model", default="opt-1.3b", help="second workload reported as an extra key ('none')")
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--chunk-size", type=int, default=16 * 2**20)
    p.add_argument("--alpha", type=float, default=0.5)
    p.add_argument("--seg-shift", type=int, default=8)
    p.add_argument("--layers", type=int, default=None, help="limit layers (debug only)")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-tp-shard", action="store_true", help="skip the single-GPU TP-8 shard measurement")
    p.add_argument("--no-index-less", action="store_true", help="skip the index-less (serial) unpack step")
    p.add_argument("--no-disk", action="store_true", help="skip the disk-tier streaming measurement")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel: str, config: dict):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/traffic.json, tools/ncu_traffic.py) when it was taken on this
    exact workload; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f)[kernel]
        if all(config.get(k) == v for k, v in e["config"].items()):
            pipes = {k: e[k] for k in ("alu_pipe_pct", "fma_pipe_pct", "issue_active_pct", "l1tex_pct") if k in e}
            return e["dram_bytes_per_launch"], e["report"], pipes
    except Exception:
        pass
    return None, None, {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_sample_decode(image_bytes: bytes, entries, budget_s: float, threads: int):
    """C oracle decoding a bounded sample of the container's chunks on host
    cores (the reference's algorithm, restated in C; oracle/)."""
    from oracle import oracle as O
    O.lib()
    import numpy as np
    jobs, labels, total = [], [], 0
    sample = []
    for i, e in enumerate(entries):
        if e["codec"] == 1:
            sample.append(i)
        if len(sample) >= max(threads * 4, 16):
            break
    blobs = [image_bytes[int(entries[i]["file_offset"]): int(entries[i]["file_offset"] + entries[i]["comp_len"])]
             for i in sample]
    outs = [np.empty(int(entries[i]["uncomp_len"]), np.uint8) for i in sample]
    nbytes = sum(o.size for o in outs)

    def run():
        from concurrent.futures import ThreadPoolExecutor
        per = max(1, -(-len(blobs) // threads))
        parts = [(list(zip(blobs[k:k + per], outs[k:k + per])), sample[k:k + per]) for k in range(0, len(blobs), per)]
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda p: O.decode_blobs_into(p[0], p[1]), parts))

    run()  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        run()
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    del jobs, labels, total
    return nbytes * reps / dt / 1e9, f"{len(sample)} ANS chunks x {reps} reps ({nbytes / 1e6:.1f} MB each rep)", threads


def synth_spec(model: str, seed: int, layers: int | None = None):
    """The bench workload, shared by both arms: (name, rows, cols) per linear
    (exporter order), a uint32 hash key per tensor for the integer-hash
    weights (synth.hash_weights on the GPU arm, oracle or_gen_weights on the
    reference arm: the same f64 values) and host-drawn channel maxima
    (log-normal(-1, 1), 2 % outlier channels x20, as SynthSpec)."""
    import numpy as np
    from paper_2502_15443_b200.tensors import model_layout  # the shape table only
    layout = model_layout(model)
    if layers is not None:
        per = sum(1 for n, _, _ in layout if n.startswith("layers.0."))
        layout = layout[: per * layers]
    keys, cms = [], []
    for i, (_, _, c) in enumerate(layout):
        keys.append((seed * 0x9E3779B1 + i * 0x7F4A7C15 + 0x632BE5AB) & 0xFFFFFFFF)
        rng = np.random.default_rng([seed, i])
        cm = rng.lognormal(-1.0, 1.0, c)
        k = int(round(0.02 * c))
        if k:
            cm[rng.choice(c, k, replace=False)] *= 20.0
        cms.append(cm)
    return layout, keys, cms


def container_digest(head: bytes) -> str:
    """sha256 of a DCC1 file's header + chunk table (every chunk's codec,
    offsets, lengths and CRC32 of its decompressed bytes): equal digests =
    the same container bytes in both arms."""
    import hashlib
    import struct
    (hlen,) = struct.unpack_from("<I", head, 6)
    (count,) = struct.unpack_from("<I", head, 10 + hlen)
    return hashlib.sha256(bytes(head[:14 + hlen + 4 + 29 * count])).hexdigest()[:32]


REF_SAMPLE_BYTES = 1 << 30  # bytes of weights one reference-arm step unpacks (whole layers)


def run_reference(args):
    """--impl reference: the reference's unpack algorithm on host cores (the
    oracle/ C port of its numba kernels + zlib CRC + tensor slicing, all host
    threads), on the SAME container our arm decodes (identical bytes: the
    digest of header + chunk table is printed), each step one bounded
    sample: a DCC1 container of whole consecutive layers (~1 GiB of weights)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    O.lib()
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    layout, keys, cms = synth_spec(args.model, args.seed, args.layers)

    def make(i):
        name, r, c = layout[i]
        s = O.compute_scale(cms[i], args.alpha)
        q, ws = O.gen_quantize(keys[i], r, c, s)
        return (name, q, ws, args.alpha, s, cms[i])

    with ThreadPoolExecutor(max_workers=threads) as ex:
        entries = list(ex.map(make, range(len(layout))))
    chunk = args.chunk_size
    data = O.pack(entries, chunk, threads=threads)
    digest = container_digest(data)
    raw_total = sum(e[1].size for e in entries)
    file_total = len(data)
    del data
    # the sample: whole layers from the front, about REF_SAMPLE_BYTES of weights
    per = sum(1 for n, _, _ in layout if n.startswith("layers.0.")) or len(layout)
    layer_bytes = sum(r * c for _, r, c in layout[:per])
    n_layers = max(1, min(len(layout) // per, REF_SAMPLE_BYTES // max(layer_bytes, 1)))
    sample = O.pack(entries[: per * n_layers], chunk, threads=threads)
    raw = sum(e[1].size for e in entries[: per * n_layers])
    del entries
    t_build = time.perf_counter() - t0
    for _ in range(args.warmup):
        O.unpack(sample, threads=threads)
    times = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        O.unpack(sample, threads=threads)
        times.append(time.perf_counter() - t1)
    dt = sum(times)
    v = raw * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args, raw_total, file_total, digest),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"unpack (decode on {threads} threads in the reference's groups of four "
                                   f"chunks + serial zlib CRC of every chunk + tensor slicing) of a DCC1 "
                                   f"container of layers 0-{n_layers - 1} ({raw / 1e6:.0f} MB of weights, "
                                   f"{-(-raw // chunk)} chunks) per step, cut from the same weights "
                                   f"as the full container (digest {digest})"},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "build_s": t_build,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, raw: int, file_bytes: int, digest: str) -> dict:
    return {"workload": f"{args.model}-shaped W8A8 weights (hash-generated ~N(0, 0.2), SynthSpec channel maxima, "
                        f"compression-aware quantized at alpha {args.alpha}), fully compressed DCC1 at "
                        f"{args.chunk_size >> 20} MiB chunks; one step = unpack the container (validate + rANS "
                        f"decode + CRC32 verify of every chunk)",
            "weights_shape": args.model, "chunk_size": args.chunk_size, "raw_bytes": raw, "file_bytes": file_bytes,
            "cr": raw / file_bytes, "container_digest": digest, "seed": args.seed,
            "n_chunks": -(-raw // args.chunk_size),
            "l2": "inputs (compressed) and outputs exceed the 126 MB L2",
            "parallelism": (f"one container chunk-sharded over {args.gpus} GPUs (contiguous chunk ranges "
                            f"balanced by decompressed bytes, no data-path collective)" if args.gpus > 1
                            else "single GPU")}


class DeviceUnpack:
    """One bench step: the reference's unpack work on a container resident in
    HBM (container.py:296-331) -- prologue validation, split-point rANS decode
    of every ANS chunk, raw copy of stored chunks, CRC32 of every decoded chunk
    compared with the chunk table -- with no host synchronisation (verdicts
    accumulate on the device and are checked after the timed region)."""

    def __init__(self, pm, dev, chunks=None):
        """``chunks`` = (c0, c1): only that chunk range (this rank's shard of
        the container under chunk sharding, sharded.plan_shards)."""
        import torch
        from paper_2502_15443_b200 import engine
        from paper_2502_15443_b200 import native as nv
        self.pm, self.nv = pm, nv
        c0, c1 = chunks or (0, pm.jobs.n)
        ent = pm.entries[c0:c1]
        j = pm.jobs
        self.jobs = j if (c0, c1) == (0, j.n) else engine.JobTable.build(
            j.blob_off[c0:c1], j.blob_len[c0:c1], j.out_off[c0:c1], j.out_len[c0:c1], j.codec[c0:c1], dev)
        ix = pm.index
        self.index = ix if (c0, c1) == (0, j.n) else engine.SegmentIndex(
            ix.seg_shift, ix.seg_base[c0:c1], ix.n_segs, ix.d_seg_base[c0:c1].contiguous(), ix.d_state, ix.d_off,
            h_off=ix.host_offsets())
        self.tasks = pm.tasks if (c0, c1) == (0, j.n) else self.index.tasks(self.jobs, np.ones(self.jobs.n, bool))
        self.range = (int(j.out_off[c0]), int(j.out_off[c1 - 1] + j.out_len[c1 - 1])) if c1 > c0 else (0, 0)
        self.raw_bytes = self.range[1] - self.range[0]
        self.ans_raw = int(ent["uncomp_len"][ent["codec"] == 1].sum())
        self.ans_comp = int(ent["comp_len"][ent["codec"] == 1].sum())
        self.out = nv.device_bytes(pm.raw_bytes, dev)
        n = max(self.jobs.n, 1)
        self.status = torch.zeros(n, dtype=torch.int32, device=dev)
        self.crc = torch.zeros(n, dtype=torch.int32, device=dev)
        self.want = torch.from_numpy(ent["crc32"].astype(np.uint32).view(np.int32).copy()).to(dev)
        self.bad = torch.zeros(1, dtype=torch.int32, device=dev)
        self.has_store = bool((ent["codec"] == 0).any())
        self.max_len = int(self.jobs.out_len.max()) if self.jobs.n else 0
        self.events = []
        self.launches = 4 + int(self.has_store)  # validate, decode, [store], crc pieces + finalize

    def __call__(self, record: bool = False):
        import torch
        from paper_2502_15443_b200 import engine
        pm, j, nv = self.pm, self.jobs, self.nv
        if j.n == 0:
            return
        sp = nv.stream_ptr()
        engine.validate(pm.image, j, self.status)
        if record:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        engine.decode_segments(pm.image, j, self.index, self.tasks, self.out, self.status)
        if record:
            ev[1].record()
            self.events.append(ev)
        if self.has_store:
            engine.store_copy(pm.image, j, self.out)
        nv.call("dc_crc32_ranges", self.out.data_ptr(), self.out.numel(), j.d_out_off.data_ptr(), j.d_out_len.data_ptr(), j.n,
                self.max_len, self.crc.data_ptr(), sp)
        self.bad |= (self.crc[: j.n] != self.want).any().to(torch.int32) | (self.status[: j.n] != 0).any().to(
            torch.int32)

    def kernel_ms(self) -> float:
        return sum(a.elapsed_time(b) for a, b in self.events) / max(len(self.events), 1)


def allreduce_max(v: float, dev) -> float:
    """Max over ranks (NCCL on the device; CPU tensor under gloo)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_steps(fn, steps: int, world: int, dev):
    """K steps between barriers + device syncs; CUDA-event time, max over ranks."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    return allreduce_max(ms, dev) if world > 1 else ms


def time_ms(fn, iters):
    import torch
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def build_packed(args, model: str, dev):
    import torch
    from paper_2502_15443_b200 import synth
    t0 = time.perf_counter()
    layout, keys, cms = synth_spec(model, args.seed, args.layers)
    m = synth.build_hash_model(model, layout, keys, cms, alpha=args.alpha, device=dev)
    pm = synth.pack_model(m, args.chunk_size, seg_shift=args.seg_shift)
    torch.cuda.synchronize()
    head = pm.image[:14].cpu().numpy().tobytes()
    hlen = int.from_bytes(head[6:10], "little")
    digest = container_digest(pm.image[:14 + hlen + 4 + 29 * pm.jobs.n].cpu().numpy().tobytes())
    return m, pm, digest, time.perf_counter() - t0


def decode_step_tokens(m, pm, out, dev, iters, batches=(1, 16), unfused_step=None):
    """Decode-step tokens/s: every linear of the model once for B tokens --
    INT8 weights vs fused compressed (decode -> TMEM -> tcgen05) [vs decode
    to HBM then INT8 GEMM].  Exactness is checked before timing."""
    import torch
    from paper_2502_15443_b200.gemm import FusedRing, GroupedInt8
    offs = m.offsets()[:-1]
    raw = m.nbytes
    w_int8 = [m.payload[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
    w_dec = [out[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
    tokens = {}
    for B in batches:
        gx = torch.Generator(device=dev)
        gx.manual_seed(7 + B)
        xs = [torch.randint(-127, 128, (B, c), generator=gx, device=dev, dtype=torch.int8) for _, c in m.shapes]
        gi = GroupedInt8(w_int8, xs, B)
        fc = FusedRing(pm.image, pm.jobs, pm.index, pm.chunk_size, m.shapes, offs, xs, B)
        gi.run()
        fc.run()
        torch.cuda.synchronize()
        if (fc.check() != 0).any() or not all(torch.equal(a, b) for a, b in zip(gi.accs, fc.accs)):
            raise SystemExit("fused decode-GEMM mismatch vs INT8 GEMM")
        t_i8 = time_ms(gi.run, iters)
        t_fu = time_ms(fc.run, iters)
        row = {"int8_tok_s": B / (t_i8 / 1e3), "compressed_fused_tok_s": B / (t_fu / 1e3), "int8_ms": t_i8,
               "fused_ms": t_fu, "fused_vs_int8": t_i8 / t_fu, "int8_weight_gbs": raw / (t_i8 / 1e3) / 1e9}
        del fc
        # the full W8A8 layer path from fp32 activations in one call: prologue
        # (X / s, per-tensor absmax, int8) + fused decode -> tcgen05 + dequant epilogue
        try:
            from paper_2502_15443_b200.gemm import CompressedLinears
            cl = CompressedLinears(pm.image, pm.jobs, pm.index, pm.chunk_size, m.shapes, offs, m.w_scales,
                                   [s.cpu().numpy() for s in m.s], B)
            for xb in cl.x_in:
                xb.normal_(generator=gx)
            cl.run()
            torch.cuda.synchronize()
            if (cl.check() != 0).any():
                raise RuntimeError("fp-activation path chain check failed")
            t_fp = time_ms(cl.run, iters)
            row.update({"compressed_fp_act_tok_s": B / (t_fp / 1e3), "fp_act_ms": t_fp})
            del cl
        except Exception as e:  # report, never hide
            row["fp_act_error"] = repr(e)[:200]
        if unfused_step is not None:
            gd = GroupedInt8(w_dec, xs, B)
            t_un = time_ms(lambda: (unfused_step(), gd.run()), iters)
            row.update({"compressed_unfused_tok_s": B / (t_un / 1e3), "unfused_ms": t_un})
            del gd
        tokens[f"B{B}"] = row
        del gi
    return tokens


def sharded_e2e(args, host_file: bytes, side: bytes, raw: int, rank: int, world: int, dev) -> dict:
    """N GPUs, end to end through the public sharded API: every rank calls
    sharded.unpack_shard(file bytes, rank, world, index=sidecar) -- it reads
    only its chunk range's bytes and split points, H2D, validate + decode +
    CRC on its GPU, verdict all-reduce -- then copies its decoded range back
    to pinned host memory.  Time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2502_15443_b200 import sharded
    times = []
    host_out = None
    for i in range(args.e2e_steps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = sharded.unpack_shard(host_file, rank, world, index=side)
        if host_out is None:
            host_out = torch.empty(r.out.numel(), dtype=torch.uint8, pin_memory=True)
        host_out.copy_(r.out[: host_out.numel()])
        torch.cuda.synchronize()
        dt = allreduce_max(time.perf_counter() - t0, dev)
        if i >= 1:
            times.append(dt)
    e2e_s = statistics.median(times)
    return {"value": raw / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": len(host_file) + len(side),
            "d2h_bytes_per_step": raw,
            "api": f"sharded.unpack_shard(file bytes, rank, {world}, index=sidecar) on every rank + D2H of each "
                   f"rank's decoded range (max over ranks)"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    args.gpus = world  # the config names the ranks actually running
    # BENCH_DIST_BACKEND=gloo + BENCH_ONE_GPU=1: every rank on cuda:0 (a
    # functional check of the N > 1 path on a one-GPU box; never a measurement)
    if os.environ.get("BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)

    from paper_2502_15443_b200 import container, engine, native
    native.require_cuda()

    m, pm, digest, t_build = build_packed(args, args.model, dev)
    raw = pm.raw_bytes
    comp = pm.comp_bytes
    cr_file = raw / pm.file_bytes
    # N GPUs: one container, chunk-sharded (sharded.plan_shards): every rank
    # unpacks only its contiguous chunk range -- strong scaling, no collective
    # on the data path
    from paper_2502_15443_b200 import sharded
    shard = sharded.plan_shards(pm.entries, world)[rank]
    unp = DeviceUnpack(pm, dev, chunks=(shard.c0, shard.c1))
    out = unp.out
    r0, r1 = unp.range

    clocks = ClockSampler(local).__enter__()
    time.sleep(0.5)  # let nvidia-smi start sampling before the timed region
    for _ in range(args.warmup):
        unp()
    torch.cuda.synchronize()
    if int(unp.bad.item()) != 0 or not torch.equal(out[r0:r1], m.payload[r0:r1]):
        raise SystemExit("unpack mismatch: status / CRC verdicts or GPU output != encoder input")
    # the timed region; the dominant kernel's own duration is taken from events
    # around its launch inside every timed step (same stream)
    ms = time_steps(lambda: unp(record=True), args.steps, world, dev)
    clocks.__exit__(None, None, None)
    if int(unp.bad.item()) != 0:
        raise SystemExit("unpack verdicts changed inside the timed region")
    kms = unp.kernel_ms()
    value = raw * args.steps / (ms / 1e3) / 1e9  # the whole container per step, all ranks together
    hbm, peak_kind = peaks()
    alg_bytes = unp.ans_raw + unp.ans_comp  # this rank's decompressed bytes written + compressed bytes read
    achieved = alg_bytes / (kms / 1e3) / 1e9

    full_status = torch.zeros(max(pm.jobs.n, 1), dtype=torch.int32, device=dev)

    def decode_only():
        engine.decode_segments(pm.image, pm.jobs, pm.index, pm.tasks, out, full_status)
        if unp.has_store:
            engine.store_copy(pm.image, pm.jobs, out)

    # decode-step tokens/s of the whole model on one GPU (N > 1: the TP key below)
    tokens = (decode_step_tokens(m, pm, out, dev, max(5, min(args.steps // 5, 20)), unfused_step=decode_only)
              if world == 1 else None)
    offs = m.offsets()[:-1]

    # GPU_CPU tier: weights in pinned host memory streamed over
    # PCIe every step, raw INT8 vs the compressed container + on-GPU decode,
    # each followed by the grouped W8A8 GEMM; with the planner's prediction
    streaming_tier = None
    try:
        if world > 1:  # N ranks would share one host's PCIe links: single-GPU measurement only
            raise RuntimeError("measured at N=1 only")
        import importlib
        from paper_2502_15443_b200 import adaptive, streaming
        latency = importlib.import_module("paper_2502_15443_b200.latency")  # the package re-exports a function of that name
        streaming_tier = streaming.measure(m.payload, m.shapes, offs, pm.image, pm.jobs, pm.index, ntok=1,
                                           iters=5, groups=16)
        h2d = adaptive.measure_h2d_gbs(1 << 28)
        prof = latency.HardwareProfile(B_stoc=7.0, B_ctog=h2d, B_gpu=hbm, D_max=raw / (kms / 1e3) / 1e9, c_sat=1.0,
                                       I_gpu=tokens["B1"]["int8_weight_gbs"], mem_gpu=1e12, mem_cpu=1e12)
        n_ch = int(pm.jobs.n)
        arch = latency.Architecture.GPU_CPU
        none = latency.CompressionPlan.block_plan(args.chunk_size, n_ch, 0)
        full = latency.CompressionPlan.block_plan(args.chunk_size, n_ch, 1)
        streaming_tier.update({
            "h2d_gbs": h2d,
            "predicted_raw_ms": latency.latency(prof, none, arch).per_sample_latency * 1e3,
            "predicted_compressed_ms": latency.latency(prof, full, arch, raw / comp).per_sample_latency * 1e3})
    except Exception as e:  # report, never hide
        streaming_tier = {"skipped" if world > 1 else "error": repr(e)[:300]}

    # GPU_DISK tier (B_stoc): raw INT8 file vs DCC1 file read from disk every
    # step (O_DIRECT), fused decode -> GEMM vs INT8 GEMM; N=1 only
    disk_tier = None
    if world == 1 and not args.no_disk:
        try:
            import importlib
            from paper_2502_15443_b200 import adaptive, streaming
            disk_tier = streaming.measure_disk(m.payload, m.shapes, offs, pm.image, pm.jobs, pm.index, ntok=1,
                                               iters=3, workdir=os.path.join(ROOT, "gpurun_out"))
            # the reference's latency model for its STORAGE architecture, B_stoc =
            # the measured raw read rate of this disk
            latency = importlib.import_module("paper_2502_15443_b200.latency")
            stoc = disk_tier["raw_read_gbs"]
            dprof = latency.HardwareProfile(B_stoc=stoc, B_ctog=adaptive.measure_h2d_gbs(1 << 28), B_gpu=hbm,
                                            D_max=raw / (kms / 1e3) / 1e9, c_sat=1.0,
                                            I_gpu=tokens["B1"]["int8_weight_gbs"], mem_gpu=1e12, mem_cpu=1e12)
            n_ch = int(pm.jobs.n)
            arch = latency.Architecture.STORAGE
            none = latency.CompressionPlan.block_plan(args.chunk_size, n_ch, 0)
            full = latency.CompressionPlan.block_plan(args.chunk_size, n_ch, 1)
            disk_tier.update({
                "B_stoc_gbs": stoc,
                "predicted_raw_ms": latency.latency(dprof, none, arch).per_sample_latency * 1e3,
                "predicted_compressed_ms": latency.latency(dprof, full, arch, raw / comp).per_sample_latency * 1e3})
        except Exception as e:  # report, never hide
            disk_tier = {"error": repr(e)[:300]}

    # config C5 under torchrun: LLaMA-13B-shaped tensor parallelism across
    # the ranks (fused compressed vs INT8 per rank + NCCL int32 all-reduce)
    tp = None
    if world > 1:
        try:
            from paper_2502_15443_b200 import tp_step
            tps = tp_step.TPDecodeStep("llama-13b", world, rank, ntok=1, device=dev)
            ok = tps.check()
            tp = tp_step.measure(tps, iters=10)
            tp.update({"model": "llama-13b", "tp": world, "ntok": 1, "fused_equals_int8": ok,
                       "int8_tok_s": 1e3 / tp["int8_step_ms"], "compressed_tok_s": 1e3 / tp["compressed_fused_step_ms"]})
            del tps
            torch.cuda.empty_cache()
        except Exception as e:  # report, never hide
            tp = {"error": repr(e)[:300]}
    elif not args.no_tp_shard:
        # one GPU: rank 0's shard of the TP-8 split, compute only (the all-reduce
        # needs the other ranks; its share is measured under torchrun)
        try:
            from paper_2502_15443_b200 import tp_step
            tps = tp_step.TPDecodeStep("llama-13b", 8, 0, ntok=1, device=dev)
            ok = tp_step.check_local(tps)
            tp = tp_step.measure_local(tps, iters=10)
            tp.update({"model": "llama-13b", "tp": 8, "rank": 0, "ntok": 1, "scope": "rank-0 shard compute only",
                       "fused_equals_int8": ok})
            del tps
            torch.cuda.empty_cache()
        except Exception as e:  # report, never hide
            tp = {"error": repr(e)[:300]}

    # e2e through the public API from host bytes (rank 0 reports its own)
    host_file = pm.image.cpu().numpy().tobytes()
    side = pm.index.to_bytes(container.binding_of(host_file))
    # the step's inputs (container file + split-point sidecar) sit in pinned
    # host memory, as the contract asks; unpack copies them straight to HBM
    pin_file = torch.empty(len(host_file), dtype=torch.uint8, pin_memory=True)
    pin_file.numpy()[:] = np.frombuffer(host_file, np.uint8)
    pin_side = torch.empty(len(side), dtype=torch.uint8, pin_memory=True)
    pin_side.numpy()[:] = np.frombuffer(side, np.uint8)
    if world > 1:
        e2e = sharded_e2e(args, host_file, side, raw, rank, world, dev)
    else:
        e2e_times = []
        e2e_phases = []
        for i in range(args.e2e_steps + 2):  # 2 untimed: pinned output blocks get cached
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            bundle = container.unpack(pin_file, index=pin_side)
            torch.cuda.synchronize()
            if i >= 2:
                e2e_times.append(time.perf_counter() - t0)
                e2e_phases.append(dict(container.LAST_UNPACK_MS))
        ok = bundle.tensors[0].qvalues.tobytes() == m.payload[: m.shapes[0][0] * m.shapes[0][1]].cpu().numpy().tobytes()
        if not ok:
            raise SystemExit("e2e mismatch")
        e2e_s = statistics.median(e2e_times)
        e2e = {"value": raw / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": len(host_file) + len(side),
               "d2h_bytes_per_step": raw + 8 * pm.jobs.n,
               "api": "container.unpack(pinned host file, index=pinned sidecar) -> host ModelBundle",
               "phases_ms": {k: statistics.median(p[k] for p in e2e_phases) for k in e2e_phases[0]}}
        del bundle
        # the reference's exact call, unpack(file) with no sidecar: every chunk is one
        # serial rANS chain on the GPU (no split points exist yet); one timed step
        if not args.no_index_less:
            container.clear_index_cache()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b2 = container.unpack(pin_file)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            same = b2.tensors[-1].qvalues.tobytes() == m.payload[-m.shapes[-1][0] * m.shapes[-1][1]:].cpu().numpy().tobytes()
            e2e["index_less"] = {"value": raw / dt / 1e9, "unit": "GB/s",
                                 "api": "container.unpack(pinned host file) -- no sidecar, first call", "seconds": dt,
                                 "equal": same}
            del b2
            container.clear_index_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            v, sample, cores = cpu_sample_decode(host_file, pm.entries, args.cpu_seconds, os.cpu_count() or 1)
            cpu = {"value": v, "unit": "GB/s", "cores": cores, "kind": "port",
                   "sample": "decode only (no CRC): " + sample}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    del host_file, pin_file, pin_side

    traffic, traffic_src, pipes = ncu_traffic("k_decode_segments", {"model": args.model,
                                                                   "chunk_size": args.chunk_size,
                                                                   "seg_shift": args.seg_shift, "layers": args.layers})
    n_tasks = int(pm.tasks.shape[0])
    n_chunks = int(pm.jobs.n)
    index_bytes = pm.index.nbytes
    file_bytes = pm.file_bytes
    launches_per_step = unp.launches
    shard_bytes = unp.raw_bytes
    del unp, out, m, pm
    torch.cuda.empty_cache()

    extra = None
    if args.extra_model != "none" and world == 1:
        try:
            m2, pm2, digest2, _ = build_packed(args, args.extra_model, dev)
            u2 = DeviceUnpack(pm2, dev)
            for _ in range(3):
                u2()
            torch.cuda.synchronize()
            if int(u2.bad.item()) != 0 or not torch.equal(u2.out, m2.payload):
                raise RuntimeError("extra-model unpack mismatch")
            ms2 = time_ms(lambda: u2(record=True), 20)
            extra = {"model": args.extra_model, "value": pm2.raw_bytes / (ms2 / 1e3) / 1e9, "unit": "GB/s",
                     "ms_per_step": ms2, "decode_kernel_ms": u2.kernel_ms(),
                     "decode_kernel_gbs": pm2.raw_bytes / (u2.kernel_ms() / 1e3) / 1e9,
                     "cr": pm2.raw_bytes / pm2.file_bytes, "container_digest": digest2,
                     "decode_step_tokens": decode_step_tokens(m2, pm2, u2.out, dev, 20)}
            del u2, m2, pm2
            torch.cuda.empty_cache()
        except Exception as e:  # report, never hide
            extra = {"model": args.extra_model, "error": repr(e)[:300]}

    if rank == 0:
        # `config` is exactly the reference arm's (same workload, same container
        # bytes); what only this arm has goes to `config_detail`
        cfg = workload_config(args, raw, file_bytes, digest)
        assert cfg["n_chunks"] == n_chunks, (cfg["n_chunks"], n_chunks)
        detail = {"seg_len": 1 << args.seg_shift, "n_tasks": n_tasks,
                  "cr_resident": raw / (file_bytes + index_bytes), "index_bytes": index_bytes,
                  "shard": {"chunks": [shard.c0, shard.c1], "decompressed_bytes": shard_bytes},
                  "build_s": t_build,
                  "reference_arm": "bench.py --impl reference builds the same container from the same spec "
                                   "(same container_digest) and unpacks whole-layer samples of it",
                  "parity": "the decoded output is checked equal to the encoder's input payload after the "
                            "warm-up, and every timed step checks every chunk's CRC32 against the container "
                            "table (verdicts re-checked after the timed region); the workload's container bytes equal "
                            "the oracle-packed container's (tests/test_bench_synth_gpu.py), whose codec is "
                            "pinned to the reference's golden vectors (tests/test_oracle_golden.py)"}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic", "config": cfg, "config_detail": detail,
            "decode_kernel_gbs": shard_bytes / (kms / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "k_decode_segments", "achieved": achieved, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "traffic_src": traffic_src, "alg_bytes_per_launch": alg_bytes, "launch_ms": kms,
                         "frac_decompressed": shard_bytes / (kms / 1e3) / 1e9 / hbm,
                         # the decode is bound by instruction issue on the ALU pipe, not HBM
                         # (same ncu capture): see DESIGN.md "Why the decode is not at the HBM roofline"
                         "ncu_pipes": pipes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "decode_step_tokens": tokens,
            "extra": extra,
            "tp_decode": tp,
            "streaming_tier": streaming_tier,
            "disk_tier": disk_tier,
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
