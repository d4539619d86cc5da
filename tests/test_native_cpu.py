"""CPU-only checks: the C-ABI library loads and exports every symbol that
include/dcomp_b200.h declares; host-side format logic (no GPU calls)."""

import os
import re
import struct

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

import paper_2502_15443_b200 as dc
from paper_2502_15443_b200 import container, engine, native


def header_symbols():
    with open(os.path.join(ROOT, "include", "dcomp_b200.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(dc_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = native.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(native.SIGNATURES), set(syms) ^ set(native.SIGNATURES)
    assert lib.dc_version() == 1


def test_library_is_sm100a():
    """The shared object carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([tool, "--list-elf", native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", ["small_bs0", "small_bs1", "small_bs2", "small_bs5", "small_short"])
def test_inspect_matches_oracle_parse(oracle, name):
    data = open(f"{GOLDEN}/{name}.dcc", "rb").read()
    info = container.inspect(data)
    cs, directory, entries = oracle.parse(data)
    assert info.chunk_size == cs
    assert [tuple(e) for e in entries] == [(c.codec, c.file_offset, c.comp_len, c.uncomp_len, c.crc32)
                                           for c in info.chunks]
    assert [d[:5] for d in directory] == info.directory


def _mutants(data, rng, count):
    for _ in range(count):
        kind = rng.integers(0, 3)
        b = bytearray(data)
        if kind == 0:
            pos = int(rng.integers(0, len(b)))
            b[pos] ^= 1 << int(rng.integers(0, 8))
            yield bytes(b)
        elif kind == 1:
            yield bytes(b[: int(rng.integers(0, len(b)))])
        else:
            yield bytes(b) + bytes(rng.integers(0, 256, int(rng.integers(1, 9))).astype(np.uint8))


def test_structural_errors_match_reference_parser(oracle):
    """Host-side parse: every structural mutation is rejected with a
    DataFormatError subclass (the payload-level ones need the GPU)."""
    data = open(f"{GOLDEN}/small_bs1.dcc", "rb").read()
    rng = np.random.default_rng(7)
    for m in _mutants(data, rng, 400):
        try:
            container.inspect(m)
        except dc.DataFormatError:
            continue
        # inspect accepted it: only payload bytes changed (decode / CRC catch those)
        cs, directory, entries = oracle.parse(m)
        assert len(m) == len(data)


def test_bad_magic_version_and_header_crc():
    data = bytearray(open(f"{GOLDEN}/small_bs2.dcc", "rb").read())
    with pytest.raises(dc.BadMagicError):
        container.inspect(b"XXXX" + bytes(data[4:]))
    v = bytearray(data)
    v[4:6] = struct.pack("<H", 2)
    with pytest.raises(dc.UnsupportedVersionError):
        container.inspect(bytes(v))
    h = bytearray(data)
    h[20] ^= 0xFF
    with pytest.raises(dc.ChecksumError) as ei:
        container.inspect(bytes(h))
    assert ei.value.chunk_index == -1
    with pytest.raises(dc.TruncatedError):
        container.inspect(bytes(data[:3]))


def test_segment_layout_and_sidecar_binding():
    ent = container._parse(open(f"{GOLDEN}/small_bs2.dcc", "rb").read())[2]
    base, n = engine.SegmentIndex.layout(ent["uncomp_len"].astype(np.uint64), ent["codec"], 9)
    want = sum(-(-int(e["uncomp_len"]) // 512) for e in ent if e["codec"] == 1)
    assert n == want
    assert base[0] == 0 and np.all(np.diff(base) >= 0)


def test_planner_matches_reference_golden(golden):
    import importlib
    L = importlib.import_module("paper_2502_15443_b200.latency")
    for c in golden["planner"]["cases"]:
        h = L.HardwareProfile.from_json(__import__("json").dumps(c["profile"]))
        plan = L.CompressionPlan.block_plan(c["cs"], c["n"], c["bs"])
        arch = L.Architecture(c["arch"])
        rep = L.latency(h, plan, arch, np.where(plan.compressed_mask, c["cr"], 1.0))
        assert rep.per_sample_latency == pytest.approx(c["latency"], rel=1e-12)
        assert rep.bottleneck.value == c["bottleneck"]
        assert rep.memory_used_gpu == pytest.approx(c["mem_gpu"], rel=1e-12)
        assert rep.memory_used_cpu == pytest.approx(c["mem_cpu"], rel=1e-12, abs=1e-9)
        pr = L.plan_partial(h, c["n"], c["cs"], c["cr"], c["budget"], arch)
        assert pr.plan.block_size == c["plan_bs"] and pr.feasible == c["feasible"]
        assert L.memory_footprint(plan, np.where(plan.compressed_mask, c["cr"], 1.0)) == pytest.approx(
            c["footprint"], rel=1e-12)
    d, cs = L.fit_speed_curve([(48.05e6, 97.76), (75.08e6, 109.64), (192.13e6, 144.01), (300.16e6, 156.08)])
    assert d == pytest.approx(golden["planner"]["fit_paper"][0], rel=1e-6)
    assert cs == pytest.approx(golden["planner"]["fit_paper"][1], rel=1e-2)


def test_block_plan_rules():
    import importlib
    L = importlib.import_module("paper_2502_15443_b200.latency")
    assert L.CompressionPlan.block_plan(4096, 10, 3).compressed_mask.tolist() == [
        False, False, True, False, False, True, False, False, True, False]
    assert L.CompressionPlan.block_plan(4096, 5, 1).compressed_mask.all()
    assert not L.CompressionPlan.block_plan(4096, 5, 0).compressed_mask.any()
    with pytest.raises(dc.DcompError):
        L.CompressionPlan.block_plan(4096, 5, 6)


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.NativeUnavailable):
        dc.compress_blob(b"abc")


def test_choose_architecture_reference_cases():
    """latency.py:234-241 with the reference's own cases (test_latency.py:183-197):
    tiers by capacity, monotone in GPU memory."""
    def profile(mem_gpu=48e9, mem_cpu=64e9):
        return dc.HardwareProfile(B_stoc=7.0, B_ctog=32.0, B_gpu=696.0, D_max=156.08, c_sat=76.72e6,
                                  I_gpu=300.0, mem_gpu=mem_gpu, mem_cpu=mem_cpu)
    A = dc.Architecture
    p = profile()
    assert dc.choose_architecture(p, 4e9, 1e9) is A.GPU_BUFFER
    assert dc.choose_architecture(p, 60e9, 1e9) is A.GPU_CPU
    assert dc.choose_architecture(p, 200e9, 1e9) is A.STORAGE
    order = [A.GPU_BUFFER, A.GPU_CPU, A.STORAGE]
    prev = len(order)
    for mem in (1e9, 10e9, 50e9, 70e9, 300e9):
        rank = order.index(dc.choose_architecture(profile(mem_gpu=mem), 60e9, 1e9))
        assert rank <= prev
        prev = rank
    # boundary: exactly full fits (<=), one byte more spills to the next tier
    assert dc.choose_architecture(profile(mem_gpu=10.0), 6.0, 4.0) is A.GPU_BUFFER
    assert dc.choose_architecture(profile(mem_gpu=10.0, mem_cpu=5.0), 6.0, 5.0) is A.GPU_CPU
    assert dc.choose_architecture(profile(mem_gpu=10.0, mem_cpu=5.0), 11.0, 5.0) is A.STORAGE


def test_host_to_bytes_parallel_fill():
    """pack's result: a bytes object filled in place by parallel slice copies
    (above 64 MiB) equals numpy's tobytes, hashes and compares like any bytes,
    and small inputs take the plain path."""
    import numpy as np

    from paper_2502_15443_b200 import native as nv
    assert nv._BYTES_OFF is not None
    for n in (0, 1000, (64 << 20) + 12345):
        a = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
        b = nv.host_to_bytes(a)
        assert type(b) is bytes and len(b) == n
        assert b == a.tobytes() and hash(b) == hash(a.tobytes())
