"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, split_concat


def test_normalize_matches_reference(oracle, codec_golden):
    for h, want in zip(codec_golden["hist"], codec_golden["normed"]):
        assert np.array_equal(oracle.normalize(h), want)


def test_blobs_match_reference(oracle, codec_golden):
    datas = split_concat(codec_golden["data"], codec_golden["data_len"])
    blobs = split_concat(codec_golden["blob"], codec_golden["blob_len"])
    for d, b, f in zip(datas, blobs, codec_golden["freq"]):
        assert np.array_equal(oracle.table_for(d), f)
        assert oracle.compress_blob(d) == b.tobytes()
        assert oracle.decompress_blob(b.tobytes(), d.size) == d.tobytes()
        assert np.array_equal(oracle.unpack_table(b[:384].tobytes()), f)


def test_corrupt_verdicts_match_reference(oracle, golden):
    for case in golden["corrupt"]["cases"]:
        blob = bytes.fromhex(case["blob_hex"])
        v = case["verdict"]
        try:
            out = oracle.decompress_blob(blob, case["out_len"])
            got = {"ok": True, "sha": hashlib.sha256(out).hexdigest()}
        except oracle.OracleError as e:
            got = {"ok": False, "cls": e.kind, "msg": e.msg}
        assert got == v, case["kind"]


def test_crc_matches_zlib(oracle):
    import zlib
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 1000, 4096, 100_003):
        d = rng.integers(0, 256, n).astype(np.uint8)
        assert oracle.crc32(d) == zlib.crc32(d.tobytes())


@pytest.mark.parametrize("name", ["small_bs0", "small_bs1", "small_bs2", "small_bs5", "small_short"])
def test_container_roundtrip_matches_reference(oracle, golden, name):
    with open(f"{GOLDEN}/{name}.dcc", "rb") as f:
        data = f.read()
    assert hashlib.sha256(data).hexdigest() == golden["containers"][name]["sha"]
    ents = oracle.unpack(data)
    cs, directory, entries = oracle.parse(data)
    mask = np.array([e[0] == 1 for e in entries])
    if name == "small_bs0":
        mask[:] = False  # plan=block 0 -> all store
    # re-pack with the reference's plan semantics: a masked chunk may still be stored
    plan_mask = {"small_bs0": 0, "small_bs1": 1, "small_bs2": 2, "small_bs5": 5, "small_short": 1}[name]
    full_mask = oracle.block_mask(len(entries), plan_mask)
    again = oracle.pack([(n, q, ws, a, s, cm) for (n, q, ws, a, s, cm) in ents], cs, full_mask)
    assert again == data


def test_empty_container(oracle, golden):
    data = bytes.fromhex(golden["containers"]["empty"]["hex"])
    assert oracle.pack([], 16 * 2**20) == data
    assert oracle.unpack(data) == []


def test_quantize_matches_reference(oracle, golden):
    for c in golden["transforms"]["quantize"]:
        w = np.array(c["w"], dtype=np.float64)
        if "cm" in c:
            s = oracle.compute_scale(np.array(c["cm"]), c["alpha"])
            assert np.array_equal(s, np.array(c["s"]))
        else:
            s = None
        q, ws = oracle.quantize(w, s)
        assert np.array_equal(q, np.array(c["q"], dtype=np.int8))
        assert ws.hex() == c["w_scale"]


def test_prune_matches_reference(oracle, golden):
    for c in golden["transforms"]["prune"]:
        q = np.array(c["q"], dtype=np.int8)
        out = oracle.prune(q, np.array(c["cm"]), c["sparsity"], c["per_row"])
        assert np.array_equal(out, np.array(c["out"], dtype=np.int8))


def test_planner_latency_matches_reference(oracle, golden):
    for c in golden["planner"]["cases"]:
        p = c["profile"]
        arch = c["arch"]
        if arch in ("gpu_only", "gpu_buffer"):
            B = p["B_gpu"]
        elif arch == "gpu_cpu":
            B = min(p["B_ctog"], p["B_gpu"])
        else:
            B = min(p["B_stoc"], p["B_ctog"], p["B_gpu"])
        mask = oracle.block_mask(c["n"], c["bs"])
        lat = oracle.latency_seconds(B, p["D_max"], p["c_sat"], p["I_gpu"], c["cs"], mask,
                                     np.where(mask, c["cr"], 1.0))
        assert lat == pytest.approx(c["latency"], rel=1e-12)


def test_u12_wire(oracle):
    rng = np.random.default_rng(3)
    f = rng.integers(0, 4095, 256).astype(np.uint32)
    packed = oracle.pack_u12(f)
    assert len(packed) == 384
    raw = np.frombuffer(packed, np.uint8).astype(np.uint32)
    back = np.empty(256, np.uint32)
    back[0::2] = raw[0::3] | ((raw[1::3] & 0xF) << 8)
    back[1::2] = (raw[1::3] >> 4) | (raw[2::3] << 4)
    assert np.array_equal(back, f)
