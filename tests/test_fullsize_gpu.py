"""Full-size checks at BASELINE.json's configurations through size-independent
properties (the CPU oracle cannot run these sizes in test time): round trips,
checksums of checksums against the container's own CRC table, sampled chunks
byte-equal to the oracle, exact integer GEMM equalities, prune idempotence."""

import zlib

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c3_opt27b_pack_decode_roundtrip(cuda, oracle):
    """C3: OPT-2.7B (2.5 GB) at 16 MiB chunks -- split-point decode returns the
    payload, every chunk's CRC equals the table's, two sampled chunks' blobs
    equal the oracle's encoding of the same bytes."""
    from paper_2502_15443_b200 import engine, synth
    m = synth.build_model("opt-2.7b")
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    res = engine.decode_jobs(pm.image, pm.jobs, pm.index, tasks=pm.tasks)
    assert (res.status == 0).all()
    assert torch.equal(res.out[: m.nbytes], m.payload)
    crc = engine.crc32_ranges(res.out, pm.jobs.d_out_off, pm.jobs.d_out_len, int(pm.jobs.out_len.max()))
    assert np.array_equal(crc.cpu().numpy().view(np.uint32), pm.entries["crc32"])
    image = pm.image.cpu().numpy()
    for c in (0, pm.jobs.n // 2):
        raw = m.payload[c * (16 << 20):(c + 1) * (16 << 20)].cpu().numpy()
        blob = image[int(pm.jobs.blob_off[c]): int(pm.jobs.blob_off[c] + pm.jobs.blob_len[c])].tobytes()
        assert blob == oracle.compress_blob(raw)
        assert zlib.crc32(raw) == int(pm.entries["crc32"][c])


def test_c4_opt67b_fused_equals_int8(cuda):
    """C4: OPT-6.7B (6.4 GB), fully compressed: the fused decode -> tcgen05 W8A8
    launch and the INT8 grouped GEMM give identical int32 outputs for every
    linear; the overlapped partially compressed step agrees with both."""
    from paper_2502_15443_b200 import synth
    from paper_2502_15443_b200.gemm import FusedRing, GroupedInt8
    m = synth.build_model("opt-6.7b")
    pm = synth.pack_model(m, 16 << 20, seg_shift=8)
    offs = m.offsets()[:-1]
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    xs = [torch.randint(-127, 128, (4, c), generator=g, device="cuda", dtype=torch.int8) for _, c in m.shapes]
    ws = [m.payload[o:o + r * c].view(torch.int8).view(r, c) for o, (r, c) in zip(offs, m.shapes)]
    gi = GroupedInt8(ws, xs, 4)
    gi.run()
    fr = FusedRing(pm.image, pm.jobs, pm.index, 16 << 20, m.shapes, offs, xs, 4)
    assert fr.run_checked()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(gi.accs, fr.accs))
    gi.run(max_ctas=100)  # persistent kernel on a capped grid
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(gi.accs, fr.accs))


def test_c5_shape_prune_idempotent_and_exact_count(cuda):
    """C5 (LLaMA-13B gate_proj shape, 70.8 M elements): per-tensor prune zeroes
    exactly floor(s * n) entries beyond the existing zeros' selection rule, a
    second prune at the same sparsity changes nothing, and per-row prune zeroes
    floor(s * cols) per row."""
    from paper_2502_15443_b200.pruning import prune_device
    g = torch.Generator(device="cuda")
    g.manual_seed(13)
    rows, cols, sp = 13824, 5120, 0.3
    q = torch.clamp(torch.round(torch.randn(rows, cols, generator=g, device="cuda") * 25), -127, 127).to(torch.int8)
    cm = torch.exp(torch.randn(cols, generator=g, device="cuda", dtype=torch.float64) - 1)
    once = prune_device(q, cm, sp)
    twice = prune_device(once, cm, sp)
    assert torch.equal(once, twice)
    k = int(np.floor(sp * rows * cols))
    assert int((once == 0).sum()) >= k and int(((once == 0) & (q != 0)).sum()) <= k
    pr = prune_device(q, cm, sp, per_row=True)
    kr = int(np.floor(sp * cols))
    newly = ((pr == 0) & (q != 0)).sum(dim=1)
    assert int(newly.max()) <= kr and int(((pr == 0).sum(dim=1) >= kr).all()) == 1
    assert torch.equal(prune_device(pr, cm, sp, per_row=True), pr)
