"""GPU_CPU tier: weights streamed from pinned host memory every step, raw vs
compressed, decoded weights and GEMM outputs identical."""

import pytest

pytestmark = pytest.mark.gpu


def test_streamed_raw_vs_compressed(cuda):
    from paper_2502_15443_b200 import streaming, synth
    m = synth.build_model("opt-125m", layers=2)
    pm = synth.pack_model(m, 4 << 20, seg_shift=8)
    r = streaming.measure(m.payload, m.shapes, m.offsets()[:-1], pm.image, pm.jobs, pm.index, ntok=2, iters=1,
                          groups=4)
    assert r["outputs_equal"]
    assert r["compressed_h2d_bytes"] < r["raw_h2d_bytes"]
    assert r["fused_bounded_outputs_equal"], r.get("fused_bounded")
    assert r["fused_bounded_groups"] >= 1


def test_streamed_fused_bounded_ring(cuda):
    """Many small layer groups through 2 device slots (every slot reused within
    a step), two steps: fused outputs equal the exact INT8 product."""
    import numpy as np
    import torch
    from paper_2502_15443_b200 import streaming, synth
    m = synth.build_model("opt-125m", layers=3)
    pm = synth.pack_model(m, 4 << 20, seg_shift=8)
    host = torch.empty(pm.image.numel(), dtype=torch.uint8, pin_memory=True)
    host.copy_(pm.image)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    xs = [torch.randint(-127, 128, (3, c), generator=g, device="cuda", dtype=torch.int8) for _, c in m.shapes]
    offs = m.offsets()[:-1]
    sf = streaming.StreamedFused(host, pm.jobs, pm.index, 4 << 20, m.shapes, offs, xs, 3, slots=2,
                                 group_bytes=1 << 20)
    assert len(sf.groups) >= 6 and sf.ring.numel() == 2 * sf.slot_bytes
    for _ in range(2):
        sf.step()
        torch.cuda.synchronize()
        assert sf.check()
        for (r, c), o, x, acc in zip(m.shapes, offs, xs, sf.accs):
            w = m.payload[o:o + r * c].view(torch.int8).view(r, c).cpu().long()
            assert torch.equal(acc.cpu().long(), x.cpu().long() @ w.T)
    assert isinstance(sf.bytes_per_step, int) and np.isfinite(sf.device_bytes)


def test_disk_tier_fused_equals_int8(cuda, tmp_path):
    """GPU_DISK tier: raw INT8 file and DCC1 image file read every step
    (O_DIRECT where the filesystem allows) -- fused outputs equal the INT8 GEMM's."""
    from paper_2502_15443_b200 import streaming, synth
    m = synth.build_model("opt-125m", layers=2)
    pm = synth.pack_model(m, 4 << 20, seg_shift=8)
    r = streaming.measure_disk(m.payload, m.shapes, m.offsets()[:-1], pm.image, pm.jobs, pm.index, ntok=2,
                               iters=1, workdir=str(tmp_path))
    assert r["outputs_equal"]
    assert r["compressed_read_bytes"] < r["raw_read_bytes"]
