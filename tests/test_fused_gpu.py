"""Grouped INT8 GEMM and the fused decode -> TMEM -> tcgen05 GEMM: exact
int32 accumulators vs an int64 CPU product of the same weights."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(256, 512), (384, 1024), (130, 512), (1000, 1536)]


def _weights(seed=0):
    g = torch.Generator().manual_seed(seed)
    ws = []
    for r, k in SHAPES:
        w = torch.round(torch.randn(r, k, generator=g) * 9).clamp_(-127, 127).to(torch.int8)
        w[:, :17] = 0
        ws.append(w)
    return ws


def _xs(ntok, seed=1):
    g = torch.Generator().manual_seed(seed)
    return [torch.randint(-127, 128, (ntok, k), generator=g, dtype=torch.int8) for _, k in SHAPES]


@pytest.mark.parametrize("ntok", [1, 5, 16])
def test_grouped_int8_exact(cuda, ntok):
    from paper_2502_15443_b200.gemm import GroupedInt8
    ws, xs = _weights(), _xs(ntok)
    gi = GroupedInt8([w.cuda() for w in ws], [x.cuda() for x in xs], ntok)
    for max_ctas in (None, 0, 1, 3, 64):  # wave kernel, persistent (all SMs / capped grids)
        gi.run(max_ctas)
        for w, x, acc in zip(ws, xs, gi.accs):
            assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)


def test_persistent_int8_split_k_exact(cuda):
    """Long-K layers are split into equal K-slices for the persistent kernel's
    round-robin (atomics accumulate the slices exactly)."""
    from paper_2502_15443_b200.gemm import GroupedInt8
    g = torch.Generator().manual_seed(3)
    shapes = [(512, 16384), (640, 12288), (256, 4096)]
    ws = [torch.randint(-127, 128, s, generator=g, dtype=torch.int8) for s in shapes]
    xs = [torch.randint(-127, 128, (2, k), generator=g, dtype=torch.int8) for _, k in shapes]
    gi = GroupedInt8([w.cuda() for w in ws], [x.cuda() for x in xs], 2)
    assert int(gi.unit_p[:, 3].max()) == 4096 and gi.unit_p.shape[0] > gi.unit_t.shape[0]
    gi.run(max_ctas=0)
    for w, x, acc in zip(ws, xs, gi.accs):
        assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)


@pytest.mark.parametrize("ntok,stored,chunk", [(1, False, 1 << 22), (5, True, 1 << 22), (16, False, 1 << 24)])
def test_fused_ring_exact(cuda, ntok, stored, chunk):
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(ntok)
    shapes = [(1024, 2048), (1500, 512), (300, 4096), (2048, 1280)]
    ws = []
    for r, k in shapes:
        w = torch.round(torch.randn(r, k, generator=g) * 9).clamp_(-127, 127).to(torch.int8)
        w[:, :33] = 0
        ws.append(w)
    xs = [torch.randint(-127, 128, (ntok, k), generator=g, dtype=torch.int8) for _, k in shapes]
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    n = -(-payload.numel() // chunk)
    plan = np.array([i % 2 == 0 for i in range(n)]) if stored else None
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, plan, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, shapes, t_offs, [x.cuda() for x in xs], ntok)
    fr.run()
    torch.cuda.synchronize()
    assert (fr.check() == 0).all()
    for w, x, acc in zip(ws, xs, fr.accs):
        assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)
    fr.run()  # re-run (ring / barrier phases carry over between launches)
    torch.cuda.synchronize()
    assert all(torch.equal(acc.cpu().long(), x.long() @ w.long().T) for w, x, acc in zip(ws, xs, fr.accs))


def test_fused_ring_skewed_streams(cuda):
    """Edge distributions: ~99.8% zeros (symbols that consume no stream byte
    for many steps), an all-zero tensor (single-symbol table, empty stream)
    and uniform bytes (incompressible -> stored chunk), in one launch."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(5)
    dense = torch.randint(-128, 128, (2048, 2048), generator=g, dtype=torch.int8)  # 8 bits/byte: stored
    sparse = torch.where(torch.rand(1024, 2048, generator=g) < 0.002, dense[:1024], torch.zeros_like(dense[:1024]))
    ws = [sparse, torch.zeros(1024, 2048, dtype=torch.int8), dense, torch.zeros(2048, 2048, dtype=torch.int8),
          sparse[:, :1024].contiguous()]
    shapes = [tuple(w.shape) for w in ws]
    ntok = 3
    xs = [torch.randint(-127, 128, (ntok, k), generator=g, dtype=torch.int8) for _, k in shapes]
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    chunk = 1 << 22
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    assert list(entries["codec"]) == [1, 0, 1, 1]  # ANS, stored (dense), single-symbol ANS, ANS
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, shapes, t_offs, [x.cuda() for x in xs], ntok)
    fr.run()
    torch.cuda.synchronize()
    assert (fr.check() == 0).all()
    for w, x, acc in zip(ws, xs, fr.accs):
        assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)


def test_fused_ring_checked_fallback(cuda):
    """A corrupted split point never yields a wrong product: run_checked()
    detects the broken chain and recomputes exactly."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(9)
    shapes = [(1024, 1024), (2048, 512)]
    ws = [torch.round(torch.randn(r, k, generator=g) * 9).clamp_(-127, 127).to(torch.int8) for r, k in shapes]
    xs = [torch.randint(-127, 128, (2, k), generator=g, dtype=torch.int8) for _, k in shapes]
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    chunk = 1 << 21
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, shapes, t_offs, [x.cuda() for x in xs], 2)
    assert fr.run_checked()
    enc.index.d_state[40] ^= 0x5A5A  # corrupt one split point
    assert not fr.run_checked()
    for w, x, acc in zip(ws, xs, fr.accs):
        assert torch.equal(acc.cpu().long(), x.long() @ w.long().T)


def test_fused_ring_dequant_epilogue(cuda):
    """decompress -> dequant -> W8A8 in one launch: fp32 outputs y = acc * (sx*sw)
    equal the exact int32 product scaled in fp32, and match the f64 W8A8 value
    within rtol 1e-6 (scaling.py:127-152 numerics)."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(11)
    shapes = [(2048, 1024), (1024, 4096)]  # several K-slices and row blocks per layer
    ws = [torch.round(torch.randn(r, k, generator=g) * 20).clamp_(-127, 127).to(torch.int8) for r, k in shapes]
    xs = [torch.randint(-127, 128, (4, k), generator=g, dtype=torch.int8) for _, k in shapes]
    scales = [3.1e-4, 7.7e-5]
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    chunk = 1 << 23
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, shapes, t_offs, [x.cuda() for x in xs], 4, scales=scales)
    for _ in range(2):  # counters reset between launches
        assert fr.run_checked()
        for w, x, acc, y, sc in zip(ws, xs, fr.accs, fr.ys, scales):
            exact = x.long() @ w.long().T
            assert torch.equal(acc.cpu().long(), exact)
            assert torch.equal(y.cpu(), exact.to(torch.float32) * np.float32(sc))
            ref = exact.to(torch.float64) * sc
            assert torch.allclose(y.cpu().double(), ref, rtol=1e-6, atol=0)


@pytest.mark.parametrize("fused_ctas", [0, 40, 100])
def test_mixed_step_overlapped_exact(cuda, fused_ctas):
    """Partially compressed step: fused (compressed) and INT8 (plain) layers on
    two streams with the fused grid capped -- results equal the exact product."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing, GroupedInt8, MixedStep
    g = torch.Generator().manual_seed(21)
    shapes = [(2048, 2048), (4096, 1024), (1024, 4096), (3000, 2048)]
    ws = [torch.round(torch.randn(r, k, generator=g) * 15).clamp_(-127, 127).to(torch.int8) for r, k in shapes]
    xs = [torch.randint(-127, 128, (3, k), generator=g, dtype=torch.int8).cuda() for _, k in shapes]
    comp, plain = [0, 2], [1, 3]
    payload = torch.cat([ws[i].reshape(-1).view(torch.uint8) for i in comp]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([ws[i].numel() for i in comp])[:-1]])
    chunk = 1 << 22
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, [shapes[i] for i in comp], t_offs, [xs[i] for i in comp], 3)
    gi = GroupedInt8([ws[i].cuda() for i in plain], [xs[i] for i in plain], 3)
    mx = MixedStep(fr, gi, fused_ctas)
    for _ in range(2):
        mx.run()
        torch.cuda.synchronize()
        assert (fr.check() == 0).all()
        for i, acc in zip(comp + plain, fr.accs + gi.accs):
            assert torch.equal(acc.cpu().long(), xs[i].cpu().long() @ ws[i].long().T)
    times = mx.tune(candidates=[30, 148], iters=2)
    assert set(times) == {30, 148} and mx.fused_ctas in times


def test_fused_ring_merges_shared_input_layers(cuda):
    """q/k/v-style layers (same activations, back to back in the payload) are
    decoded as one taller matrix; per-layer accumulators stay exact views."""
    from paper_2502_15443_b200 import container
    from paper_2502_15443_b200.gemm import FusedRing
    g = torch.Generator().manual_seed(8)
    shapes = [(640, 1024), (640, 1024), (640, 1024), (1024, 2048), (384, 2048)]
    ws = [torch.round(torch.randn(r, k, generator=g) * 12).clamp_(-127, 127).to(torch.int8) for r, k in shapes]
    x_attn = torch.randint(-127, 128, (2, 1024), generator=g, dtype=torch.int8).cuda()
    x_other = torch.randint(-127, 128, (2, 2048), generator=g, dtype=torch.int8).cuda()
    xs = [x_attn, x_attn, x_attn, x_other, x_other.clone()]  # last: equal values, different tensor
    payload = torch.cat([w.reshape(-1).view(torch.uint8) for w in ws]).cuda()
    t_offs = np.concatenate([[0], np.cumsum([w.numel() for w in ws])[:-1]])
    chunk = 1 << 22
    image, enc, entries = container.pack_device(payload, b"\x00" * 8, chunk, None, seg_shift=8)
    jobs = container.jobs_for(entries, image.device)
    fr = FusedRing(image, jobs, enc.index, chunk, shapes, t_offs, xs, 2)
    assert fr.merged_layers == 2 and len(fr.accs) == len(shapes)
    assert fr.run_checked()
    for w, x, acc in zip(ws, xs, fr.accs):
        assert acc.shape == (2, w.shape[0])
        assert torch.equal(acc.cpu().long(), x.cpu().long() @ w.long().T)
