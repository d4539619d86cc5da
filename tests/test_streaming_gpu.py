"""GPU_CPU tier: weights streamed from pinned host memory every step, raw vs
compressed, decoded weights and GEMM outputs identical."""

import pytest

pytestmark = pytest.mark.gpu


def test_streamed_raw_vs_compressed(cuda):
    from paper_2502_15443_b200 import streaming, synth
    m = synth.build_model("opt-125m", layers=2)
    pm = synth.pack_model(m, 1 << 20, seg_shift=8)
    r = streaming.measure(m.payload, m.shapes, m.offsets()[:-1], pm.image, pm.jobs, pm.index, ntok=2, iters=1,
                          groups=4)
    assert r["outputs_equal"]
    assert r["compressed_h2d_bytes"] < r["raw_h2d_bytes"]
