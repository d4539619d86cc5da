"""TP decode step on one GPU (NCCL world of 1): fused-compressed and INT8
paths give identical reduced outputs; timing harness runs."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_tp_step_world1(cuda):
    import torch.distributed as dist
    from paper_2502_15443_b200 import tp_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        st = tp_step.TPDecodeStep("llama-13b", 1, 0, ntok=4, layers=1)
        assert st.check()
        r = tp_step.measure(st, iters=3)
        assert r["allreduces_per_step"] == 2 and r["int8_step_ms"] > 0
    finally:
        dist.destroy_process_group()


def test_tp_step_cuda_graph_world1(cuda):
    """The TP step (grouped launch + row-parallel NCCL all-reduces) captured
    as one CUDA graph replays to the eager step's outputs."""
    import torch.distributed as dist
    from paper_2502_15443_b200 import tp_step
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        st = tp_step.TPDecodeStep("llama-13b", 1, 0, ntok=2, layers=2)
        for comp in (False, True):
            st.step(comp)
            torch.cuda.synchronize()
            want = [a.clone() for a in (st.fused if comp else st.int8).accs]
            g = st.graph(comp)
            for a in (st.fused if comp else st.int8).accs:
                a.fill_(7)
            g.replay()
            torch.cuda.synchronize()
            assert all(torch.equal(a, b) for a, b in zip(want, (st.fused if comp else st.int8).accs))
        r = tp_step.measure(st, iters=3)
        assert r["int8_graph_step_ms"] > 0 and r["compressed_fused_graph_step_ms"] > 0
    finally:
        dist.destroy_process_group()
