"""Multi-GPU layouts for the compressed-weight path (one process per GPU).

Chunk sharding (config C3): DCC1 chunks are independent streams
(reference container.py:20-21), so model-wide decompression shards by
contiguous chunk ranges with no data-path collective (weak scaling).

Tensor parallelism (config C5): Megatron-style split of each transformer
layer.  Column-parallel linears (q/k/v, gate/up, fc1) shard output rows;
row-parallel linears (o/down, out_proj/fc2) shard K.  K shards are cut on
512-byte boundaries (the fused kernel's K-slice) so every rank's shard is
decodable by the fused decode-GEMM; the int32 partial accumulators of
row-parallel layers are summed with one all-reduce per layer output -- exact,
because W8A8 products are integers.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from .tensors import MODEL_SHAPES, model_layout

ROW_PARALLEL = ("out_proj", "fc2", "o_proj", "down_proj")
K_ALIGN = 256


def shard_ranges(weights, world: int) -> list[tuple[int, int]]:
    """Contiguous [start, end) chunk ranges, one per rank, balancing the sum
    of ``weights`` (e.g. uncompressed chunk bytes = decode work)."""
    w = np.asarray(weights, dtype=np.float64)
    n = len(w)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        cuts.append(int(np.clip(np.searchsorted(cum, target), cuts[-1], n)))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def _split(n: int, world: int, align: int = 1) -> list[tuple[int, int]]:
    """Split [0, n) into `world` contiguous parts on multiples of `align`."""
    units = -(-n // align)
    out, pos = [], 0
    for r in range(world):
        take = units // world + (1 if r < units % world else 0)
        end = min(n, (pos // align + take) * align) if r < world - 1 else n
        out.append((pos, end))
        pos = end
    return out


@dataclasses.dataclass(frozen=True)
class TPShard:
    name: str
    kind: str              # "col" (shard rows) or "row" (shard K)
    rows: int              # global shape
    cols: int
    r0: int                # local slice
    r1: int
    c0: int
    c1: int

    @property
    def local_shape(self) -> tuple[int, int]:
        return self.r1 - self.r0, self.c1 - self.c0


def tp_layout(model: str, world: int, rank: int, layers: int | None = None) -> list[TPShard]:
    """This rank's slice of every linear of ``model`` under TP-``world``."""
    lay = model_layout(model)
    if layers is not None:
        per = sum(1 for n, _, _ in lay if n.startswith("layers.0."))
        lay = lay[: per * layers]
    out = []
    for name, r, c in lay:
        if name.rsplit(".", 1)[-1] in ROW_PARALLEL:
            c0, c1 = _split(c, world, K_ALIGN)[rank]
            out.append(TPShard(name, "row", r, c, 0, r, c0, c1))
        else:
            r0, r1 = _split(r, world)[rank]
            out.append(TPShard(name, "col", r, c, r0, r1, 0, c))
    return out


def allreduce_partials(accs: list[torch.Tensor], group=None) -> None:
    """Sum row-parallel int32 partial accumulators across ranks (exact)."""
    import torch.distributed as dist
    for a in accs:
        dist.all_reduce(a, op=dist.ReduceOp.SUM, group=group)


def hidden_size(model: str) -> int:
    return MODEL_SHAPES[model][0]
