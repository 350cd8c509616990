"""Row sharding of packed layers across the GPUs of one node.

The SparseGemv shards by output rows: every row's K-reduction is local, so a
shard needs no partial-sum exchange and the per-row accumulation order is the
single-GPU order.  The one exchange step is an all-gather of the y slices
(rows/G x 4 B per rank) -- NCCL over NVLink on the B200 node, gloo in the
CPU tests.  Shards are 16-row aligned (the fragment tile) and zero-copy
(`DeviceMatrix.slice_rows`).  Small layers and independent request streams are
replicated instead (bench.py --gpus N runs N replicas of the layer sweep).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

TILE_ROWS = 16


@dataclass(frozen=True)
class RowShardPlan:
    rows: int
    world: int
    bounds: tuple  # (r0, r1) per rank, contiguous, 16-row aligned except the end

    @staticmethod
    def make(rows: int, world: int, align: int = TILE_ROWS) -> "RowShardPlan":
        if world < 1:
            raise ValueError("shard plan: world size must be positive")
        tiles = (rows + align - 1) // align
        base, extra = divmod(tiles, world)
        bounds, t0 = [], 0
        for r in range(world):
            t1 = t0 + base + (1 if r < extra else 0)
            bounds.append((min(rows, t0 * align), min(rows, t1 * align)))
            t0 = t1
        return RowShardPlan(rows, world, tuple(bounds))

    @property
    def max_rows(self) -> int:
        return max(r1 - r0 for r0, r1 in self.bounds)

    def local(self, rank: int) -> tuple:
        return self.bounds[rank]


def gather_rows(y_local: torch.Tensor, plan: RowShardPlan, group=None) -> torch.Tensor:
    """All-gather the per-rank y slices ([M x rows_local] or [rows_local]) into
    the full [M x rows] output.  Slices are padded to the largest shard so the
    collective is one all_gather_into_tensor."""
    rank = dist.get_rank(group)
    r0, r1 = plan.local(rank)
    one_d = y_local.dim() == 1
    y2 = y_local.reshape(1, -1) if one_d else y_local
    M = y2.shape[0]
    pad = torch.zeros((M, plan.max_rows), dtype=y2.dtype, device=y2.device)
    pad[:, : r1 - r0] = y2
    buf = torch.empty((plan.world * M, plan.max_rows), dtype=y2.dtype, device=y2.device)
    dist.all_gather_into_tensor(buf, pad.contiguous(), group=group)
    buf = buf.view(plan.world, M, plan.max_rows)
    out = torch.empty((M, plan.rows), dtype=y2.dtype, device=y2.device)
    for r, (a, b) in enumerate(plan.bounds):
        out[:, a:b] = buf[r, :, : b - a]
    return out.reshape(-1) if one_d else out


class ShardedSpmv:
    """y = W x with W's rows split across the ranks of `group`: local
    SparseGemv on this rank's zero-copy shard, then one all-gather."""

    def __init__(self, full, group=None):
        self.group = group
        self.plan = RowShardPlan.make(full.rows, dist.get_world_size(group))
        r0, r1 = self.plan.local(dist.get_rank(group))
        self.local = full.slice_rows(r0, r1)
        self.cols = full.cols

    def __call__(self, x: torch.Tensor, stream=None) -> torch.Tensor:
        y_local = self.local.spmv(x, stream)
        return gather_rows(y_local, self.plan, self.group)
