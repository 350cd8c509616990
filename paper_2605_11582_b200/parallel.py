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


# ------------------------------------------------ fused all-gather over NVLink
# The product kernel stores each y row straight into every rank's buffer
# (CUDA IPC mappings of the peers' HBM over NVLink) and exchanges arrival
# counters from its last CTA, so "spmv + all-gather" is one kernel with no
# NCCL call (include/egt_b200.h, egt_spmv_allgather).

class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (zero-copy for torch.as_tensor)."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def exchange_handles(handle: bytes, group=None) -> list:
    """Every rank's 64-byte IPC handle, in rank order (all_gather_object:
    works over NCCL and gloo)."""
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return out


class PeerBuffer:
    """One rank's [control block | y] buffer: allocated here (owner, with an
    IPC handle to export) or opened from a peer's handle."""

    def __init__(self, y_floats: int = 0, handle: bytes | None = None):
        import ctypes as C

        from .native import IpcHandle, check, lib

        self._lib = lib()
        self.ptr = C.c_void_p()
        if handle is None:
            h = IpcHandle()
            check(self._lib.egt_peer_buffer_alloc(y_floats, C.byref(self.ptr), C.byref(h)))
            self.handle = bytes(h.bytes)
            self.owner = True
        else:
            h = IpcHandle()
            C.memmove(h.bytes, handle, 64)
            check(self._lib.egt_peer_buffer_open(C.byref(h), C.byref(self.ptr)))
            self.handle = bytes(handle)
            self.owner = False

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            (self._lib.egt_peer_buffer_free if self.owner else self._lib.egt_peer_buffer_close)(self.ptr)
            self.ptr = None


class PeerGroup:
    """All ranks' buffers in rank order, seen from `rank`."""

    def __init__(self, bufs: list, rank: int):
        import ctypes as C

        from .native import check, lib

        self._lib = lib()
        self.bufs = bufs  # keep the buffers alive
        self.world, self.rank = len(bufs), rank
        arr = (C.c_void_p * self.world)(*[b.ptr for b in bufs])
        self._g = C.c_void_p()
        check(self._lib.egt_peer_group_create(self.world, rank, arr, C.byref(self._g)))

    @staticmethod
    def local_ranks(world: int, y_floats: int) -> list:
        """`world` groups over buffers on the CURRENT device (ranks sharing one
        GPU: tests and single-GPU runs); call with EGT_PEER_NOWAIT + wait()."""
        bufs = [PeerBuffer(y_floats) for _ in range(world)]
        return [PeerGroup(bufs, r) for r in range(world)]

    def y(self, shape: tuple):
        import torch

        ptr = self._lib.egt_peer_group_y(self._g)
        return torch.as_tensor(_CudaArray(ptr, tuple(shape)), device="cuda")

    def spmv(self, shard, x, row0: int, ldy: int, stream=None, nowait: bool = False,
             independent: bool = False) -> None:
        from .native import PEER_NOWAIT, check
        from .packed import _stream_ptr

        M = 1 if x.dim() == 1 else x.shape[0]
        ldx = x.shape[-1] if x.dim() == 2 else shard.cols
        flags = (PEER_NOWAIT if nowait else 0) | (1 if independent else 0)
        check(self._lib.egt_spmv_allgather(shard.handle, C_ptr(x), M, ldx, self._g, row0, ldy, flags,
                                           _stream_ptr(stream)))

    def wait(self, stream=None) -> None:
        from .native import check
        from .packed import _stream_ptr

        check(self._lib.egt_peer_wait(self._g, _stream_ptr(stream)))

    def check(self) -> None:
        from .native import check

        check(self._lib.egt_peer_group_check(self._g))

    def __del__(self):
        if getattr(self, "_g", None) is not None and self._g.value:
            self._lib.egt_peer_group_destroy(self._g)
            self._g = None


def C_ptr(t):
    import ctypes as C

    return C.c_void_p(t.data_ptr())


class FusedShardedSpmv:
    """ShardedSpmv with the all-gather fused into the product kernel: each
    rank's epilogue stores its y rows into every rank's buffer over NVLink.
    Returns a view of this rank's gathered y (overwritten by the next call)."""

    def __init__(self, full, group=None, max_tokens: int = 1):
        self.group = group
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.plan = RowShardPlan.make(full.rows, world)
        self.r0, r1 = self.plan.local(rank)
        self.local = full.slice_rows(self.r0, r1)
        self.rows, self.cols, self.max_tokens = full.rows, full.cols, max_tokens
        own = PeerBuffer(max_tokens * full.rows)
        handles = exchange_handles(own.handle, group)
        bufs = [own if r == rank else PeerBuffer(handle=h) for r, h in enumerate(handles)]
        self.peers = PeerGroup(bufs, rank)

    def __call__(self, x, stream=None):
        M = 1 if x.dim() == 1 else x.shape[0]
        if M > self.max_tokens:
            raise ValueError("FusedShardedSpmv: more tokens than the peer buffers hold")
        self.peers.spmv(self.local, x, self.r0, self.rows, stream)
        return self.peers.y((self.rows,) if x.dim() == 1 else (M, self.rows))
