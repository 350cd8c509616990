"""Persistent GEMV programs (include/egt_b200.h, egt_program_*).

A ``Program`` is an ordered list of batch-1 products

    y_j = residual_j + W_j f_j(x_j),   f_j in {identity, rmsnorm, silu}

run by ONE persistent launch (csrc/program.cu): every SM streams its share of
every op's packed weights through one shared-memory ring, so the weights of
op j+1 are in flight while op j's output is still being produced.  ``wait``
orders ops: op j with wait=w reads its inputs only after ops 0..w are
complete.  The glue is the reference's forward_impl (model.cpp:155-190):
rmsnorm (model.cpp:57-67), silu (model.cpp:80-84), x += t (model.cpp:186,190).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import native as N
from .native import check, lib
from .packed import DeviceMatrix, _stream_ptr

NONE, RMSNORM, SILU = N.INPUT_NONE, N.INPUT_RMSNORM, N.INPUT_SILU
NORM_EPS = 1e-6  # model.cpp:27


@dataclass
class Op:
    w: DeviceMatrix
    x: object  # torch CUDA f32 tensor [cols]
    y: object  # torch CUDA f32 tensor [rows]
    residual: object = None
    input: int = NONE
    wait: int = -1
    eps: float = NORM_EPS


class Program:
    def __init__(self, ops: list[Op], stream=None):
        self.ops = list(ops)
        arr = (N.ProgramOp * len(self.ops))()
        for i, o in enumerate(self.ops):
            for t in (o.x, o.y) + ((o.residual,) if o.residual is not None else ()):
                if not t.is_cuda or not t.is_contiguous():
                    raise N.InvalidArgument(N.EGT_EINVAL, f"program: op {i}: vectors must be contiguous CUDA tensors")
            if o.x.numel() != o.w.cols:
                raise N.InvalidArgument(N.EGT_EINVAL, "spmv: input length differs from columns")
            if o.y.numel() != o.w.rows:
                raise N.InvalidArgument(N.EGT_EINVAL, f"program: op {i}: output length differs from rows")
            arr[i] = N.ProgramOp(o.w.handle.value, o.x.data_ptr(), o.y.data_ptr(),
                                 o.residual.data_ptr() if o.residual is not None else None,
                                 o.input, o.eps, o.wait)
        h = C.c_void_p()
        check(lib().egt_program_create(arr, len(self.ops), _stream_ptr(stream), C.byref(h)))
        self._h = h
        info = N.ProgramInfo()
        check(lib().egt_program_query(h, C.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in N.ProgramInfo._fields_}

    def run(self, stream=None) -> None:
        check(lib().egt_program_run(self._h, _stream_ptr(stream)))

    @property
    def algorithmic_bytes(self) -> int:
        """SURVEY 8(d) bytes of every op: packed weights + tables + x + y."""
        return sum(o.w.algorithmic_bytes + 4 * o.w.cols + 4 * o.w.rows for o in self.ops)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_program_destroy(h)
            self._h = C.c_void_p()
