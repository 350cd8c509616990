"""EGTQ compressed-model files -> device layers (include/egt_b200.h
egt_egtq_*; the reader restates egtq_io.cpp:110-235 with the reference's
checks and FormatError messages)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native as N
from .native import check, lib
from .packed import DeviceMatrix, _stream_ptr

PATTERNS = {0: "dense", 1: "1:4", 2: "2:4"}


@dataclass
class LayerInfo:
    name: str
    pattern: str
    has_quant: bool
    has_index: bool
    rows: int
    cols: int


class EgtqFile:
    def __init__(self, data: bytes, context: str = "egtq"):
        buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        h = C.c_void_p()
        check(lib().egt_egtq_parse(buf.ctypes.data_as(N.u8p), len(data), context.encode(), C.byref(h)))
        self._h = h
        self.layers = []
        for i in range(lib().egt_egtq_layer_count(h)):
            info = N.EgtqLayerInfo()
            check(lib().egt_egtq_query(h, i, C.byref(info)))
            self.layers.append(LayerInfo(info.name.decode(errors="replace"), PATTERNS[info.pattern], bool(info.has_quant),
                                         bool(info.has_index), info.rows, info.cols))

    @classmethod
    def load(cls, path: str) -> "EgtqFile":
        with open(path, "rb") as f:
            return cls(f.read(), path)

    def upload(self, i: int, stream=None, round_fp16: bool = False) -> DeviceMatrix:
        """Layer i as a device matrix (mixed dispatch on pattern x storage).
        Sparse-FP layers whose f32 values fp16 cannot hold exactly raise
        InvalidArgument unless round_fp16."""
        h = C.c_void_p()
        check(lib().egt_egtq_upload_ex(self._h, i, N.UPLOAD_ROUND_FP16 if round_fp16 else 0, _stream_ptr(stream),
                                       C.byref(h)))
        return DeviceMatrix(h.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_egtq_destroy(h)
            self._h = C.c_void_p()
