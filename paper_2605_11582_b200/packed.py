"""Python mirror of the reference's SparseGemv API (proj/include/egt/packed.hpp,
compress.hpp) over the C-ABI.  Same names, argument meaning and error classes:

* host encoder (C++ in csrc/host, byte-identical to the reference):
  ``fit_group``, ``quantize_matrix``, ``pack`` / ``pack_f32``, ``footprint``;
* device side (sm_100a kernels): ``DeviceMatrix`` (upload + validation once),
  ``spmv`` (packed.cpp:211-220), ``unpack`` (packed.cpp:197-209), M-row
  products for the verify pass, zero-copy row shards.

Arrays: W row-major [rows x cols] f32; masks are PruneMask bitmaps (bit
r*cols+c, LSB-first); codes one per byte for retained positions.
Device tensors are torch CUDA tensors (torch is the allocator/stream
plumbing only).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import native as N
from .native import check, lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


# ---------------------------------------------------------------- containers
@dataclass
class QuantizedMatrix:
    """compress.hpp:59-71"""

    rows: int
    cols: int
    group_sizes: np.ndarray
    group_offsets: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray
    codes: np.ndarray
    mask: np.ndarray | None = None  # PruneMask bits; None = all retained


@dataclass
class PackedSparseMatrix:
    """packed.hpp:37-67 (kind 1 INT4, 0 f32)."""

    n: int
    m: int
    rows: int
    cols: int
    kind: int
    index_words: np.ndarray
    value_bytes: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    group_sizes: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    group_offsets: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    scales: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    zero_points: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    values: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    @property
    def nnz(self) -> int:
        return self.rows * self.cols * self.n // self.m

    def view(self) -> N.PackedView:
        keep = {}
        for name, dt in (("index_words", np.uint16), ("value_bytes", np.uint8), ("group_sizes", np.uint32),
                         ("group_offsets", np.uint32), ("scales", np.float32), ("zero_points", np.uint8),
                         ("values", np.float32)):
            keep[name] = np.ascontiguousarray(getattr(self, name), dtype=dt)
        v = N.PackedView(
            self.n, self.m, self.rows, self.cols, self.kind,
            _p(keep["index_words"], N.u16p), keep["index_words"].size,
            _p(keep["value_bytes"], N.u8p), keep["value_bytes"].size,
            _p(keep["group_sizes"], N.u32p), keep["group_sizes"].size,
            _p(keep["group_offsets"], N.u32p), keep["group_offsets"].size,
            _p(keep["scales"], N.f32p), keep["scales"].size,
            _p(keep["zero_points"], N.u8p), keep["zero_points"].size,
            _p(keep["values"], N.f32p), keep["values"].size)
        v._keep = keep
        return v


def mask_bytes(rows: int, cols: int) -> int:
    return (rows * cols + 7) // 8


# ---------------------------------------------------------------- host encoder
def fit_group(values) -> tuple[float, int]:
    """fit_group (compress.cpp:77-90)."""
    v = np.ascontiguousarray(values, np.float64)
    s, z = C.c_float(), C.c_uint8()
    lib().egt_host_fit_group(_p(v, N.f64p), v.size, C.byref(s), C.byref(z))
    return s.value, z.value


def quantize_matrix(w: np.ndarray, group_sizes, mask: np.ndarray | None = None) -> QuantizedMatrix:
    """quantize_matrix (compress.cpp:157-208)."""
    w = np.ascontiguousarray(w, np.float32)
    rows, cols = w.shape
    gs = np.ascontiguousarray(np.broadcast_to(np.asarray(group_sizes, np.uint32), (rows,)), np.uint32)
    total = lib().egt_host_group_count(rows, cols, _p(gs, N.u32p))
    goff = np.zeros(rows + 1, np.uint32)
    scales = np.zeros(max(total, 1), np.float32)
    zps = np.zeros(max(total, 1), np.uint8)
    codes = np.zeros(max(rows * cols, 1), np.uint8)
    nc = C.c_size_t()
    mb = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    check(lib().egt_host_quantize(_p(w, N.f32p), rows, cols, _p(gs, N.u32p), _p(mb, N.u8p), _p(goff, N.u32p),
                                  _p(scales, N.f32p), _p(zps, N.u8p), _p(codes, N.u8p), C.byref(nc)))
    return QuantizedMatrix(rows, cols, gs, goff, scales[:total].copy(), zps[:total].copy(),
                           codes[: nc.value].copy(), None if mb is None else mb.copy())


def pack(mask: np.ndarray, quant: QuantizedMatrix, n: int, m: int = 4) -> PackedSparseMatrix:
    """pack(mask, QuantizedMatrix, n, m) (packed.cpp:92-128)."""
    mb = np.ascontiguousarray(mask, np.uint8)
    rows, cols = quant.rows, quant.cols
    if quant.mask is not None and not np.array_equal(quant.mask, mb):
        raise N.InvalidArgument(N.EGT_EINVAL, "pack: quantized mask differs from prune mask")
    cap = rows * cols
    words = np.zeros(max((cap + 7) // 8, 1), np.uint16)
    vb = np.zeros(max((cap + 1) // 2, 1), np.uint8)
    nw, nv = C.c_size_t(), C.c_size_t()
    codes = np.ascontiguousarray(quant.codes, np.uint8)
    check(lib().egt_host_pack_int4(_p(mb, N.u8p), rows, cols, n, m, _p(codes, N.u8p), codes.size,
                                   int(quant.mask is None), _p(words, N.u16p), C.byref(nw), _p(vb, N.u8p),
                                   C.byref(nv)))
    return PackedSparseMatrix(n, m, rows, cols, N.KIND_INT4, words[: nw.value].copy(), vb[: nv.value].copy(),
                              quant.group_sizes.copy(), quant.group_offsets.copy(), quant.scales.copy(),
                              quant.zero_points.copy())


def pack_f32(mask: np.ndarray, w: np.ndarray, n: int, m: int = 4) -> PackedSparseMatrix:
    """pack(mask, Matrix, n, m) (packed.cpp:130-141)."""
    mb = np.ascontiguousarray(mask, np.uint8)
    w = np.ascontiguousarray(w, np.float32)
    rows, cols = w.shape
    words = np.zeros(max((rows * cols + 7) // 8, 1), np.uint16)
    vals = np.zeros(max(rows * cols, 1), np.float32)
    nw, nv = C.c_size_t(), C.c_size_t()
    check(lib().egt_host_pack_f32(_p(mb, N.u8p), rows, cols, n, m, _p(w, N.f32p), _p(words, N.u16p),
                                  C.byref(nw), _p(vals, N.f32p), C.byref(nv)))
    return PackedSparseMatrix(n, m, rows, cols, N.KIND_F32, words[: nw.value].copy(), values=vals[: nv.value].copy())


def footprint(p: PackedSparseMatrix) -> dict:
    """footprint (packed.cpp:222-240)."""
    out = (C.c_uint64 * 5)()
    ratio = C.c_double()
    v = p.view()
    check(lib().egt_host_footprint(C.byref(v), out, C.byref(ratio)))
    d = dict(zip(("index_bytes", "value_bytes", "scale_bytes", "packed_bytes", "baseline_bytes"), map(int, out)))
    d["ratio"] = ratio.value
    return d


# ---------------------------------------------------------------- device
def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


class DeviceMatrix:
    """A packed layer resident in HBM (immutable).  See include/egt_b200.h."""

    def __init__(self, handle: int, parent: "DeviceMatrix | None" = None):
        self._h = C.c_void_p(handle)
        self._parent = parent
        info = N.DevInfo()
        check(lib().egt_dev_packed_query(self._h, C.byref(info)))
        self.rows, self.cols = info.rows, info.cols
        self.n, self.kind = info.n, info.kind
        self.format = N.FMT_NAMES[info.format]
        self.path = N.PATH_NAMES[info.path]
        self.device_bytes = info.device_bytes
        self.algorithmic_bytes = info.algorithmic_bytes
        self.nnz = info.nnz

    @classmethod
    def from_packed(cls, p: PackedSparseMatrix, stream=None, round_fp16: bool = False) -> "DeviceMatrix":
        """Upload (egt_dev_packed_create_ex).  Sparse-FP values fp16 cannot
        hold exactly raise InvalidArgument unless round_fp16."""
        v = p.view()
        h = C.c_void_p()
        check(lib().egt_dev_packed_create_ex(C.byref(v), N.UPLOAD_ROUND_FP16 if round_fp16 else 0,
                                             _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    @classmethod
    def dense_i4(cls, q: QuantizedMatrix, stream=None) -> "DeviceMatrix":
        """Dense INT4 layer (quant_dense_gemv arm, packed.cpp:266-281)."""
        if q.mask is not None:
            raise N.InvalidArgument(N.EGT_EINVAL, "dense int4: quantized matrix has a prune mask")
        keep = [np.ascontiguousarray(a, dt) for a, dt in ((q.group_sizes, np.uint32), (q.group_offsets, np.uint32),
                                                           (q.scales, np.float32), (q.zero_points, np.uint8),
                                                           (q.codes, np.uint8))]
        v = N.QuantView(q.rows, q.cols, _p(keep[0], N.u32p), _p(keep[1], N.u32p), _p(keep[2], N.f32p),
                        keep[2].size, _p(keep[3], N.u8p), _p(keep[4], N.u8p), keep[4].size)
        h = C.c_void_p()
        check(lib().egt_dev_dense_i4_create(C.byref(v), _stream_ptr(stream), C.byref(h)))
        return cls(h.value)

    def slice_rows(self, r0: int, r1: int) -> "DeviceMatrix":
        h = C.c_void_p()
        check(lib().egt_dev_packed_slice_rows(self._h, r0, r1, C.byref(h)))
        return DeviceMatrix(h.value, parent=self)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_dev_packed_destroy(h)
            self._h = C.c_void_p()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    # products -------------------------------------------------------
    def spmv_into(self, x, y, stream=None, independent: bool = False) -> None:
        """y[M x rows] = x[M x cols] @ W^T on the device (torch CUDA f32 tensors).
        independent=True: x was not written by the previous kernel on the
        stream (EGT_SPMV_INDEPENDENT), so this product may overlap it."""
        if x.dim() == 1:
            M, ldx = 1, x.shape[0]
        else:
            M, ldx = x.shape[0], x.stride(0)
        ldy = y.shape[-1] if y.dim() == 1 else y.stride(0)
        if x.dim() == 1 and x.shape[0] != self.cols:
            raise N.InvalidArgument(N.EGT_EINVAL, "spmv: input length differs from columns")
        check(lib().egt_spmv_ex(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), M, ldx, ldy,
                                1 if independent else 0, _stream_ptr(stream)))

    def spmv_fused_into(self, x, y, residual=None, input: int = 0, eps: float = 1e-6, stream=None,
                        independent: bool = False, l2_next: "DeviceMatrix | None" = None,
                        output_silu: bool = False) -> None:
        """y = residual + f(x) @ W^T with f = identity / rmsnorm (per token) /
        silu (N.INPUT_*): the forward_impl glue (model.cpp:155-190) fused into
        the product.  residual may be y itself."""
        M, ldx = (1, x.shape[0]) if x.dim() == 1 else (x.shape[0], x.stride(0))
        ldy = y.shape[-1] if y.dim() == 1 else y.stride(0)
        if x.dim() == 1 and x.shape[0] != self.cols:
            raise N.InvalidArgument(N.EGT_EINVAL, "spmv: input length differs from columns")
        rp, ldr = None, 0
        if residual is not None:
            rp = residual.data_ptr()
            ldr = residual.shape[-1] if residual.dim() == 1 else residual.stride(0)
        check(lib().egt_spmv_fused(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), M, ldx, ldy,
                                   rp, ldr, input, eps, (1 if independent else 0) | (2 if output_silu else 0),
                                   l2_next.handle if l2_next is not None else None, _stream_ptr(stream)))

    def spmv(self, x, stream=None):
        """Device product; returns a new tensor [M x rows] (or [rows] for 1-D x)."""
        import torch

        out_shape = (self.rows,) if x.dim() == 1 else (x.shape[0], self.rows)
        y = torch.empty(out_shape, dtype=torch.float32, device=x.device)
        self.spmv_into(x, y, stream)
        return y

    def spmv_host(self, x: np.ndarray, stream=None) -> np.ndarray:
        """The drop-in call: host x -> host y (H2D, product, D2H, sync)."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(max(self.rows, 1), np.float32)
        check(lib().egt_spmv_host(self._h, _p(x, N.f32p), x.size, _p(y, N.f32p), _stream_ptr(stream)))
        return y[: self.rows]

    def dequant(self, stream=None):
        """Bit-exact device unpack -> (W [rows x cols] f32 tensor, PruneMask bits np.uint8)."""
        import torch

        n = self.rows * self.cols
        w = torch.empty((self.rows, self.cols), dtype=torch.float32, device="cuda")
        words = torch.empty(max((n + 31) // 32, 1), dtype=torch.int32, device="cuda")
        check(lib().egt_dequant(self._h, C.c_void_p(w.data_ptr()), C.c_void_p(words.data_ptr()),
                                _stream_ptr(stream)))
        bits = words.cpu().numpy().view(np.uint8)[: mask_bytes(self.rows, self.cols)].copy()
        return w, bits


def spmv_fused_multi(mats, x, ys, input: int = 0, eps: float = 1e-6, stream=None, independent: bool = False):
    """ys[i] = f(x) @ W_i^T for up to three same-shape matrices in one launch
    (egt_spmv_fused_multi; the decode step's Q, K, V)."""
    n = len(mats)
    hs = (C.c_void_p * n)(*[m.handle.value for m in mats])
    yp = (C.c_void_p * n)(*[y.data_ptr() for y in ys])
    check(lib().egt_spmv_fused_multi(hs, n, C.c_void_p(x.data_ptr()), yp, input, eps, 1 if independent else 0,
                                     _stream_ptr(stream)))


def spmm_multi(mats, x, ys, input: int = 0, eps: float = 1e-6, stream=None):
    """ys[i] = f(x) @ W_i^T (x: M x cols, f = identity / rmsnorm) for up to
    three matrices sharing x (egt_spmm_multi; the verify pass's Q, K, V: one
    tcgen05 launch)."""
    n = len(mats)
    M, ldx = (1, x.shape[0]) if x.dim() == 1 else (x.shape[0], x.stride(0))
    ldy = ys[0].shape[-1] if ys[0].dim() == 1 else ys[0].stride(0)
    hs = (C.c_void_p * n)(*[m.handle.value for m in mats])
    yp = (C.c_void_p * n)(*[y.data_ptr() for y in ys])
    check(lib().egt_spmm_multi(hs, n, C.c_void_p(x.data_ptr()), M, ldx, yp, ldy, input, eps, _stream_ptr(stream)))


def spmv(w, x):
    """spmv (packed.hpp:83-85): host vectors in/out.  w: DeviceMatrix or PackedSparseMatrix."""
    if isinstance(w, PackedSparseMatrix):
        x = np.asarray(x, np.float32)
        if x.size != w.cols:
            raise N.InvalidArgument(N.EGT_EINVAL, "spmv: input length differs from columns")
        w = DeviceMatrix.from_packed(w)
    return w.spmv_host(x)


def unpack(w):
    """unpack (packed.hpp:81) on the device: (values np [rows x cols], mask bits)."""
    if isinstance(w, PackedSparseMatrix):
        w = DeviceMatrix.from_packed(w)
    vals, bits = w.dequant()
    return vals.cpu().numpy(), bits


def set_pdl(enabled: bool) -> None:
    lib().egt_set_pdl(int(enabled))


def launch_count() -> int:
    return int(lib().egt_launch_count())


# ---------------------------------------------------------------- GPU compression
# (include/egt_b200.h egt_gpu_*) torch CUDA tensors in/out.
def gpu_importance(w, x_norms, grad_abs, stream=None):
    """importance_scores (compress.cpp:230-244) on the device."""
    import torch

    rows, cols = w.shape
    out = torch.empty((rows, cols), dtype=torch.float32, device=w.device)
    check(lib().egt_gpu_importance(C.c_void_p(w.data_ptr()), C.c_void_p(x_norms.data_ptr()),
                                   C.c_void_p(grad_abs.data_ptr()), rows, cols, C.c_void_p(out.data_ptr()),
                                   _stream_ptr(stream)))
    return out


def gpu_prune_nm(scores, n: int, m: int = 4, stream=None):
    """prune_nm (compress.cpp:246-278): PruneMask bitmap (uint8 CUDA tensor)."""
    import torch

    rows, cols = scores.shape
    mask = torch.empty(max(1, (rows * cols + 7) // 8), dtype=torch.uint8, device=scores.device)
    check(lib().egt_gpu_prune_nm(C.c_void_p(scores.data_ptr()), rows, cols, n, m, C.c_void_p(mask.data_ptr()),
                                 _stream_ptr(stream)))
    return mask[: (rows * cols + 7) // 8]


def gpu_quantize_pack(w, mask, n: int, group_sizes, stream=None, want_raw: bool = True, want_matrix: bool = True):
    """quantize_matrix + pack on the device.  Returns (DeviceMatrix or None,
    dict of the reference-layout arrays as CUDA tensors or None)."""
    import torch

    rows, cols = w.shape
    gs = np.ascontiguousarray(np.broadcast_to(np.asarray(group_sizes, np.uint32), (rows,)))
    nnz = rows * cols * n // 4
    groups = int(sum((cols + int(g) - 1) // int(g) for g in gs)) if rows and np.all(gs > 0) else 0
    raw = None
    ro = None
    if want_raw:
        dev = w.device
        raw = {"index_words": torch.empty(max(1, (nnz + 7) // 8), dtype=torch.int16, device=dev),
               "value_bytes": torch.empty(max(1, (nnz + 1) // 2), dtype=torch.uint8, device=dev),
               "group_offsets": torch.empty(rows + 1, dtype=torch.int32, device=dev),
               "scales": torch.empty(max(1, groups), dtype=torch.float32, device=dev),
               "zero_points": torch.empty(max(1, groups), dtype=torch.uint8, device=dev)}
        ro = N.GpuPackedOut(*[C.c_void_p(raw[k].data_ptr()) for k in
                              ("index_words", "value_bytes", "group_offsets", "scales", "zero_points")])
    h = C.c_void_p()
    check(lib().egt_gpu_quantize_pack(C.c_void_p(w.data_ptr()), C.c_void_p(mask.data_ptr()), rows, cols, n,
                                      _p(gs, N.u32p), C.byref(ro) if ro is not None else None, _stream_ptr(stream),
                                      C.byref(h) if want_matrix else None))
    if raw is not None:
        raw["index_words"] = raw["index_words"][: (nnz + 7) // 8]
        raw["value_bytes"] = raw["value_bytes"][: (nnz + 1) // 2]
        raw["scales"] = raw["scales"][:groups]
        raw["zero_points"] = raw["zero_points"][:groups]
    return (DeviceMatrix(h.value) if want_matrix else None), raw


def gemv_f32(w, x, stream=None):
    """y = W x for a dense f32 CUDA tensor W (the dense-FP baseline arm)."""
    import torch

    rows, cols = w.shape
    y = torch.empty(rows, dtype=torch.float32, device=w.device)
    check(lib().egt_gemv_f32(C.c_void_p(w.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), rows,
                             cols, _stream_ptr(stream)))
    return y


def bench_spmv(shapes, reps: int = 5, seed: int = 0) -> str:
    """bench_spmv + bench_csv (packed.cpp:310-393) on the device: the CSV text
    (variant,rows,cols,pattern,median_ns,p95_ns,bytes)."""
    rows = np.ascontiguousarray([s[0] for s in shapes], np.uint32)
    cols = np.ascontiguousarray([s[1] for s in shapes], np.uint32)
    n = C.c_size_t()
    cap = 256 + 160 * 4 * max(1, len(shapes))
    buf = C.create_string_buffer(cap)
    check(lib().egt_bench_spmv(_p(rows, N.u32p), _p(cols, N.u32p), len(shapes), reps, C.c_uint64(seed), buf, cap,
                               C.byref(n)))
    return buf.value.decode()
