"""ctypes front end for the test oracles (TEST INFRASTRUCTURE ONLY).

Two checkers with the same flat interface:

* ``Oracle("port")``      -- oracle/_build/libegt_oracle.so, the C restatement
  in oracle/egt_oracle.c (each function cites the reference file:line);
* ``Oracle("reference")`` -- oracle/_ref/libegt_ref.so, the reference's own
  packed.cpp / compress.cpp compiled unmodified (oracle/build_ref.sh).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product package never does.

Arrays follow the reference containers: W is row-major [rows x cols] f32,
masks are PruneMask bitmaps (bit r*cols+c, LSB-first, compress.hpp:36-45),
codes are one per byte for retained positions (compress.hpp:59-71).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libegt_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libegt_ref.so")

_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)


class OracleError(Exception):
    """Raised with the reference's exception class name and message."""

    KIND = {1: "invalid_argument", 2: "FormatError", 3: "InvariantError", 4: "exception"}

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = self.KIND.get(code, "unknown")
        super().__init__(f"{self.kind}: {msg}")


class _Packed(C.Structure):
    _fields_ = [
        ("n", C.c_uint8), ("m", C.c_uint8), ("rows", C.c_uint32), ("cols", C.c_uint32),
        ("kind", C.c_uint8),
        ("index_words", _u16p), ("n_index_words", C.c_size_t),
        ("value_bytes", _u8p), ("n_value_bytes", C.c_size_t),
        ("group_sizes", _u32p), ("n_group_sizes", C.c_size_t),
        ("group_offsets", _u32p), ("n_group_offsets", C.c_size_t),
        ("scales", _f32p), ("n_scales", C.c_size_t),
        ("zero_points", _u8p), ("n_zero_points", C.c_size_t),
        ("values", _f32p), ("n_values", C.c_size_t),
    ]


def _ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


@dataclass
class Quantized:
    """QuantizedMatrix (compress.hpp:59-71)."""

    rows: int
    cols: int
    group_sizes: np.ndarray
    group_offsets: np.ndarray
    scales: np.ndarray
    zero_points: np.ndarray
    codes: np.ndarray
    mask: np.ndarray | None = None  # PruneMask bits; None = all retained


@dataclass
class Packed:
    """PackedSparseMatrix (packed.hpp:37-67); kind 1 = INT4, 0 = f32."""

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

    def struct(self) -> _Packed:
        # keep contiguous copies alive on the struct
        keep = {}
        for name, dt in (("index_words", np.uint16), ("value_bytes", np.uint8),
                         ("group_sizes", np.uint32), ("group_offsets", np.uint32),
                         ("scales", np.float32), ("zero_points", np.uint8),
                         ("values", np.float32)):
            keep[name] = np.ascontiguousarray(getattr(self, name), dtype=dt)
        s = _Packed(
            self.n, self.m, self.rows, self.cols, self.kind,
            _ptr(keep["index_words"], _u16p), keep["index_words"].size,
            _ptr(keep["value_bytes"], _u8p), keep["value_bytes"].size,
            _ptr(keep["group_sizes"], _u32p), keep["group_sizes"].size,
            _ptr(keep["group_offsets"], _u32p), keep["group_offsets"].size,
            _ptr(keep["scales"], _f32p), keep["scales"].size,
            _ptr(keep["zero_points"], _u8p), keep["zero_points"].size,
            _ptr(keep["values"], _f32p), keep["values"].size,
        )
        s._keep = keep
        return s


def mask_bytes(rows: int, cols: int) -> int:
    return (rows * cols + 7) // 8


def mask_from_bool(b: np.ndarray) -> np.ndarray:
    """Dense bool [rows x cols] -> PruneMask bits (LSB-first)."""
    flat = np.ascontiguousarray(b, dtype=bool).reshape(-1)
    return np.packbits(flat, bitorder="little")


def mask_to_bool(bits: np.ndarray, rows: int, cols: int) -> np.ndarray:
    return np.unpackbits(np.asarray(bits, np.uint8), bitorder="little")[: rows * cols].reshape(rows, cols).astype(bool)


class Oracle:
    def __init__(self, which: str = "port"):
        self.which = which
        path = PORT_LIB if which == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run oracle/build_ref.sh")
        self.lib = C.CDLL(path)
        p = "egto_" if which == "port" else "ref_"
        self.p = p
        L = self.lib
        err = getattr(L, "egto_last_error" if which == "port" else "ref_last_error")
        err.restype = C.c_char_p
        self._err = err
        if which == "port":
            L.egto_fit_group.argtypes = [_f64p, C.c_size_t, _f32p, _u8p]
        else:
            L.ref_fit_group.argtypes = [_f64p, C.c_size_t, _f32p, _u8p]
        getattr(L, p + "encode_value").argtypes = [C.c_double, C.c_float, C.c_uint8]
        getattr(L, p + "encode_value").restype = C.c_uint8
        getattr(L, p + "decode_value").argtypes = [C.c_uint8, C.c_float, C.c_uint8]
        getattr(L, p + "decode_value").restype = C.c_float
        for fn in ("unpack", "spmv", "footprint"):
            getattr(L, p + fn).restype = C.c_int

    # ------------------------------------------------------------ helpers
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._err().decode(errors="replace"))

    # ------------------------------------------------------------ quant
    def fit_group(self, values) -> tuple[float, int]:
        v = np.ascontiguousarray(values, dtype=np.float64)
        s = C.c_float()
        z = C.c_uint8()
        getattr(self.lib, self.p + "fit_group")(_ptr(v, _f64p), v.size, C.byref(s), C.byref(z))
        return s.value, z.value

    def encode_value(self, value: float, scale: float, zp: int) -> int:
        return getattr(self.lib, self.p + "encode_value")(value, scale, zp)

    def decode_value(self, code: int, scale: float, zp: int) -> float:
        return getattr(self.lib, self.p + "decode_value")(code, scale, zp)

    def quantize(self, w: np.ndarray, group_sizes, mask: np.ndarray | None = None) -> Quantized:
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        gs = np.ascontiguousarray(group_sizes, dtype=np.uint32)
        total = int(sum((cols + int(g) - 1) // int(g) for g in gs)) if np.all(gs > 0) else 0
        goff = np.zeros(rows + 1, np.uint32)
        scales = np.zeros(max(total, 1), np.float32)
        zps = np.zeros(max(total, 1), np.uint8)
        codes = np.zeros(max(rows * cols, 1), np.uint8)
        nc = C.c_size_t()
        mb = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        rc = getattr(self.lib, self.p + "quantize")(
            _ptr(w, _f32p), rows, cols, _ptr(gs, _u32p), _ptr(mb, _u8p), _ptr(goff, _u32p),
            _ptr(scales, _f32p), _ptr(zps, _u8p), _ptr(codes, _u8p), C.byref(nc))
        self._check(rc)
        return Quantized(rows, cols, gs.copy(), goff, scales[:total].copy(), zps[:total].copy(),
                         codes[: nc.value].copy(), None if mb is None else mb.copy())

    def importance(self, w: np.ndarray, x_norms: np.ndarray, grad_abs: np.ndarray) -> np.ndarray:
        """importance_scores (compress.cpp:230-244)."""
        w = np.ascontiguousarray(w, np.float32)
        xn = np.ascontiguousarray(x_norms, np.float32)
        g = np.ascontiguousarray(grad_abs, np.float32)
        out = np.zeros(w.shape, np.float32)
        self._check(getattr(self.lib, self.p + "importance")(_ptr(w, _f32p), _ptr(xn, _f32p), _ptr(g, _f32p),
                                                             w.shape[0], w.shape[1], _ptr(out, _f32p)))
        return out

    def prune_nm(self, scores: np.ndarray, n: int, m: int = 4) -> np.ndarray:
        """prune_nm (compress.cpp:246-278): the PruneMask bitmap."""
        s = np.ascontiguousarray(scores, np.float32)
        rows, cols = s.shape
        bits = np.zeros(max(1, (rows * cols + 7) // 8), np.uint8)
        self._check(getattr(self.lib, self.p + "prune_nm")(_ptr(s, _f32p), rows, cols, n, m, _ptr(bits, _u8p)))
        return bits[: (rows * cols + 7) // 8]

    def dequantize(self, q: Quantized) -> np.ndarray:
        out = np.zeros((q.rows, q.cols), np.float32)
        mb = None if q.mask is None else np.ascontiguousarray(q.mask, np.uint8)
        if self.which == "port":
            rc = self.lib.egto_dequantize(
                q.rows, q.cols, _ptr(q.group_sizes, _u32p), _ptr(q.group_offsets, _u32p),
                _ptr(q.scales, _f32p), _ptr(q.zero_points, _u8p), _ptr(mb, _u8p),
                _ptr(q.codes, _u8p), C.c_size_t(q.codes.size), _ptr(out, _f32p))
        else:
            rc = self.lib.ref_dequantize(
                q.rows, q.cols, _ptr(q.group_sizes, _u32p), _ptr(q.group_offsets, _u32p),
                _ptr(q.scales, _f32p), _ptr(q.zero_points, _u8p), C.c_size_t(q.scales.size),
                _ptr(mb, _u8p), _ptr(q.codes, _u8p), C.c_size_t(q.codes.size), _ptr(out, _f32p))
        self._check(rc)
        return out

    # ------------------------------------------------------------ pack
    def pack_int4(self, mask: np.ndarray, rows: int, cols: int, q: Quantized, n: int, m: int = 4) -> Packed:
        mb = np.ascontiguousarray(mask, np.uint8)
        nnz_cap = rows * cols
        words = np.zeros(max((nnz_cap + 7) // 8, 1), np.uint16)
        vb = np.zeros(max((nnz_cap + 1) // 2, 1), np.uint8)
        nw = C.c_size_t()
        nv = C.c_size_t()
        if self.which == "port":
            if q.rows != rows or q.cols != cols:
                raise OracleError(1, "pack: quantized shape differs from mask")
            dense = q.mask is None
            if not dense and not np.array_equal(q.mask, mb):
                raise OracleError(1, "pack: quantized mask differs from prune mask")
            self._check(self.lib.egto_pack_index(_ptr(mb, _u8p), rows, cols, n, m, _ptr(words, _u16p), C.byref(nw)))
            self._check(self.lib.egto_pack_codes(_ptr(mb, _u8p), rows, cols, n, _ptr(q.codes, _u8p),
                                                 C.c_size_t(q.codes.size), int(dense), _ptr(vb, _u8p), C.byref(nv)))
        else:
            qm = None if q.mask is None else np.ascontiguousarray(q.mask, np.uint8)
            self._check(self.lib.ref_pack_int4(
                _ptr(mb, _u8p), rows, cols, n, m, q.rows, q.cols, _ptr(q.group_sizes, _u32p),
                _ptr(q.group_offsets, _u32p), _ptr(q.scales, _f32p), _ptr(q.zero_points, _u8p),
                C.c_size_t(q.scales.size), _ptr(qm, _u8p), _ptr(q.codes, _u8p), C.c_size_t(q.codes.size),
                _ptr(words, _u16p), C.byref(nw), _ptr(vb, _u8p), C.byref(nv)))
        return Packed(n, m, rows, cols, 1, words[: nw.value].copy(), vb[: nv.value].copy(),
                      q.group_sizes.copy(), q.group_offsets.copy(), q.scales.copy(), q.zero_points.copy())

    def pack_f32(self, mask: np.ndarray, rows: int, cols: int, w: np.ndarray, n: int, m: int = 4) -> Packed:
        mb = np.ascontiguousarray(mask, np.uint8)
        w = np.ascontiguousarray(w, np.float32)
        words = np.zeros(max((rows * cols + 7) // 8, 1), np.uint16)
        vals = np.zeros(max(rows * cols, 1), np.float32)
        nw = C.c_size_t()
        nv = C.c_size_t()
        if self.which == "port":
            if w.shape != (rows, cols):
                raise OracleError(1, "pack: value shape differs from mask")
            self._check(self.lib.egto_pack_index(_ptr(mb, _u8p), rows, cols, n, m, _ptr(words, _u16p), C.byref(nw)))
            self._check(self.lib.egto_pack_values(_ptr(mb, _u8p), rows, cols, _ptr(w, _f32p), _ptr(vals, _f32p), C.byref(nv)))
        else:
            self._check(self.lib.ref_pack_f32(_ptr(mb, _u8p), rows, cols, n, m, _ptr(w, _f32p), w.shape[0], w.shape[1],
                                              _ptr(words, _u16p), C.byref(nw), _ptr(vals, _f32p), C.byref(nv)))
        return Packed(n, m, rows, cols, 0, words[: nw.value].copy(), values=vals[: nv.value].copy())

    def unpack(self, p: Packed) -> tuple[np.ndarray, np.ndarray]:
        vals = np.zeros((p.rows, p.cols), np.float32)
        bits = np.zeros(max(mask_bytes(p.rows, p.cols), 1), np.uint8)
        s = p.struct()
        self._check(getattr(self.lib, self.p + "unpack")(C.byref(s), _ptr(vals, _f32p), _ptr(bits, _u8p)))
        return vals, bits[: mask_bytes(p.rows, p.cols)]

    def spmv(self, p: Packed, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(max(p.rows, 1), np.float32)
        s = p.struct()
        self._check(getattr(self.lib, self.p + "spmv")(C.byref(s), _ptr(x, _f32p), C.c_size_t(x.size), _ptr(y, _f32p)))
        return y[: p.rows]

    def footprint(self, p: Packed) -> dict:
        out = (C.c_uint64 * 5)()
        ratio = C.c_double()
        s = p.struct()
        self._check(getattr(self.lib, self.p + "footprint")(C.byref(s), out, C.byref(ratio)))
        keys = ("index_bytes", "value_bytes", "scale_bytes", "packed_bytes", "baseline_bytes")
        d = {k: int(v) for k, v in zip(keys, out)}
        d["ratio"] = ratio.value
        return d

    # ------------------------------------------------------------ port-only
    def quant_dense_gemv(self, q: Quantized, x: np.ndarray) -> np.ndarray:
        assert self.which == "port", "quant_dense_gemv is file-private in the reference"
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(q.rows, np.float32)
        self.lib.egto_quant_dense_gemv(q.rows, q.cols, _ptr(q.group_sizes, _u32p), _ptr(q.group_offsets, _u32p),
                                       _ptr(q.scales, _f32p), _ptr(q.zero_points, _u8p), _ptr(q.codes, _u8p),
                                       _ptr(x, _f32p), _ptr(y, _f32p))
        return y

    def magnitude_mask(self, w: np.ndarray, n: int, m: int = 4) -> np.ndarray:
        assert self.which == "port"
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        bits = np.zeros(max(mask_bytes(rows, cols), 1), np.uint8)
        self.lib.egto_magnitude_mask(_ptr(w, _f32p), rows, cols, n, m, _ptr(bits, _u8p))
        return bits[: mask_bytes(rows, cols)]

    def sinusoidal_positions(self, max_positions: int, d_model: int) -> np.ndarray:
        out = np.zeros((max_positions, d_model), np.float32)
        self.lib.egto_sinusoidal_positions(max_positions, d_model, _ptr(out, _f32p))
        return out

    def forward(self, cfg: dict, embedding, layers, head, positions, tokens, pos, mask) -> np.ndarray:
        """forward (model.cpp:358-361). layers: list of dicts wq,wk,wv,wo,ff1,ff2."""
        assert self.which == "port"

        class Cfg(C.Structure):
            _fields_ = [(k, C.c_uint32) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_positions")]

        c = Cfg(*(int(cfg[k]) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_positions")))
        keep = []
        ptrs = (_f32p * (6 * len(layers)))()
        for li, L in enumerate(layers):
            for j, name in enumerate(("wq", "wk", "wv", "wo", "ff1", "ff2")):
                a = np.ascontiguousarray(L[name], np.float32)
                keep.append(a)
                ptrs[6 * li + j] = _ptr(a, _f32p)
        emb = np.ascontiguousarray(embedding, np.float32)
        hd = np.ascontiguousarray(head, np.float32)
        ps = np.ascontiguousarray(positions, np.float32)
        tk = np.ascontiguousarray(tokens, np.int32)
        po = np.ascontiguousarray(pos, np.int32)
        mk = np.ascontiguousarray(mask, np.uint8)
        n = tk.size
        logits = np.zeros((n, int(cfg["vocab_size"])), np.float32)
        self._check(self.lib.egto_forward(C.byref(c), _ptr(emb, _f32p), ptrs, _ptr(hd, _f32p), _ptr(ps, _f32p),
                                          tk.ctypes.data_as(C.POINTER(C.c_int)), po.ctypes.data_as(C.POINTER(C.c_int)),
                                          _ptr(mk, _u8p), n, _ptr(logits, _f32p)))
        return logits

    def log_softmax(self, row: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(row, np.float32)
        out = np.zeros_like(r)
        self.lib.egto_log_softmax(_ptr(r, _f32p), C.c_size_t(r.size), _ptr(out, _f32p))
        return out

    # ------------------------------------------------------------ reference-only timing
    def ref_timed_spmv(self, p: Packed, x: np.ndarray, calls: int, threads: int) -> tuple[float, np.ndarray]:
        assert self.which == "reference"
        L = self.lib
        L.ref_packed_new.restype = C.c_void_p
        L.ref_packed_free.argtypes = [C.c_void_p]
        s = p.struct()
        h = L.ref_packed_new(C.byref(s))
        if not h:
            raise OracleError(4, "ref_packed_new failed")
        try:
            x = np.ascontiguousarray(x, np.float32)
            y = np.zeros(p.rows, np.float32)
            sec = C.c_double()
            L.ref_spmv_timed.argtypes = [C.c_void_p, _f32p, C.c_size_t, C.c_int, C.c_int, _f64p, _f32p]
            self._check(L.ref_spmv_timed(h, _ptr(x, _f32p), C.c_size_t(x.size), calls, threads, C.byref(sec), _ptr(y, _f32p)))
            return sec.value, y
        finally:
            L.ref_packed_free(h)

    def ref_egtq_serialize(self, layers: list) -> bytes:
        """serialize_compressed (egtq_io.cpp:212-219) of layers given as dicts
        {name, pattern (0 dense, 1 1:4, 2 2:4), quant (bool), w [rows x cols]
        f32, mask (bitmap or None), group}."""
        assert self.which == "reference"
        n = len(layers)
        names = (C.c_char_p * n)(*[l["name"].encode() for l in layers])
        pats = (C.c_uint8 * n)(*[l["pattern"] for l in layers])
        quant = (C.c_uint8 * n)(*[1 if l["quant"] else 0 for l in layers])
        rows = (C.c_uint32 * n)(*[l["w"].shape[0] for l in layers])
        cols = (C.c_uint32 * n)(*[l["w"].shape[1] for l in layers])
        ws = [np.ascontiguousarray(l["w"], np.float32) for l in layers]
        ms = [None if l.get("mask") is None else np.ascontiguousarray(l["mask"], np.uint8) for l in layers]
        wp = (_f32p * n)(*[_ptr(w, _f32p) for w in ws])
        mp = (_u8p * n)(*[_ptr(m, _u8p) if m is not None else _u8p() for m in ms])
        groups = (C.c_uint32 * n)(*[l.get("group", 32) for l in layers])
        cap = sum(w.size * 6 for w in ws) + 4096
        buf = np.zeros(cap, np.uint8)
        ln = C.c_size_t()
        self.lib.ref_egtq_serialize.restype = C.c_int
        self._check(self.lib.ref_egtq_serialize(n, names, pats, quant, rows, cols, wp, mp, groups, _ptr(buf, _u8p),
                                                C.c_size_t(cap), C.byref(ln)))
        return bytes(buf[: ln.value])

    def ref_egtq_parse(self, data: bytes) -> int:
        """parse_compressed (egtq_io.cpp:221-235): layer count or OracleError."""
        assert self.which == "reference"
        arr = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        n = C.c_uint32()
        self.lib.ref_egtq_parse.restype = C.c_int
        self._check(self.lib.ref_egtq_parse(_ptr(arr, _u8p), C.c_size_t(len(data)), C.byref(n)))
        return n.value

    def ref_bench_spmv(self, rows: int, cols: int, reps: int, seed: int):
        assert self.which == "reference"
        med = (C.c_uint64 * 4)()
        p95 = (C.c_uint64 * 4)()
        by = (C.c_uint64 * 4)()
        self._check(self.lib.ref_bench_spmv(rows, cols, reps, C.c_uint64(seed), med, p95, by))
        return list(med), list(p95), list(by)


# ---------------------------------------------------------------- input generators
def random_nm_mask(rng: np.random.Generator, rows: int, cols: int, n: int) -> np.ndarray:
    """Exactly n kept per aligned group of 4 (test_packed.cpp:38-52 semantics)."""
    g = cols // 4
    keys = rng.random((rows, g, 4))
    order = np.argsort(keys, axis=2)[:, :, :n]
    b = np.zeros((rows, g, 4), bool)
    np.put_along_axis(b, order, True, axis=2)
    return mask_from_bool(b.reshape(rows, cols))
