"""ctypes bindings to the reference's OWN model / decoder code (model.cpp,
decode.cpp and compress.cpp's plan_sparsity, compiled unmodified into
oracle/_ref/libegt_ref.so by oracle/build_ref.sh; wrappers in
oracle/ref/ref_model_capi.cpp).  TEST INFRASTRUCTURE ONLY: the pinned oracle
of the verify path (forward model.cpp:118-202, verify_parallel
decode.cpp:336-421, decode decode.cpp:423-483, constrained_step
decode.cpp:122-190, estimate_trigger decode.cpp:192-207, CostModelEstimator
decode.cpp:84-120, plan_sparsity compress.cpp:298-326).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs use it."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .oracle import REF_LIB, OracleError

_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)
PARTS = ("wq", "wk", "wv", "wo", "ff1", "ff2")


class _Cfg(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_positions")]


class _Trie(C.Structure):
    _fields_ = [("n_nodes", C.c_uint32), ("token", _u32p), ("parent", _u32p), ("payload", _i64p)]


class _Session(C.Structure):
    _fields_ = [("prompt", _i32p), ("prompt_len", C.c_uint32), ("n_beams", C.c_uint32), ("beam_node", _u32p),
                ("beam_log_prob", _f64p), ("beam_len", _u32p), ("beam_tokens", _i32p)]


class _Out(C.Structure):
    _fields_ = [("n_selected", C.c_uint32), ("score", _f64p), ("payload", _i64p), ("beam", _u32p),
                ("len", _u32p), ("tokens", _i32p), ("tokens_stride", C.c_uint32), ("flattened_nodes", C.c_uint32),
                ("rows", C.c_uint32)]


class _Opt(C.Structure):
    _fields_ = [("beam_size", C.c_int), ("mode", C.c_int), ("forced_depth", C.c_int), ("t_step", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double), ("node_cap", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(f"{REF_LIB} missing: run oracle/build_ref.sh")
        L = C.CDLL(REF_LIB)
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_new.restype = C.c_void_p
        L.ref_model_new.argtypes = [C.POINTER(_Cfg), _f32p, C.POINTER(_f32p), _f32p]
        L.ref_model_free.argtypes = [C.c_void_p]
        for fn in ("ref_forward", "ref_verify_parallel", "ref_decode", "ref_tree_mask", "ref_constrained_steps",
                   "ref_estimate_trigger", "ref_cost_estimator", "ref_plan_sparsity", "ref_model_positions",
                   "ref_log_softmax"):
            getattr(L, fn).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().ref_last_error().decode(errors="replace"))


def _p(a, t):
    return a.ctypes.data_as(t)


def trie_view(token, parent, payload):
    t = np.ascontiguousarray(token, np.uint32)
    p = np.ascontiguousarray(parent, np.uint32)
    q = np.ascontiguousarray(payload, np.int64)
    v = _Trie(t.size, _p(t, _u32p), _p(p, _u32p), _p(q, _i64p))
    v._keep = (t, p, q)
    return v


def session_view(prompt, beams):
    """beams: objects with .tokens, .log_prob, .node (model.Beam) or dicts."""
    def g(b, k):
        return b[k] if isinstance(b, dict) else getattr(b, k)

    pr = np.ascontiguousarray(prompt, np.int32)
    bn = np.array([g(b, "node") for b in beams], np.uint32)
    bl = np.array([g(b, "log_prob") for b in beams], np.float64)
    blen = np.array([len(g(b, "tokens")) for b in beams], np.uint32)
    btok = np.array([t for b in beams for t in g(b, "tokens")] or [0], np.int32)
    v = _Session(_p(pr, _i32p), pr.size, len(beams), _p(bn, _u32p), _p(bl, _f64p), _p(blen, _u32p), _p(btok, _i32p))
    v._keep = (pr, bn, bl, blen, btok)
    return v


def _out(beam_size, stride=64):
    a = dict(score=np.zeros(beam_size, np.float64), payload=np.zeros(beam_size, np.int64),
             beam=np.zeros(beam_size, np.uint32), len=np.zeros(beam_size, np.uint32),
             tokens=np.zeros(max(1, beam_size) * stride, np.int32))
    o = _Out(0, _p(a["score"], _f64p), _p(a["payload"], _i64p), _p(a["beam"], _u32p), _p(a["len"], _u32p),
             _p(a["tokens"], _i32p), stride, 0, 0)
    return o, a


def _read(o, a, stride=64):
    res = []
    for j in range(o.n_selected):
        n = int(a["len"][j])
        res.append({"tokens": a["tokens"][j * stride: j * stride + n].tolist(), "score": float(a["score"][j]),
                    "payload": int(a["payload"][j]), "beam": int(a["beam"][j])})
    return res


class RefModel:
    """The reference's ToyTransformer (model.hpp:53-59) over given dense f32
    weights; layers: list of dicts wq..ff2 (row-major [out x in])."""

    def __init__(self, cfg: dict, embedding, layers, head):
        L = lib()
        self.cfg = dict(cfg)
        c = _Cfg(*(int(cfg[k]) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff", "max_positions")))
        keep = []
        ptrs = (_f32p * (6 * len(layers)))()
        for li, lw in enumerate(layers):
            for j, name in enumerate(PARTS):
                a = np.ascontiguousarray(lw[name], np.float32)
                keep.append(a)
                ptrs[6 * li + j] = _p(a, _f32p)
        emb = np.ascontiguousarray(embedding, np.float32)
        hd = np.ascontiguousarray(head, np.float32)
        h = L.ref_model_new(C.byref(c), _p(emb, _f32p), ptrs, _p(hd, _f32p))
        if not h:
            raise OracleError(1, L.ref_last_error().decode(errors="replace"))
        self._h = C.c_void_p(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.ref_model_free(h)
            self._h = C.c_void_p()

    def positions(self) -> np.ndarray:
        out = np.zeros((self.cfg["max_positions"], self.cfg["d_model"]), np.float32)
        _check(lib().ref_model_positions(self._h, _p(out, _f32p)))
        return out

    def forward(self, tokens, positions, mask) -> np.ndarray:
        """forward (model.cpp:358-361): logits [M x vocab]; mask bool [M x M]."""
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int32)
        bits = np.packbits(np.ascontiguousarray(mask, bool).reshape(-1), bitorder="little")
        out = np.zeros((t.size, self.cfg["vocab_size"]), np.float32)
        _check(lib().ref_forward(self._h, _p(t, _i32p), _p(p, _i32p), _p(bits, _u8p), t.size, _p(out, _f32p)))
        return out

    def verify_parallel(self, trie, prompt, beams, beam_size: int):
        """flatten_subtree + build_tree_mask + verify_parallel (decode.cpp:209-421):
        (selected leaves, node scores, info)."""
        tv = trie_view(trie.token, trie.parent, trie.payload)
        sv = session_view(prompt, beams)
        o, a = _out(beam_size)
        cap = 1 << 16
        ns = np.zeros(cap, np.float64)
        _check(lib().ref_verify_parallel(self._h, C.byref(tv), C.byref(sv), beam_size, C.byref(o), _p(ns, _f64p), cap))
        return _read(o, a), ns[: o.flattened_nodes], {"flattened_nodes": o.flattened_nodes, "rows": o.rows}

    def decode(self, trie, prompt, beam_size=4, mode="ptpv", forced_depth=0, cost=(0.0, 0.0, 0.0), node_cap=4096):
        """decode (decode.cpp:423-483); mode: autoregressive | ptpv | forced."""
        tv = trie_view(trie.token, trie.parent, trie.payload)
        pr = np.ascontiguousarray(prompt, np.int32)
        m = {"autoregressive": 0, "ptpv": 1, "forced": 2}[mode]
        opt = _Opt(beam_size, m, forced_depth, cost[0], cost[1], cost[2], node_cap)
        o, a = _out(beam_size)
        st = (C.c_int32 * 4)()
        _check(lib().ref_decode(self._h, C.byref(tv), _p(pr, _i32p), pr.size, C.byref(opt), C.byref(o), st))
        return _read(o, a), {"steps": st[0], "forward_passes": st[1], "trigger_step": st[2],
                             "flattened_nodes": st[3]}

    def constrained_steps(self, trie, prompt, beams, beam_size: int, n_steps: int = 1, stride: int = 64):
        """constrained_step (decode.cpp:122-190) n_steps times: the new beams
        as dicts {tokens, log_prob, node}, best first."""
        tv = trie_view(trie.token, trie.parent, trie.payload)
        sv = session_view(prompt, beams)
        cap = max(64, beam_size * 4)
        nb = C.c_uint32()
        node = np.zeros(cap, np.uint32)
        lp = np.zeros(cap, np.float64)
        ln = np.zeros(cap, np.uint32)
        tk = np.zeros(cap * stride, np.int32)
        _check(lib().ref_constrained_steps(self._h, C.byref(tv), C.byref(sv), beam_size, n_steps, cap, stride,
                                           C.byref(nb), _p(node, _u32p), _p(lp, _f64p), _p(ln, _u32p), _p(tk, _i32p)))
        return [{"tokens": tk[b * stride: b * stride + int(ln[b])].tolist(), "log_prob": float(lp[b]),
                 "node": int(node[b])} for b in range(nb.value)]


def tree_mask(trie, prompt, beams):
    """flatten_subtree + build_tree_mask (decode.cpp:209-299) by the reference:
    (flat nodes as dict of arrays, vis bool [R x R], tokens, positions,
    padded_len, flat_offset)."""
    tv = trie_view(trie.token, trie.parent, trie.payload)
    sv = session_view(prompt, beams)
    capn, capr = 1 << 14, 1 << 14
    nn, nr, pl, fo = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    ft, fpar, fd, ftr, fb = (np.zeros(capn, np.uint32), np.zeros(capn, np.int32), np.zeros(capn, np.uint32),
                             np.zeros(capn, np.uint32), np.zeros(capn, np.uint32))
    toks, pos = np.zeros(capr, np.int32), np.zeros(capr, np.int32)
    # the visibility buffer is sized after a first call reports the row count
    vis = np.zeros(1, np.uint8)
    rc = lib().ref_tree_mask(C.byref(tv), C.byref(sv), capn, C.byref(nn), _p(ft, _u32p), _p(fpar, _i32p),
                             _p(fd, _u32p), _p(ftr, _u32p), _p(fb, _u32p), 0, C.byref(nr), _p(toks, _i32p),
                             _p(pos, _i32p), _p(vis, _u8p), C.byref(pl), C.byref(fo))
    R = nr.value
    vis = np.zeros((R * R + 7) // 8 + 1, np.uint8)
    _check(lib().ref_tree_mask(C.byref(tv), C.byref(sv), capn, C.byref(nn), _p(ft, _u32p), _p(fpar, _i32p),
                               _p(fd, _u32p), _p(ftr, _u32p), _p(fb, _u32p), R, C.byref(nr), _p(toks, _i32p),
                               _p(pos, _i32p), _p(vis, _u8p), C.byref(pl), C.byref(fo)))
    del rc
    n = nn.value
    flat = dict(token=ft[:n].copy(), parent=fpar[:n].copy(), depth=fd[:n].copy(), trie_node=ftr[:n].copy(),
                beam=fb[:n].copy())
    v = np.unpackbits(vis, bitorder="little")[: R * R].reshape(R, R).astype(bool)
    return flat, v, toks[:R].copy(), pos[:R].copy(), pl.value, fo.value


def estimate_trigger(trie, prompt, beams, cost, node_cap=4096):
    """estimate_trigger (decode.cpp:192-207): (trigger, predicted_saving)."""
    tv = trie_view(trie.token, trie.parent, trie.payload)
    sv = session_view(prompt, beams)
    trig, sav = C.c_int(), C.c_double()
    _check(lib().ref_estimate_trigger(C.byref(tv), C.byref(sv), C.c_double(cost[0]), C.c_double(cost[1]),
                                      C.c_double(cost[2]), C.c_uint64(node_cap), C.byref(trig), C.byref(sav)))
    return bool(trig.value), sav.value


def cost_estimator(observations, initial=(0.0, 0.0, 0.0)):
    """CostModelEstimator (decode.cpp:84-120) fed observations
    [("step", seconds) | ("verify", nodes, seconds)]: (t_step, alpha, beta)."""
    n = len(observations)
    kind = (C.c_int * max(1, n))(*[0 if o[0] == "step" else 1 for o in observations])
    nodes = (C.c_uint64 * max(1, n))(*[0 if o[0] == "step" else int(o[1]) for o in observations])
    secs = (C.c_double * max(1, n))(*[float(o[-1]) for o in observations])
    out = (C.c_double * 3)()
    _check(lib().ref_cost_estimator(n, kind, nodes, secs, C.c_double(initial[0]), C.c_double(initial[1]),
                                    C.c_double(initial[2]), out))
    return tuple(out)


def plan_sparsity(scores, weights, rho_s: float) -> list:
    """plan_sparsity (compress.cpp:298-326): per layer 1 (1:4) or 2 (2:4)."""
    n = len(scores)
    ss = [np.ascontiguousarray(s, np.float32) for s in scores]
    ws = [np.ascontiguousarray(w, np.float32) for w in weights]
    rows = (C.c_uint32 * n)(*[s.shape[0] for s in ss])
    cols = (C.c_uint32 * n)(*[s.shape[1] for s in ss])
    sp = (_f32p * n)(*[_p(s, _f32p) for s in ss])
    wp = (_f32p * n)(*[_p(w, _f32p) for w in ws])
    out = np.zeros(n, np.uint8)
    _check(lib().ref_plan_sparsity(n, rows, cols, sp, wp, C.c_double(rho_s), _p(out, _u8p)))
    return out.tolist()
