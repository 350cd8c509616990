"""Planning around the hot path (include/egt_b200.h, csrc/host/planning.cpp):
layer-adaptive sparsity (plan_sparsity, compress.cpp:298-326), the decode
cost model (CostModelEstimator, decode.cpp:84-120) fed device-measured
times, and the trigger / tree-mask builders on host views
(decode.cpp:192-299)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N
from .native import SessionView, TrieView, check, lib
from .packed import _stream_ptr

PATTERN = {0: "dense", 1: "1:4", 2: "2:4"}


def plan_sparsity(scores, weights, rho_s: float) -> list:
    """Per layer 2 (2:4) for the ceil(rho_s * L) layers of highest
    mean(score) / mean(|w|), 1 (1:4) for the rest."""
    n = len(scores)
    ss = [np.ascontiguousarray(s, np.float32) for s in scores]
    ws = [np.ascontiguousarray(w, np.float32) for w in weights]
    rows = (C.c_uint32 * max(1, n))(*[s.shape[0] for s in ss])
    cols = (C.c_uint32 * max(1, n))(*[s.shape[1] for s in ss])
    sp = (N.f32p * max(1, n))(*[s.ctypes.data_as(N.f32p) for s in ss])
    wp = (N.f32p * max(1, n))(*[w.ctypes.data_as(N.f32p) for w in ws])
    out = np.zeros(max(1, n), np.uint8)
    check(lib().egt_host_plan_sparsity(n, rows, cols, sp, wp, C.c_double(rho_s), out.ctypes.data_as(N.u8p)))
    return out[:n].tolist()


class CostModelEstimator:
    """decode.cpp:84-120: EMA 0.9 of step seconds, 32-sample least squares of
    verify seconds over node count."""

    def __init__(self, t_step: float = 0.0, alpha: float = 0.0, beta: float = 0.0):
        h = C.c_void_p()
        check(lib().egt_cost_estimator_create(t_step, alpha, beta, C.byref(h)))
        self._h = h

    def observe_step(self, seconds: float) -> None:
        check(lib().egt_cost_estimator_observe_step(self._h, seconds))

    def observe_verify(self, nodes: int, seconds: float) -> None:
        check(lib().egt_cost_estimator_observe_verify(self._h, nodes, seconds))

    def model(self) -> tuple:
        out = (C.c_double * 3)()
        check(lib().egt_cost_estimator_model(self._h, out))
        return tuple(out)

    def measure(self, model, prompt_len: int, n_beams: int, node_counts, reps: int = 3, stream=None) -> tuple:
        """Feed device-measured (CUDA event) forward times of `model`
        (a DeviceModel): one constrained step, one verify pass per node count."""
        nc = np.ascontiguousarray(node_counts, np.uint32)
        check(lib().egt_measure_cost_model(model._h, prompt_len, n_beams, nc.ctypes.data_as(N.u32p), nc.size, reps,
                                           self._h, _stream_ptr(stream)))
        return self.model()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_cost_estimator_destroy(h)
            self._h = C.c_void_p()


def _session(prompt, beams):
    pr = np.ascontiguousarray(prompt, np.int32)
    bn = np.array([b.node for b in beams], np.uint32)
    bl = np.array([b.log_prob for b in beams], np.float64)
    blen = np.array([len(b.tokens) for b in beams], np.uint32)
    btok = np.array([t for b in beams for t in b.tokens] or [0], np.int32)
    v = SessionView(pr.ctypes.data_as(C.POINTER(C.c_int32)), pr.size, len(beams), bn.ctypes.data_as(N.u32p),
                    bl.ctypes.data_as(N.f64p), blen.ctypes.data_as(N.u32p), btok.ctypes.data_as(C.POINTER(C.c_int32)))
    v._keep = (pr, bn, bl, blen, btok)
    return v


def estimate_trigger(trie, prompt, beams, cost, node_cap: int = 4096):
    """estimate_trigger (decode.cpp:192-207): (trigger, predicted saving)."""
    tv = trie.view()
    sv = _session(prompt, beams)
    trig, sav = C.c_int(), C.c_double()
    check(lib().egt_host_estimate_trigger(C.byref(tv), C.byref(sv), cost[0], cost[1], cost[2], node_cap,
                                          C.byref(trig), C.byref(sav)))
    return bool(trig.value), sav.value


def tree_mask(trie, prompt, beams):
    """flatten_subtree + build_tree_mask (decode.cpp:209-299): (flat node
    arrays, visibility bool [R x R], tokens, positions, padded_len,
    flat_offset)."""
    tv = trie.view()
    sv = _session(prompt, beams)
    capn = max(1, len(trie.token) * max(1, len(beams)))
    lmax = len(prompt) + max((len(b.tokens) for b in beams), default=0)
    capr = len(beams) * lmax + capn
    capb = (capr * capr + 7) // 8
    nn, nr, pl, fo = C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    ft, fp, fd, ftr, fb = (np.zeros(capn, np.uint32), np.zeros(capn, np.int32), np.zeros(capn, np.uint32),
                           np.zeros(capn, np.uint32), np.zeros(capn, np.uint32))
    toks, pos, bits = np.zeros(capr, np.int32), np.zeros(capr, np.int32), np.zeros(capb, np.uint8)
    i32 = C.POINTER(C.c_int32)
    check(lib().egt_host_tree_mask(C.byref(tv), C.byref(sv), capn, C.byref(nn), ft.ctypes.data_as(N.u32p),
                                   fp.ctypes.data_as(i32), fd.ctypes.data_as(N.u32p), ftr.ctypes.data_as(N.u32p),
                                   fb.ctypes.data_as(N.u32p), capr, C.byref(nr), toks.ctypes.data_as(i32),
                                   pos.ctypes.data_as(i32), bits.ctypes.data_as(N.u8p), capb, C.byref(pl),
                                   C.byref(fo)))
    n, R = nn.value, nr.value
    flat = dict(token=ft[:n], parent=fp[:n], depth=fd[:n], trie_node=ftr[:n], beam=fb[:n])
    vis = np.unpackbits(bits, bitorder="little")[: R * R].reshape(R, R).astype(bool)
    return flat, vis, toks[:R], pos[:R], pl.value, fo.value
