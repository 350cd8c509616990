"""Verify substrate on the B200: the reference's ToyTransformer forward
(model.cpp:118-202) over packed layers, prefix-tree verification
(decode.cpp:336-421) and trie-constrained decoding (decode.cpp:423-483),
through the C-ABI (egt_model_*, egt_forward, egt_verify_parallel, egt_decode).

Mixed dispatch (compress.hpp:115-148): every linear layer is one of
INT4 2:4 / INT4 1:4 (2bit-CSR), sparse-FP16 2:4 / 1:4, or dense INT4.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native as N
from .native import DecodeOptions, ModelConfig, SessionView, TrieView, VerifyOut, check, lib
from .packed import DeviceMatrix, _stream_ptr, pack, pack_f32, quantize_matrix

LAYER_PARTS = ("wq", "wk", "wv", "wo", "ff1", "ff2")  # linear_layer_names, model.cpp:379-388


def _lib():
    return lib()


@dataclass
class Trie:
    """PrefixTrie as parent links (node 0 = root; parents precede children)."""

    token: np.ndarray
    parent: np.ndarray
    payload: np.ndarray

    def view(self) -> TrieView:
        t = np.ascontiguousarray(self.token, np.uint32)
        p = np.ascontiguousarray(self.parent, np.uint32)
        q = np.ascontiguousarray(self.payload, np.int64)
        v = TrieView(t.size, t.ctypes.data_as(N.u32p), p.ctypes.data_as(N.u32p), q.ctypes.data_as(C.POINTER(C.c_int64)))
        v._keep = (t, p, q)
        return v

    def children(self, i: int) -> list[int]:
        ch = [j for j in range(1, len(self.token)) if self.parent[j] == i]
        return sorted(ch, key=lambda j: int(self.token[j]))


@dataclass
class Beam:
    tokens: list
    log_prob: float = 0.0
    node: int = 0


def _verify_out(beam_size: int, stride: int):
    arrs = dict(score=np.zeros(beam_size, np.float64), payload=np.zeros(beam_size, np.int64),
                beam=np.zeros(beam_size, np.uint32), len=np.zeros(beam_size, np.uint32),
                tokens=np.zeros(beam_size * stride, np.int32))
    o = VerifyOut(0, arrs["score"].ctypes.data_as(N.f64p), arrs["payload"].ctypes.data_as(C.POINTER(C.c_int64)),
                  arrs["beam"].ctypes.data_as(N.u32p), arrs["len"].ctypes.data_as(N.u32p),
                  arrs["tokens"].ctypes.data_as(C.POINTER(C.c_int32)), stride, 0, 0)
    return o, arrs


def _read_out(o, arrs, stride):
    res = []
    for j in range(o.n_selected):
        n = int(arrs["len"][j])
        res.append({"tokens": arrs["tokens"][j * stride: j * stride + n].tolist(), "score": float(arrs["score"][j]),
                    "payload": int(arrs["payload"][j]), "beam": int(arrs["beam"][j])})
    return res


class DeviceModel:
    """ToyTransformer (model.hpp:53-59) with every linear layer resident as a
    packed device matrix.  layers: n_layers*6 DeviceMatrix (wq wk wv wo ff1
    ff2), head: DeviceMatrix [vocab x d]."""

    def __init__(self, cfg: dict, embedding: np.ndarray, layers: list, head: DeviceMatrix, stream=None):
        L = _lib()
        self.cfg = dict(cfg)
        self.layers = list(layers)
        self.head = head
        c = ModelConfig(*(int(cfg[k]) for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_ff",
                                                "max_positions")))
        emb = np.ascontiguousarray(embedding, np.float32)
        hs = (C.c_void_p * len(self.layers))(*[d.handle.value for d in self.layers])
        h = C.c_void_p()
        check(L.egt_model_create(C.byref(c), emb.ctypes.data_as(N.f32p), hs, head.handle, _stream_ptr(stream),
                                 C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_model_destroy(h)
            self._h = C.c_void_p()

    def forward(self, tokens, positions, mask: np.ndarray, stream=None):
        """forward (model.hpp:71-72): logits [M x vocab] (torch CUDA tensor).
        mask: bool [M x M], mask[q, k] = query q sees key k."""
        import torch

        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int32)
        bits = np.packbits(np.ascontiguousarray(mask, bool).reshape(-1), bitorder="little")
        out = torch.empty((t.size, self.cfg["vocab_size"]), dtype=torch.float32, device="cuda")
        check(_lib().egt_forward(self._h, t.ctypes.data_as(C.POINTER(C.c_int32)), p.ctypes.data_as(C.POINTER(C.c_int32)),
                                 bits.ctypes.data_as(N.u8p) if bits.size else None, t.size, C.c_void_p(out.data_ptr()),
                                 _stream_ptr(stream)))
        return out

    def forward_tree(self, tokens, positions, committed_len, padded_len: int, parent, beam, stream=None):
        """forward with the prefix-tree mask built on the device from the
        compact encoding (egt_forward_tree): committed blocks of padded_len rows
        per beam, then one row per flattened node (parent index, beam)."""
        import torch

        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int32)
        cl = np.ascontiguousarray(committed_len, np.uint32)
        par = np.ascontiguousarray(parent, np.int32)
        bm = np.ascontiguousarray(beam, np.uint32)
        view = N.TreeView(cl.size, padded_len, cl.ctypes.data_as(N.u32p), par.size,
                          par.ctypes.data_as(C.POINTER(C.c_int32)), bm.ctypes.data_as(N.u32p))
        out = torch.empty((t.size, self.cfg["vocab_size"]), dtype=torch.float32, device="cuda")
        check(_lib().egt_forward_tree(self._h, t.ctypes.data_as(C.POINTER(C.c_int32)),
                                      p.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(view),
                                      C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def verify_parallel(self, trie: Trie, prompt, beams: list, beam_size: int, stream=None):
        """flatten_subtree + build_tree_mask + verify_parallel (decode.cpp:209-421)."""
        tv = trie.view()
        pr = np.ascontiguousarray(prompt, np.int32)
        bn = np.array([b.node for b in beams], np.uint32)
        bl = np.array([b.log_prob for b in beams], np.float64)
        blen = np.array([len(b.tokens) for b in beams], np.uint32)
        btok = np.array([t for b in beams for t in b.tokens] or [0], np.int32)
        sv = SessionView(pr.ctypes.data_as(C.POINTER(C.c_int32)), pr.size, len(beams), bn.ctypes.data_as(N.u32p),
                         bl.ctypes.data_as(N.f64p), blen.ctypes.data_as(N.u32p),
                         btok.ctypes.data_as(C.POINTER(C.c_int32)))
        stride = 64
        o, arrs = _verify_out(beam_size, stride)
        check(_lib().egt_verify_parallel(self._h, C.byref(tv), C.byref(sv), beam_size, C.byref(o), _stream_ptr(stream)))
        return _read_out(o, arrs, stride), {"flattened_nodes": o.flattened_nodes, "rows": o.rows}

    def decode(self, trie: Trie, prompt, beam_size=4, mode="ptpv", forced_depth=0, cost=(0.0, 0.0, 0.0),
               node_cap=4096, kv_cache=False, stream=None):
        """decode (decode.cpp:423-483); mode: autoregressive | ptpv | forced.
        kv_cache: constrained steps on a KV pool (one new row per beam per step)."""
        tv = trie.view()
        pr = np.ascontiguousarray(prompt, np.int32)
        m = {"autoregressive": 0, "ptpv": 1, "forced": 2}[mode]
        opt = DecodeOptions(beam_size, m, forced_depth, cost[0], cost[1], cost[2], node_cap, 1 if kv_cache else 0)
        stride = 64
        o, arrs = _verify_out(beam_size, stride)
        stats = (C.c_int32 * 4)()
        check(_lib().egt_decode(self._h, C.byref(tv), pr.ctypes.data_as(C.POINTER(C.c_int32)), pr.size, C.byref(opt),
                                C.byref(o), stats, _stream_ptr(stream)))
        return _read_out(o, arrs, stride), {"steps": stats[0], "forward_passes": stats[1],
                                            "trigger_step": stats[2], "flattened_nodes": stats[3]}


class Decoder:
    """KV-cached batch-1 greedy decode loop on the device (egt_decoder_*):
    one CUDA graph replay per token, position and token device-resident."""

    def __init__(self, model: DeviceModel, max_len: int):
        self.model = model
        self.max_len = max_len
        h = C.c_void_p()
        check(_lib().egt_decoder_create(model._h, max_len, C.byref(h)))
        self._h = h

    def start(self, prompt, stream=None) -> None:
        pr = np.ascontiguousarray(prompt, np.int32)
        check(_lib().egt_decoder_start(self._h, pr.ctypes.data_as(C.POINTER(C.c_int32)), pr.size,
                                       _stream_ptr(stream)))

    def step(self, n: int = 1, stream=None) -> None:
        """n tokens (asynchronous, stream-ordered)."""
        check(_lib().egt_decoder_step(self._h, n, _stream_ptr(stream)))

    def read(self, logits=None, stream=None):
        """(tokens at positions [0, position], position); logits: optional
        torch CUDA tensor [vocab] receiving the last step's logits."""
        toks = np.zeros(self.max_len, np.int32)
        pos = C.c_uint32()
        check(_lib().egt_decoder_read(self._h, toks.ctypes.data_as(C.POINTER(C.c_int32)), self.max_len,
                                      C.byref(pos), C.c_void_p(logits.data_ptr()) if logits is not None else None,
                                      _stream_ptr(stream)))
        return toks[: min(pos.value + 1, self.max_len)], pos.value

    def generate(self, prompt, n_new: int, stream=None):
        """Greedy continuation: prompt + n_new tokens (host list)."""
        self.start(prompt, stream)
        self.step(len(prompt) - 1 + n_new, stream)
        toks, pos = self.read(stream=stream)
        return toks.tolist()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and N is not None and N._lib is not None:
            N._lib.egt_decoder_destroy(h)
            self._h = C.c_void_p()


def compress_layer(w: np.ndarray, kind: str, group: int):
    """One mixed-dispatch layer from dense weights: kind in {int4-2:4, int4-1:4,
    int4-dense, fp16-2:4, fp16-1:4}.  Masks keep the largest |w| per group of
    4 (magnitude_mask semantics, packed.cpp:245-264, ties to the lower column).
    Returns (DeviceMatrix, host artifact): the PackedSparseMatrix, or the
    all-kept QuantizedMatrix for dense INT4."""
    rows, cols = w.shape
    if kind == "int4-dense":
        q = quantize_matrix(w, group)
        return DeviceMatrix.dense_i4(q), q
    n = 2 if kind.endswith("2:4") else 1
    a = np.abs(w.reshape(rows, cols // 4, 4))
    order = np.argsort(-a, axis=2, kind="stable")[:, :, :n]
    keep = np.zeros_like(a, dtype=bool)
    np.put_along_axis(keep, order, True, axis=2)
    mask = np.packbits(keep.reshape(-1), bitorder="little")
    if kind.startswith("int4"):
        p = pack(mask, quantize_matrix(w, group, mask), n)
    else:
        p = pack_f32(mask, w.astype(np.float16).astype(np.float32), n)
    return DeviceMatrix.from_packed(p), p
