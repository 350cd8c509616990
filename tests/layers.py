"""Seeded synthetic layers for the parity tests: the same inputs go through the
product (C++ encoder + CUDA) and through the oracle (oracle/egt_oracle.c)."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Oracle, Packed, random_nm_mask


def make_int4(rng, rows, cols, n, group, port: Oracle):
    """W ~ U(-1,1), exact-N mask, group-wise INT4 (compress.cpp:157-197).
    group: int, or a per-row array.  Returns (oracle Packed, mask, w)."""
    w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
    mask = random_nm_mask(rng, rows, cols, n)
    gs = np.broadcast_to(np.asarray(group, np.uint32), (rows,)).copy()
    q = port.quantize(w, gs, mask)
    return port.pack_int4(mask, rows, cols, q, n), mask, w


def make_f16(rng, rows, cols, n, port: Oracle):
    """Sparse-FP layer with fp16-representable values (lossless FP16 storage)."""
    w = rng.uniform(-1, 1, (rows, cols)).astype(np.float16).astype(np.float32)
    mask = random_nm_mask(rng, rows, cols, n)
    return port.pack_f32(mask, rows, cols, w, n), mask, w


def to_product(p: Packed):
    from paper_2605_11582_b200.packed import PackedSparseMatrix

    return PackedSparseMatrix(p.n, p.m, p.rows, p.cols, p.kind, p.index_words, p.value_bytes, p.group_sizes,
                              p.group_offsets, p.scales, p.zero_points, p.values)


def close(got, want, tol=1e-3):
    """The reference's convention |got - want| <= tol * (1 + |want|)
    (test_packed.cpp:279, acceptance_main.cpp:177-179)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    err = np.abs(got - want) / (1.0 + np.abs(want))
    return bool(np.all(err <= tol)), float(err.max(initial=0.0))
