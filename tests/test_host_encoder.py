"""CPU tests of the product's host side: the C++ encoder behind the C-ABI is
byte-identical to the reference (golden vectors from the unmodified reference
sources, and the oracle), the error contract matches, and the shared library
exports every symbol include/egt_b200.h declares.  No GPU calls."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_vectors.npz")


@pytest.fixture(scope="module")
def egt():
    from paper_2605_11582_b200 import _build

    _build.build()
    import paper_2605_11582_b200 as egt

    return egt


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "egt_b200.h")).read()
    return sorted(set(re.findall(r"EGT_API\s+[\w\s\*]+?\b(egt_\w+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol(egt):
    import ctypes

    from paper_2605_11582_b200 import native

    L = ctypes.CDLL(native.LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(native.SIGNATURES), set(syms) ^ set(native.SIGNATURES)
    assert native.lib().egt_abi_version() == 1


def test_library_is_sm100a_only(egt):
    import subprocess

    from paper_2605_11582_b200 import native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", native.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "HMMA.SP.16832.F32" in sass  # the tensor-core 2:4 gather


def _cases():
    g = np.load(GOLDEN)
    for i in range(int(g["n_cases"])):
        yield i, {k[len(f"c{i}_"):]: g[k] for k in g.files if k.startswith(f"c{i}_")}


def test_encoder_matches_reference_golden(egt):
    for i, c in _cases():
        rows, cols, n, quant, dense_codes = (int(v) for v in c["meta"])
        if quant:
            q = egt.quantize_matrix(c["w"], c["group_sizes"], None if dense_codes else c["mask"])
            assert np.array_equal(q.group_offsets, c["group_offsets"]), i
            assert np.array_equal(q.scales.view(np.uint32), c["scales"].view(np.uint32)), i
            assert np.array_equal(q.zero_points, c["zero_points"]), i
            assert np.array_equal(q.codes, c["codes"]), i
            p = egt.pack(c["mask"], q, n)
            assert np.array_equal(p.value_bytes, c["value_bytes"]), i
        else:
            p = egt.pack_f32(c["mask"], c["w"], n)
            assert np.array_equal(p.values.view(np.uint32), c["values"].view(np.uint32)), i
        assert np.array_equal(p.index_words, c["index_words"]), i
        f = egt.footprint(p)
        assert [f[k] for k in ("index_bytes", "value_bytes", "scale_bytes", "packed_bytes",
                               "baseline_bytes")] == c["footprint"].tolist(), i


def test_encoder_matches_oracle_fuzz(egt, port):
    from oracle.oracle import random_nm_mask

    rng = np.random.default_rng(99)
    for _ in range(60):
        rows, cols, n = int(rng.integers(1, 10)), 4 * int(rng.integers(1, 48)), int(rng.integers(1, 3))
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        m = random_nm_mask(rng, rows, cols, n)
        gs = rng.choice([4, 8, 16, 32, 64, 128, 256], rows).astype(np.uint32)
        q, qo = egt.quantize_matrix(w, gs, m), port.quantize(w, gs, m)
        assert np.array_equal(q.codes, qo.codes)
        assert np.array_equal(q.scales.view(np.uint32), qo.scales.view(np.uint32))
        assert np.array_equal(q.zero_points, qo.zero_points)
        p, po = egt.pack(m, q, n), port.pack_int4(m, rows, cols, qo, n)
        assert np.array_equal(p.index_words, po.index_words)
        assert np.array_equal(p.value_bytes, po.value_bytes)


def test_group_fit_known_answers(egt):
    s, z = egt.fit_group([0.0, 1.0, 2.0, 3.0])
    assert np.float32(s) == np.float32(0.2) and z == 0
    s, z = egt.fit_group([-1.0, 1.0])
    assert z == 8
    s, z = egt.fit_group([])
    assert np.float32(s) == np.float32(1e-8) and z == 0


def test_worked_index_word(egt):
    from oracle.oracle import mask_from_bool

    b = np.zeros((1, 8), bool)
    b[0, [1, 3, 4, 6]] = True
    p = egt.pack_f32(mask_from_bool(b), np.ones((1, 8), np.float32), 2)
    assert p.index_words.tolist() == [0x7200]


def test_encoder_error_contract(egt):
    from oracle.oracle import random_nm_mask

    from paper_2605_11582_b200 import InvalidArgument

    rng = np.random.default_rng(5)
    w = rng.uniform(-1, 1, (2, 8)).astype(np.float32)
    m = random_nm_mask(rng, 2, 8, 2)
    with pytest.raises(InvalidArgument, match="dense"):
        egt.pack_f32(m, w, 4)
    rag = m.copy()
    rag[0] ^= 1
    with pytest.raises(InvalidArgument, match="keeps"):
        egt.pack_f32(rag, w, 2)
    with pytest.raises(InvalidArgument, match="zero group size"):
        egt.quantize_matrix(w, [0, 4])
    f = egt.footprint(egt.pack(m, egt.quantize_matrix(w, [8, 8], m), 2))
    assert f["packed_bytes"] == f["index_bytes"] + f["value_bytes"] + f["scale_bytes"]
