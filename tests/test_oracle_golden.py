"""Pins the oracle (oracle/egt_oracle.c) before anything is checked against it.

1. The reference's own known-answer tests, restated:
   test_packed.cpp:75-91 (0x7200), :93-106 (naive bit writer), :108-128
   (nibble order), :147-179 (argument errors), :181-206 (exact round trip),
   :208-234 (malformed streams), :236-262 (hand spmv = 1.0), :264-292 (spmv vs
   dense), :294-356 (footprint); test_compress.cpp:87-127 (group fits),
   :231-256 (fit over retained values only).
2. tests/golden/ref_vectors.npz, produced by the unmodified reference sources
   (tests/golden/make_golden.py): bit-exact equality of every output.
3. When oracle/_ref is built, a live fuzz of port vs reference.
"""
import os

import numpy as np
import pytest

from oracle.oracle import OracleError, Packed, Quantized, mask_from_bool, mask_to_bool, random_nm_mask

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_vectors.npz")


def naive_index_words(mask_bits, rows, cols):
    """test_packed.cpp:56-71: two bits per kept offset, MSB of each word first."""
    b = mask_to_bool(mask_bits, rows, cols)
    bits = []
    for r in range(rows):
        for c in range(cols):
            if b[r, c]:
                off = c % 4
                bits += [(off >> 1) & 1, off & 1]
    while len(bits) % 16:
        bits.append(0)
    words = np.zeros(len(bits) // 16, np.uint16)
    for i, v in enumerate(bits):
        if v:
            words[i // 16] |= np.uint16(1 << (15 - i % 16))
    return words


def test_worked_index_example(port):
    b = np.zeros((1, 8), bool)
    b[0, [1, 3, 4, 6]] = True
    p = port.pack_f32(mask_from_bool(b), 1, 8, np.ones((1, 8), np.float32), 2)
    assert p.index_words.tolist() == [0x7200]
    assert np.array_equal(p.index_words, naive_index_words(mask_from_bool(b), 1, 8))
    assert p.nnz == 4 and p.values.tolist() == [1.0] * 4


def test_index_stream_matches_naive_writer(port):
    rng = np.random.default_rng(41)
    for n in (1, 2):
        for _ in range(20):
            rows, cols = int(rng.integers(1, 8)), 4 * int(rng.integers(1, 10))
            m = random_nm_mask(rng, rows, cols, n)
            p = port.pack_f32(m, rows, cols, rng.uniform(-1, 1, (rows, cols)).astype(np.float32), n)
            assert np.array_equal(p.index_words, naive_index_words(m, rows, cols))
            assert p.index_words.size == (p.nnz + 7) // 8


def test_nibble_order(port):
    b = np.zeros((1, 8), bool)
    b[0, [0, 1, 4, 5]] = True
    m = mask_from_bool(b)
    w = np.array([[1, 2, 0, 0, 3, 5, 0, 0]], np.float32)
    q = port.quantize(w, [8], m)
    p = port.pack_int4(m, 1, 8, q, 2)
    assert p.value_bytes.size == 2
    assert p.value_bytes[0] & 0xF == q.codes[0] and p.value_bytes[0] >> 4 == q.codes[1]
    assert p.value_bytes[1] & 0xF == q.codes[2] and p.value_bytes[1] >> 4 == q.codes[3]


def test_dense_and_kept_codes(port):
    rng = np.random.default_rng(43)
    w = rng.uniform(-1, 1, (4, 16)).astype(np.float32)
    m = random_nm_mask(rng, 4, 16, 2)
    a = port.pack_int4(m, 4, 16, port.quantize(w, [8] * 4, m), 2)
    d = port.pack_int4(m, 4, 16, port.quantize(w, [8] * 4), 2)
    assert np.array_equal(a.index_words, d.index_words)
    assert a.value_bytes.size == d.value_bytes.size


def test_argument_validation(port):
    rng = np.random.default_rng(47)
    w = rng.uniform(-1, 1, (2, 8)).astype(np.float32)
    m = random_nm_mask(rng, 2, 8, 2)
    with pytest.raises(OracleError, match="dense"):
        port.pack_f32(m, 2, 8, w, 4)
    for n, mm in ((0, 4), (2, 8)):
        with pytest.raises(OracleError) as e:
            port.pack_f32(m, 2, 8, w, n, mm)
        assert e.value.kind == "invalid_argument"
    rag = m.copy()
    rag[0] ^= 1
    with pytest.raises(OracleError, match="keeps"):
        port.pack_f32(rag, 2, 8, w, 2)
    with pytest.raises(OracleError):
        port.pack_f32(np.array([0x03], np.uint8), 1, 6, np.ones((1, 6), np.float32), 2)


def test_unpack_round_trip_exact(port):
    rng = np.random.default_rng(53)
    for n in (1, 2):
        for _ in range(100):
            rows, cols = int(rng.integers(1, 7)), 4 * int(rng.integers(1, 9))
            m = random_nm_mask(rng, rows, cols, n)
            w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
            kept = mask_to_bool(m, rows, cols)
            vals, bits = port.unpack(port.pack_f32(m, rows, cols, w, n))
            assert np.array_equal(bits, m)
            assert np.array_equal(vals, np.where(kept, w, 0))
            q = port.quantize(w, [min(8, cols)] * rows, m)
            vals, bits = port.unpack(port.pack_int4(m, rows, cols, q, n))
            assert np.array_equal(bits, m)
            assert np.array_equal(vals.view(np.uint32), port.dequantize(q).view(np.uint32))


def test_malformed_streams(port):
    rng = np.random.default_rng(59)
    m = random_nm_mask(rng, 2, 8, 2)
    p = port.pack_f32(m, 2, 8, rng.uniform(-1, 1, (2, 8)).astype(np.float32), 2)
    bad = Packed(**{**p.__dict__})
    first = (int(p.index_words[0]) >> 14) & 3
    bad.index_words = p.index_words.copy()
    bad.index_words[0] = (int(p.index_words[0]) & 0x0FFF) | (first << 14) | (first << 12)
    with pytest.raises(OracleError, match="offsets") as e:
        port.unpack(bad)
    assert e.value.kind == "FormatError"
    for mutate in (lambda q: setattr(q, "index_words", np.append(q.index_words, 0)),
                   lambda q: setattr(q, "values", q.values[:-1]),
                   lambda q: setattr(q, "cols", 10)):
        q = Packed(**{**p.__dict__})
        mutate(q)
        with pytest.raises(OracleError) as e:
            port.unpack(q)
        assert e.value.kind == "FormatError"


def test_spmv_hand_checked(port):
    b = np.zeros((1, 4), bool)
    b[0, [1, 3]] = True
    m = mask_from_bool(b)
    w = np.array([[0, 2, 0, -1]], np.float32)
    x = np.ones(4, np.float32)
    assert port.spmv(port.pack_f32(m, 1, 4, w, 2), x)[0] == 1.0
    q = port.quantize(w, [4], m)
    assert port.spmv(port.pack_int4(m, 1, 4, q, 2), x)[0] == 1.0
    with pytest.raises(OracleError) as e:
        port.spmv(port.pack_f32(m, 1, 4, w, 2), np.ones(5, np.float32))
    assert e.value.kind == "invalid_argument"


def test_spmv_vs_dense(port):
    rng = np.random.default_rng(61)
    for n in (1, 2):
        for _ in range(150):
            rows, cols = int(rng.integers(1, 9)), 4 * int(rng.integers(1, 13))
            m = random_nm_mask(rng, rows, cols, n)
            w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
            x = rng.uniform(-1, 1, cols).astype(np.float32)
            p = port.pack_f32(m, rows, cols, w, n)
            want = port.unpack(p)[0].astype(np.float64) @ x
            got = port.spmv(p, x)
            assert np.all(np.abs(got - want) <= 1e-4 * (1 + np.abs(want)))
            q = port.quantize(w, [min(16, cols)] * rows, m)
            want = port.dequantize(q).astype(np.float64) @ x
            got = port.spmv(port.pack_int4(m, rows, cols, q, n), x)
            assert np.all(np.abs(got - want) <= 1e-4 * (1 + np.abs(want)))


def test_footprint_worked_example(port):
    rng = np.random.default_rng(67)
    m = random_nm_mask(rng, 1, 64, 2)
    q = port.quantize(rng.uniform(-1, 1, (1, 64)).astype(np.float32), [64], m)
    f = port.footprint(port.pack_int4(m, 1, 64, q, 2))
    assert (f["index_bytes"], f["value_bytes"], f["scale_bytes"], f["packed_bytes"], f["baseline_bytes"]) == (8, 16, 5, 29, 136)
    assert f["ratio"] == pytest.approx(29 / 136, rel=1e-12)


def test_footprint_ratio_gate(port):
    rng = np.random.default_rng(71)
    for rows in (16, 64):
        for cols in (64, 128, 256):
            for g in (64, 128):
                if g > cols:
                    continue
                for n in (1, 2):
                    m = random_nm_mask(rng, rows, cols, n)
                    q = port.quantize(rng.uniform(-1, 1, (rows, cols)).astype(np.float32), [g] * rows, m)
                    assert port.footprint(port.pack_int4(m, rows, cols, q, n))["ratio"] <= 0.30


def test_group_fit_known_answers(port):
    s, z = port.fit_group([0.0, 1.0, 2.0, 3.0])
    assert np.float32(s) == np.float32(0.2) and z == 0
    assert [port.encode_value(v, s, z) for v in (0.0, 1.0, 3.0)] == [0, 5, 15]
    assert [port.decode_value(c, s, z) for c in (0, 5, 10, 15)] == [0.0, 1.0, 2.0, 3.0]
    s, z = port.fit_group([-1.0, 1.0])
    assert s == pytest.approx(2.0 / 15.0, rel=1e-7) and z == 8
    for vals in ([0.0, 0.0, 0.0], []):
        s, z = port.fit_group(vals)
        assert np.float32(s) == np.float32(1e-8) and z == 0
    s, z = port.fit_group([2.5, 2.5])
    assert port.encode_value(2.5, s, z) == 15


def test_fit_over_retained_only(port):
    w = np.array([[-1, 1, 1000, 2000, 3000, 4000, -1, 0.5]], np.float32)
    b = np.zeros((1, 8), bool)
    b[0, [0, 1, 6, 7]] = True
    q = port.quantize(w, [4], mask_from_bool(b))
    assert q.codes.size == 4
    assert q.scales[0] == pytest.approx(2.0 / 15.0, rel=1e-7)
    back = port.dequantize(q)
    assert back[0, 2] == 0 and back[0, 3] == 0


def _golden_cases():
    g = np.load(GOLDEN)
    for i in range(int(g["n_cases"])):
        yield i, {k[len(f"c{i}_"):]: g[k] for k in g.files if k.startswith(f"c{i}_")}


def test_golden_vectors_bit_exact(port):
    """The restatement reproduces the reference's outputs bit for bit."""
    for i, c in _golden_cases():
        rows, cols, n, quant, dense_codes = (int(v) for v in c["meta"])
        if quant:
            q = port.quantize(c["w"], c["group_sizes"], None if dense_codes else c["mask"])
            assert np.array_equal(q.group_offsets, c["group_offsets"]), i
            assert np.array_equal(q.scales.view(np.uint32), c["scales"].view(np.uint32)), i
            assert np.array_equal(q.zero_points, c["zero_points"]), i
            assert np.array_equal(q.codes, c["codes"]), i
            assert np.array_equal(port.dequantize(q).view(np.uint32), c["dequant"].view(np.uint32)), i
            p = port.pack_int4(c["mask"], rows, cols, q, n)
            assert np.array_equal(p.value_bytes, c["value_bytes"]), i
        else:
            p = port.pack_f32(c["mask"], rows, cols, c["w"], n)
            assert np.array_equal(p.values.view(np.uint32), c["values"].view(np.uint32)), i
        assert np.array_equal(p.index_words, c["index_words"]), i
        vals, bits = port.unpack(p)
        assert np.array_equal(vals.view(np.uint32), c["unpack_values"].view(np.uint32)), i
        assert np.array_equal(bits, c["unpack_mask"]), i
        assert np.array_equal(port.spmv(p, c["x"]).view(np.uint32), c["y"].view(np.uint32)), i
        f = port.footprint(p)
        assert [f[k] for k in ("index_bytes", "value_bytes", "scale_bytes", "packed_bytes",
                               "baseline_bytes")] == c["footprint"].tolist(), i


def test_golden_group_fits(port):
    g = np.load(GOLDEN)
    vals = ([0.0, 1.0, 2.0, 3.0], [-1.0, 1.0], [0.0, 0.0, 0.0], [], [2.5, 2.5],
            [-0.7, 0.3, 0.9], [1e-9, 2e-9], [-3.0, -1.0])
    for v, s, z in zip(vals, g["fit_scale"], g["fit_zp"]):
        ps, pz = port.fit_group(v)
        assert np.float32(ps) == s and pz == z


def test_port_matches_live_reference(port, ref):
    rng = np.random.default_rng(7)
    for _ in range(40):
        rows, cols, n = int(rng.integers(1, 12)), 4 * int(rng.integers(1, 40)), int(rng.integers(1, 3))
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        m = random_nm_mask(rng, rows, cols, n)
        gs = rng.choice([4, 8, 16, 32, 64, 128], rows).astype(np.uint32)
        qp, qr = port.quantize(w, gs, m), ref.quantize(w, gs, m)
        assert np.array_equal(qp.codes, qr.codes)
        assert np.array_equal(qp.scales.view(np.uint32), qr.scales.view(np.uint32))
        pp, pr = port.pack_int4(m, rows, cols, qp, n), ref.pack_int4(m, rows, cols, qr, n)
        assert np.array_equal(pp.index_words, pr.index_words)
        assert np.array_equal(pp.value_bytes, pr.value_bytes)
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        assert np.array_equal(port.spmv(pp, x).view(np.uint32), ref.spmv(pr, x).view(np.uint32))


def test_importance_prune_port_matches_reference(port, ref):
    """The oracle port's importance_scores / prune_nm against the unmodified
    reference (compress.cpp:230-278) on ties, zeros and negative scores."""
    P, R = port, ref
    rng = np.random.default_rng(17)
    for rows, cols in [(7, 13), (16, 64), (33, 130)]:
        w = rng.normal(size=(rows, cols)).astype(np.float32)
        xn = rng.uniform(0, 2, cols).astype(np.float32)
        g = np.abs(rng.normal(size=(rows, cols))).astype(np.float32)
        assert np.array_equal(P.importance(w, xn, g).view(np.uint32), R.importance(w, xn, g).view(np.uint32))
        s = (np.round(rng.normal(size=(rows, cols)) * 2) / 2).astype(np.float32)
        for n in (1, 2, 3):
            assert np.array_equal(P.prune_nm(s, n), R.prune_nm(s, n))
