"""Pins the verify-path oracles to the reference's OWN model / decoder code
(model.cpp, decode.cpp compiled unmodified into oracle/_ref by
oracle/build_ref.sh, bindings oracle/ref_model.py):

* the C restatement of the forward (oracle/egt_oracle.c egto_forward,
  model.cpp:118-202) against the reference's forward;
* the Python restatement of flatten / tree mask / verify_parallel
  (tests/verify_oracle.py, decode.cpp:209-421) against the reference's;
* the reference's own pinned properties, re-run through the reference
  (tree-vs-sequential logits, acceptance_main.cpp:496-532; switch-point
  invariance, test_decode.cpp:605-646).

CPU only: these tests fix what the GPU parity tests compare against."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_LIB
from tests import verify_oracle as vo

pytestmark = pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")

CFG = dict(vocab_size=48, d_model=64, n_layers=2, n_heads=4, d_ff=128, max_positions=64)


def dense_model(cfg, seed):
    """init_model-style U(-1/sqrt(d), 1/sqrt(d)) weights (model.hpp:61-62)."""
    rng = np.random.default_rng(seed)
    d, dff, V = cfg["d_model"], cfg["d_ff"], cfg["vocab_size"]
    b = 1.0 / np.sqrt(d)
    emb = rng.uniform(-b, b, (V, d)).astype(np.float32)
    shapes = dict(wq=(d, d), wk=(d, d), wv=(d, d), wo=(d, d), ff1=(dff, d), ff2=(d, dff))
    layers = [{k: rng.uniform(-b, b, s).astype(np.float32) for k, s in shapes.items()} for _ in range(cfg["n_layers"])]
    head = rng.uniform(-b, b, (V, d)).astype(np.float32)
    return emb, layers, head


def random_trie(rng, depth=3, lo=2, hi=4):
    from types import SimpleNamespace

    token, parent, payload = [1], [0], [-1]
    frontier = [0]
    for _ in range(depth):
        nxt = []
        for node in frontier:
            for dgt in range(int(rng.integers(lo, hi + 1))):
                token.append(4 + dgt)
                parent.append(node)
                payload.append(-1)
                nxt.append(len(token) - 1)
        frontier = nxt
    for i, n in enumerate(frontier):
        payload[n] = i
    return SimpleNamespace(token=np.array(token, np.uint32), parent=np.array(parent, np.uint32),
                           payload=np.array(payload, np.int64))


class B:
    def __init__(self, tokens, log_prob, node):
        self.tokens, self.log_prob, self.node = tokens, log_prob, node


@pytest.fixture(scope="module")
def ref_model():
    from oracle.ref_model import RefModel

    emb, layers, head = dense_model(CFG, 5)
    return RefModel(CFG, emb, layers, head), (emb, layers, head)


def test_positions_match_port(ref_model, port):
    m, _ = ref_model
    assert np.array_equal(m.positions(), port.sinusoidal_positions(CFG["max_positions"], CFG["d_model"]))


def test_port_forward_pinned(ref_model, port):
    """egto_forward (the C restatement) == the reference's forward on the same
    dense weights, masks with empty rows included."""
    m, (emb, layers, head) = ref_model
    ptab = port.sinusoidal_positions(CFG["max_positions"], CFG["d_model"])
    rng = np.random.default_rng(3)
    worst = 0.0
    for M in (1, 5, 33):
        tokens = rng.integers(0, CFG["vocab_size"], M).astype(np.int32)
        pos = rng.integers(0, CFG["max_positions"], M).astype(np.int32)
        vis = rng.random((M, M)) < 0.4
        vis[0, :] = False
        want = m.forward(tokens, pos, vis)
        got = port.forward(CFG, emb, layers, head, ptab, tokens, pos, vis.astype(np.uint8))
        worst = max(worst, float(np.max(np.abs(got - want) / (1 + np.abs(want)))))
    assert worst <= 1e-6, worst


def test_reference_errors_pinned(ref_model):
    from oracle.oracle import OracleError

    m, _ = ref_model
    with pytest.raises(OracleError, match="token out of range"):
        m.forward([CFG["vocab_size"]], [0], np.ones((1, 1), bool))
    with pytest.raises(OracleError, match="position out of range"):
        m.forward([1], [CFG["max_positions"]], np.ones((1, 1), bool))


def _sessions(trie):
    kids = vo.children(trie, 0)
    return [[B([], 0.0, 0)],
            [B([int(trie.token[kids[0]])], -0.7, kids[0]), B([int(trie.token[kids[-1]])], -1.1, kids[-1])]]


def test_tree_mask_restatement_pinned():
    from oracle import ref_model as R

    rng = np.random.default_rng(4)
    for trial in range(6):
        trie = random_trie(rng, depth=3, lo=1, hi=3)
        for beams in _sessions(trie):
            prompt = [1] + rng.integers(4, 40, int(rng.integers(0, 4))).tolist()
            flat, vis, toks, pos, lmax, off = R.tree_mask(trie, prompt, beams)
            pf = vo.flatten_subtree(trie, beams)
            pv, pt, pp, plmax, poff = vo.build_tree_mask(pf, prompt, beams)
            assert [f["token"] for f in pf] == flat["token"].tolist()
            assert [f["parent"] for f in pf] == flat["parent"].tolist()
            assert [f["depth"] for f in pf] == flat["depth"].tolist()
            assert [f["trie_node"] for f in pf] == flat["trie_node"].tolist()
            assert (plmax, poff) == (lmax, off)
            assert np.array_equal(pv, vis) and np.array_equal(pt, toks) and np.array_equal(pp, pos)


def test_verify_restatement_pinned(ref_model):
    """verify_oracle.verify_parallel over the reference's forward == the
    reference's verify_parallel (same selections, scores to 1e-12)."""
    m, _ = ref_model
    rng = np.random.default_rng(12)
    for trial in range(3):
        trie = random_trie(rng)
        prompt = [1, 9, 13]
        for beams in _sessions(trie):
            for bs in (1, 4, 20):
                want, scores, info = m.verify_parallel(trie, prompt, beams, bs)
                got, ginfo = vo.verify_parallel(m.forward, trie, prompt, beams, bs)
                assert ginfo == {k: info[k] for k in ("flattened_nodes", "rows")}
                assert [(g["tokens"], g["payload"], g["beam"]) for g in got] == \
                       [(w["tokens"], w["payload"], w["beam"]) for w in want]
                assert np.allclose([g["score"] for g in got], [w["score"] for w in want], rtol=0, atol=1e-12)


def test_reference_properties(ref_model):
    """The reference's own verify pins, re-run on the reference itself: the
    tree pass equals exhaustive autoregressive decoding (acceptance_main.cpp:
    536-598), for forced switch depths 0..2 (test_decode.cpp:605-646)."""
    m, _ = ref_model
    rng = np.random.default_rng(13)
    trie = random_trie(rng, depth=3, lo=2, hi=3)
    n_leaves = sum(1 for i in range(len(trie.token)) if vo.is_leaf(trie, i))
    prompt = [1, 22, 7]
    ar, ast = m.decode(trie, prompt, n_leaves, mode="autoregressive")
    assert ast["trigger_step"] == -1 and ast["forward_passes"] == 3
    want = sorted((tuple(s["tokens"]), s["score"]) for s in ar)
    for depth in (0, 1, 2):
        fv, fst = m.decode(trie, prompt, n_leaves, mode="forced", forced_depth=depth)
        assert fst["trigger_step"] == depth
        got = sorted((tuple(s["tokens"]), s["score"]) for s in fv)
        assert [g[0] for g in got] == [w[0] for w in want]
        assert np.allclose([g[1] for g in got], [w[1] for w in want], atol=1e-4)


def test_reference_cost_model_and_plan():
    from oracle import ref_model as R

    t, a, b = R.cost_estimator([("step", 2.0), ("step", 1.0), ("verify", 10, 3.0), ("verify", 20, 5.0)])
    assert abs(t - (0.9 * 2.0 + 0.1 * 1.0)) < 1e-15
    assert abs(a - 0.2) < 1e-12 and abs(b - 1.0) < 1e-12
    rng = np.random.default_rng(0)
    ws = [rng.uniform(-1, 1, (8, 16)).astype(np.float32) for _ in range(5)]
    ss = [np.abs(w) * (i + 1) for i, w in enumerate(ws)]
    assert R.plan_sparsity(ss, ws, 0.4) == [1, 1, 1, 2, 2]
