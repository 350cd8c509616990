"""Host planning around the hot path against the reference's own code
(oracle/_ref: compress.cpp's plan_sparsity, decode.cpp's CostModelEstimator,
estimate_trigger, flatten_subtree / build_tree_mask), on CPU:
* plan_sparsity: identical patterns, ties included;
* CostModelEstimator (a20): identical (t_step, alpha, beta) after the same
  observations, including the 32-sample window and the zero-spread case;
  the reference's own errors;
* estimate_trigger and the tree mask (a17, a20): identical outputs."""
import os

import numpy as np
import pytest

from oracle.oracle import REF_LIB

pytestmark = pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")


def test_plan_sparsity_matches_reference():
    from oracle import ref_model as R
    from paper_2605_11582_b200 import planning as P

    rng = np.random.default_rng(1)
    for trial in range(20):
        L = int(rng.integers(1, 12))
        shapes = [(int(rng.integers(1, 9)), 4 * int(rng.integers(1, 9))) for _ in range(L)]
        ws = [rng.uniform(-1, 1, s).astype(np.float32) for s in shapes]
        ss = [np.abs(w) * rng.uniform(0, 2, w.shape).astype(np.float32) for w in ws]
        if trial % 4 == 0:  # exact ties: identical layers
            ws = [ws[0]] * L
            ss = [ss[0]] * L
        if trial % 5 == 0:
            ws[0] = np.zeros_like(ws[0])  # mean |w| = 0 -> importance 0
        for rho in (0.0, 0.25, 0.5, 1.0 / 3.0, 1.0):
            assert P.plan_sparsity(ss, ws, rho) == R.plan_sparsity(ss, ws, rho), (trial, rho)


def test_plan_sparsity_errors():
    import paper_2605_11582_b200 as egt
    from paper_2605_11582_b200 import planning as P

    w = np.ones((2, 4), np.float32)
    with pytest.raises(egt.InvalidArgument, match="rho_s must be in"):
        P.plan_sparsity([w], [w], 1.5)


def test_cost_estimator_matches_reference():
    from oracle import ref_model as R
    from paper_2605_11582_b200 import planning as P

    rng = np.random.default_rng(2)
    for trial in range(10):
        init = tuple(rng.uniform(0, 1e-2, 3))
        obs = []
        for _ in range(int(rng.integers(1, 80))):
            if rng.random() < 0.4:
                obs.append(("step", float(rng.uniform(1e-4, 1e-2))))
            else:
                n = int(rng.integers(1, 400)) if trial % 3 else 64  # zero spread -> beta only
                obs.append(("verify", n, float(2e-6 * n + 1e-3 + rng.normal(0, 1e-5))))
        est = P.CostModelEstimator(*init)
        for o in obs:
            if o[0] == "step":
                est.observe_step(o[1])
            else:
                est.observe_verify(o[1], o[2])
        want = R.cost_estimator(obs, init)
        assert np.allclose(est.model(), want, rtol=1e-12, atol=0), (trial, est.model(), want)


def test_cost_estimator_errors():
    import paper_2605_11582_b200 as egt
    from paper_2605_11582_b200 import planning as P

    est = P.CostModelEstimator()
    with pytest.raises(egt.InvalidArgument, match="step time must be finite"):
        est.observe_step(float("nan"))
    with pytest.raises(egt.InvalidArgument, match="verification over zero nodes"):
        est.observe_verify(0, 1.0)
    with pytest.raises(egt.InvalidArgument, match="verification time must be finite"):
        est.observe_verify(3, -1.0)


def _trie(rng, depth=3, lo=1, hi=3):
    from paper_2605_11582_b200.model import Trie

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
    return Trie(np.array(token, np.uint32), np.array(parent, np.uint32), np.array(payload, np.int64))


def _sessions(trie):
    from paper_2605_11582_b200.model import Beam

    kids = trie.children(0)
    out = [[Beam([], 0.0, 0)]]
    if len(kids) >= 2:
        out.append([Beam([int(trie.token[kids[0]])], -0.5, kids[0]),
                    Beam([int(trie.token[kids[-1]])], -1.5, kids[-1])])
    return out


def test_trigger_and_tree_mask_match_reference():
    from oracle import ref_model as R
    from paper_2605_11582_b200 import planning as P

    rng = np.random.default_rng(3)
    for trial in range(12):
        trie = _trie(rng)
        for beams in _sessions(trie):
            prompt = [1] + rng.integers(4, 50, int(rng.integers(0, 5))).tolist()
            got = P.tree_mask(trie, prompt, beams)
            want = R.tree_mask(trie, prompt, beams)
            for k in ("token", "parent", "depth", "trie_node", "beam"):
                assert np.array_equal(got[0][k], want[0][k]), k
            for a, b in zip(got[1:], want[1:]):
                assert np.array_equal(np.asarray(a), np.asarray(b))
            for cost in ((1.0, 1e-3, 0.0), (1e-3, 1.0, 0.0), (2e-3, 1e-5, 1e-3), (0.0, 0.0, 0.0)):
                for cap in (4096, 3):
                    assert P.estimate_trigger(trie, prompt, beams, cost, cap) == \
                        R.estimate_trigger(trie, prompt, beams, cost, cap), (cost, cap)
