"""GPU parity of the verify substrate: the device forward over mixed-dispatch
packed layers against the C oracle's forward (model.cpp:118-202) on the
dense reconstructions of the same layers, and prefix-tree verification /
decoding against the Python restatement of decode.cpp and the reference's
own properties (tree-vs-sequential, switch-point invariance)."""
import numpy as np
import pytest

from tests import verify_oracle as vo

pytestmark = pytest.mark.gpu

CFG = dict(vocab_size=48, d_model=64, n_layers=2, n_heads=4, d_ff=128, max_positions=64)
PLAN = [["int4-2:4", "int4-1:4", "fp16-2:4", "int4-dense", "int4-2:4", "fp16-1:4"],
        ["int4-2:4"] * 6]


def _dense_of(port, art):
    from oracle.oracle import Packed, Quantized

    from paper_2605_11582_b200.packed import PackedSparseMatrix

    if isinstance(art, PackedSparseMatrix):
        p = Packed(art.n, art.m, art.rows, art.cols, art.kind, art.index_words, art.value_bytes, art.group_sizes,
                   art.group_offsets, art.scales, art.zero_points, art.values)
        return port.unpack(p)[0]
    q = Quantized(art.rows, art.cols, art.group_sizes, art.group_offsets, art.scales, art.zero_points, art.codes)
    return port.dequantize(q)


def build_model(port, cfg=CFG, plan=PLAN, seed=5, group=32):
    """init_model-style weights U(-1/sqrt(d), 1/sqrt(d)) (model.hpp:61-62),
    each linear layer compressed by the product's encoder."""
    from paper_2605_11582_b200.model import DeviceModel, compress_layer

    rng = np.random.default_rng(seed)
    d, dff, V = cfg["d_model"], cfg["d_ff"], cfg["vocab_size"]
    bound = 1.0 / np.sqrt(d)
    emb = rng.uniform(-bound, bound, (V, d)).astype(np.float32)
    shapes = [(d, d)] * 4 + [(dff, d), (d, dff)]
    handles, dense_layers = [], []
    for li in range(cfg["n_layers"]):
        layer = {}
        for part, shape, kind in zip(("wq", "wk", "wv", "wo", "ff1", "ff2"), shapes, plan[li % len(plan)]):
            w = rng.uniform(-bound, bound, shape).astype(np.float32)
            h, art = compress_layer(w, kind, group)
            handles.append(h)
            layer[part] = _dense_of(port, art)
        dense_layers.append(layer)
    hw = rng.uniform(-bound, bound, (V, d)).astype(np.float32)
    head, hart = compress_layer(hw, "int4-2:4", 32)
    model = DeviceModel(cfg, emb, handles, head)
    model._keep = handles
    ptab = port.sinusoidal_positions(cfg["max_positions"], d)
    dense_head = _dense_of(port, hart)

    def oracle_forward(tokens, positions, vis):
        return port.forward(cfg, emb, dense_layers, dense_head, ptab, tokens, positions, vis.astype(np.uint8))

    return model, oracle_forward


def random_trie(rng, depth=3, lo=2, hi=4):
    """Semantic-ID trie: digit d -> token 4 + d (trie.hpp:38), payload per leaf."""
    from paper_2605_11582_b200.model import Trie

    token, parent, payload = [1], [0], [-1]
    frontier = [0]
    for level in range(depth):
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


@pytest.fixture(scope="module")
def model_pair(port):
    return build_model(port)


def _close(got, want, tol=1e-3):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return np.max(np.abs(got - want) / (1 + np.abs(want)))


def test_forward_matches_oracle(model_pair):
    model, oracle_forward = model_pair
    rng = np.random.default_rng(11)
    for M in (1, 7, 33):
        tokens = rng.integers(0, CFG["vocab_size"], M).astype(np.int32)
        pos = rng.integers(0, CFG["max_positions"], M).astype(np.int32)
        vis = rng.random((M, M)) < 0.4
        vis[0, :] = False  # a row with no visible key -> zero attention output
        got = model.forward(tokens, pos, vis).cpu().numpy()
        want = oracle_forward(tokens, pos, vis)
        assert _close(got, want) <= 1e-3, f"M={M}: {_close(got, want):.2e}"


def test_forward_errors(model_pair):
    import paper_2605_11582_b200 as egt

    model, _ = model_pair
    with pytest.raises(egt.InvalidArgument, match="token out of range"):
        model.forward([CFG["vocab_size"]], [0], np.ones((1, 1), bool))
    with pytest.raises(egt.InvalidArgument, match="position out of range"):
        model.forward([1], [CFG["max_positions"]], np.ones((1, 1), bool))


def test_verify_matches_python_restatement(model_pair):
    from paper_2605_11582_b200.model import Beam

    model, oracle_forward = model_pair
    rng = np.random.default_rng(12)
    trie = random_trie(rng)
    prompt = [1, 9, 13]
    # a fresh session (one empty beam at the root) and a two-beam session one level down
    root_children = vo.children(trie, 0)
    sessions = [[Beam([], 0.0, 0)],
                [Beam([int(trie.token[root_children[0]])], -0.7, root_children[0]),
                 Beam([int(trie.token[root_children[-1]])], -1.1, root_children[-1])]]
    for beams in sessions:
        got, gstat = model.verify_parallel(trie, prompt, beams, 4)
        want, wstat = vo.verify_parallel(oracle_forward, trie, prompt, beams, 4)
        assert gstat == wstat
        assert [(g["tokens"], g["payload"], g["beam"]) for g in got] == \
               [(w["tokens"], w["payload"], w["beam"]) for w in want]
        assert np.allclose([g["score"] for g in got], [w["score"] for w in want], atol=1e-4)


def test_switch_point_invariance(model_pair):
    """decode with a forced switch at depth 0/1/2, and with the cost model,
    gives the exhaustive autoregressive result (test_decode.cpp:605-646):
    with a beam covering every leaf the sets and scores agree (<= 1e-4)."""
    model, _ = model_pair
    rng = np.random.default_rng(13)
    trie = random_trie(rng, depth=3, lo=2, hi=3)
    n_leaves = sum(1 for i in range(len(trie.token)) if vo.is_leaf(trie, i))
    prompt = [1, 22, 7]
    ar, ast = model.decode(trie, prompt, n_leaves, mode="autoregressive")
    assert ast["trigger_step"] == -1 and ast["forward_passes"] == 3
    want = sorted((tuple(s["tokens"]), s["score"]) for s in ar)
    for depth in (0, 1, 2):
        fv, fst = model.decode(trie, prompt, n_leaves, mode="forced", forced_depth=depth)
        assert fst["trigger_step"] == depth and fst["forward_passes"] == depth + 1
        got = sorted((tuple(s["tokens"]), s["score"]) for s in fv)
        assert [g[0] for g in got] == [w[0] for w in want]
        assert np.allclose([g[1] for g in got], [w[1] for w in want], atol=1e-4)
    _, cst = model.decode(trie, prompt, 4, mode="ptpv", cost=(1.0, 1e-3, 0.0))
    assert cst["trigger_step"] == 0  # cheap verification fires at once
    _, cst = model.decode(trie, prompt, 4, mode="ptpv", cost=(1e-3, 1.0, 0.0))
    assert cst["trigger_step"] == -1  # expensive verification never fires


def test_verify_equals_exhaustive_enumeration(model_pair):
    """Every leaf's verified score equals the sum of per-step restricted
    log-probs computed by sequential (causal) forwards (acceptance_main.cpp:496-598)."""
    model, oracle_forward = model_pair
    rng = np.random.default_rng(14)
    trie = random_trie(rng, depth=2, lo=2, hi=3)
    prompt = [1, 3]
    n_leaves = sum(1 for i in range(len(trie.token)) if vo.is_leaf(trie, i))
    from paper_2605_11582_b200.model import Beam

    got, _ = model.verify_parallel(trie, prompt, [Beam([], 0.0, 0)], n_leaves)
    for leaf in got:
        seq = list(prompt)
        node, score = 0, 0.0
        for t in leaf["tokens"]:
            M = len(seq)
            logits = model.forward(seq, list(range(M)), np.tril(np.ones((M, M), bool))).cpu().numpy()
            ch, lp = vo.restrict_row(logits[-1], trie, node)
            nxt = [c for c in ch if int(trie.token[c]) == t][0]
            score += float(lp[ch.index(nxt)])
            node = nxt
            seq.append(t)
        assert abs(score - leaf["score"]) <= 1e-4


@pytest.mark.parametrize("cfg", [CFG, dict(vocab_size=97, d_model=256, n_layers=2, n_heads=4, d_ff=512,
                                           max_positions=64)])
def test_kv_decoder_matches_forward(port, cfg):
    """The KV-cached device decode loop (egt_decoder_*) against the oracle's
    full-prefix forward (model.cpp:118-202, causal mask) on the decoder's own
    token sequence: the last step's logits agree within 1e-3 (1+|want|) and
    every generated token is the oracle's argmax (up to a 1e-3 near-tie)."""
    import torch

    from paper_2605_11582_b200.model import Decoder

    model, oracle_forward = build_model(port, cfg)
    dec = Decoder(model, 40)
    prompt = [3, 1, 4, 1, 5]
    n_new = 12
    toks = dec.generate(prompt, n_new)
    assert toks[: len(prompt)] == prompt and len(toks) == len(prompt) + n_new
    n = len(toks) - 1  # positions 0..n-1 have been run; toks[n] is the next token
    seq = np.array(toks[:n], np.int32)
    causal = np.tril(np.ones((n, n), bool))
    want = oracle_forward(seq, np.arange(n, dtype=np.int32), causal)
    logits = torch.empty(cfg["vocab_size"], device="cuda")
    dec.read(logits)
    got = logits.cpu().numpy()
    err = np.abs(got - want[n - 1]) / (1 + np.abs(want[n - 1]))
    assert err.max() <= 1e-3, err.max()
    for i in range(len(prompt) - 1, n):  # token i+1 chosen from row i
        row = want[i]
        assert row[toks[i + 1]] >= row.max() - 1e-3 * (1 + abs(row.max())), (i, toks[i + 1], int(row.argmax()))
    # a second run from a different prompt reuses the graph and cache
    toks2 = dec.generate([7, 2], 5)
    assert toks2[:2] == [7, 2] and len(toks2) == 7


def test_forward_tree_equals_dense_mask(model_pair):
    """Compact tree encoding (egt_forward_tree): the device
    builds the same mask as build_tree_mask (decode.cpp:240-299), so the
    logits equal the dense-bitmap forward bit for bit; bad encodings raise
    the reference's messages."""
    import paper_2605_11582_b200 as egt
    from tests import verify_oracle as vo

    model, _ = model_pair
    rng = np.random.default_rng(23)
    trie = random_trie(rng, depth=3, lo=2, hi=3)

    class B:
        def __init__(self, node, tokens):
            self.node, self.tokens = node, tokens

    kids = vo.children(trie, 0)
    beams = [B(0, []), B(int(kids[0]), [int(trie.token[kids[0]])])]
    prompt = [1, 2, 3]
    flat = vo.flatten_subtree(trie, beams)
    vis, tokens, pos, lmax, off = vo.build_tree_mask(flat, prompt, beams)
    lens = [len(prompt) + len(b.tokens) for b in beams]
    got = model.forward_tree(tokens, pos, lens, lmax, [f["parent"] for f in flat], [f["beam"] for f in flat])
    want = model.forward(tokens, pos, vis)
    assert np.array_equal(got.cpu().numpy(), want.cpu().numpy())
    with pytest.raises(egt.InvalidArgument, match="parent does not precede"):
        model.forward_tree(tokens, pos, lens, lmax, [1] + [f["parent"] for f in flat][1:], [f["beam"] for f in flat])
    with pytest.raises(egt.InvalidArgument, match="missing beam"):
        model.forward_tree(tokens, pos, lens, lmax, [f["parent"] for f in flat], [5] * len(flat))


def test_cost_model_from_device_timings(model_pair):
    """CostModelEstimator (decode.cpp:84-120) fed CUDA-event timings of this
    model's constrained-step and verify forwards (egt_measure_cost_model,
    SURVEY 8(a) a20); decode with the measured model fires where
    estimate_trigger says and returns the exhaustive autoregressive result
    (switch-point invariance, test_decode.cpp:605-646)."""
    from paper_2605_11582_b200 import planning as P

    model, _ = model_pair
    est = P.CostModelEstimator()
    t_step, alpha, beta = est.measure(model, prompt_len=3, n_beams=2, node_counts=[4, 8, 16, 32], reps=3)
    assert t_step > 0 and np.isfinite(alpha) and np.isfinite(beta)
    assert alpha * 32 + beta > 0  # a verify pass costs time
    rng = np.random.default_rng(15)
    trie = random_trie(rng, depth=3, lo=2, hi=3)
    n_leaves = sum(1 for i in range(len(trie.token)) if vo.is_leaf(trie, i))
    prompt = [1, 22, 7]
    fire, _ = P.estimate_trigger(trie, prompt, [type("B", (), dict(tokens=[], log_prob=0.0, node=0))()],
                                 (t_step, alpha, beta))
    ar, _ = model.decode(trie, prompt, n_leaves, mode="autoregressive")
    got, st = model.decode(trie, prompt, n_leaves, mode="ptpv", cost=(t_step, alpha, beta))
    assert (st["trigger_step"] == 0) == fire
    assert sorted(tuple(s["tokens"]) for s in got) == sorted(tuple(s["tokens"]) for s in ar)
    assert np.allclose(sorted(s["score"] for s in got), sorted(s["score"] for s in ar), atol=1e-4)


@pytest.mark.parametrize("beam", [1, 3, 8])
def test_kv_cached_beam_decode_matches_reference(port, beam):
    """The KV-cached trie-constrained beam step (SURVEY 8(f) row 1,
    constrained_step_kv: one new row per beam per step against its cached
    prefix) against the REFERENCE's full-recompute decode (decode.cpp:122-190,
    423-483, oracle/_ref) on the dense reconstructions of the same layers:
    the same sequences, payloads and step counts, scores within 1e-4; and the
    same as the product's own full-recompute steps."""
    import os

    from oracle.oracle import REF_LIB

    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built")
    from oracle.ref_model import RefModel
    from paper_2605_11582_b200.model import DeviceModel, compress_layer

    rng = np.random.default_rng(40 + beam)
    cfg = dict(vocab_size=64, d_model=128, n_layers=2, n_heads=4, d_ff=256, max_positions=64)
    d, dff, V = cfg["d_model"], cfg["d_ff"], cfg["vocab_size"]
    b = 1.0 / np.sqrt(d)
    emb = rng.uniform(-b, b, (V, d)).astype(np.float32)
    shapes = [(d, d)] * 4 + [(dff, d), (d, dff)]
    handles, dense = [], []
    for li in range(cfg["n_layers"]):
        layer = {}
        for part, shape, kind in zip(("wq", "wk", "wv", "wo", "ff1", "ff2"), shapes, PLAN[li % len(PLAN)]):
            w = rng.uniform(-b, b, shape).astype(np.float32)
            h, art = compress_layer(w, kind, 32)
            handles.append(h)
            layer[part] = _dense_of(port, art)
        dense.append(layer)
    hw = rng.uniform(-b, b, (V, d)).astype(np.float32)
    head, hart = compress_layer(hw, "int4-2:4", 32)
    model = DeviceModel(cfg, emb, handles, head)
    model._keep = handles
    ref = RefModel(cfg, emb, dense, _dense_of(port, hart))
    trie = random_trie(rng, depth=4, lo=2, hi=4)
    prompt = [1, 17, 5, 33, 9]
    got, gst = model.decode(trie, prompt, beam, mode="autoregressive", kv_cache=True)
    full, fst = model.decode(trie, prompt, beam, mode="autoregressive")
    want, wst = ref.decode(trie, prompt, beam, mode="autoregressive")
    assert gst == fst and gst["steps"] == wst["steps"] and gst["forward_passes"] == wst["forward_passes"]
    for g, f, w in zip(got, full, want):
        assert g["tokens"] == f["tokens"] == w["tokens"] and g["payload"] == w["payload"]
        assert abs(g["score"] - w["score"]) <= 1e-4 and abs(g["score"] - f["score"]) <= 1e-4
    assert len(got) == len(want)
