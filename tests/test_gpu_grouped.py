"""INT4 2:4 with the reference's default fine groups (g_fine = 16,
config.hpp:50-51; mixed with g_coarse = 64 per row) against the port's f32
spmv (packed.cpp:211-220): on the tiled path (16-column scale entries, two
mma.sp per k-tile; cols % 32 == 0) and on the grouped-stream kernel
(reference-order stream, cols % 32 == 16): 7B shapes, M = 1..9, the fused
rmsnorm / silu inputs and residual / silu epilogue (model.cpp:57-67, 80-84,
186-190), x over the whole f32 range, bit-exact unpack."""
import numpy as np
import pytest

from tests.layers import close, make_int4, to_product

pytestmark = pytest.mark.gpu


def _layer(port, rng, rows, cols, g):
    import paper_2605_11582_b200 as egt

    p, _, _ = make_int4(rng, rows, cols, 2, g, port)
    d = egt.DeviceMatrix.from_packed(to_product(p))
    assert d.path == ("tiled-mma.sp" if cols % 32 == 0 else "general"), (cols, d.path)
    return p, d


@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (4096, 11008), (40, 96), (4096, 4080), (33, 112)])
@pytest.mark.parametrize("groups", ["g16", "g16/64"])
@pytest.mark.parametrize("M", [1, 2, 4, 9])
def test_grouped_products(port, shape, groups, M):
    import torch

    rows, cols = shape
    rng = np.random.default_rng(rows + cols + M)
    g = 16 if groups == "g16" else np.where(np.arange(rows) % 2 == 0, 16, 64).astype(np.uint32)
    p, d = _layer(port, rng, rows, cols, g)
    xs = rng.uniform(-1, 1, (M, cols)).astype(np.float32)
    y = d.spmv(torch.from_numpy(xs).cuda() if M > 1 else torch.from_numpy(xs[0]).cuda()).cpu().numpy()
    y = y.reshape(M, rows)
    for m in range(M):
        ok, err = close(y[m], port.spmv(p, xs[m]))
        assert ok, (shape, groups, M, m, err)


@pytest.mark.parametrize("cols", [1024, 1008])
def test_grouped_fused(port, cols):
    """y = silu(res + rmsnorm(x) W^T) and y = silu(x) W^T (tiled / stream)."""
    import torch

    from paper_2605_11582_b200 import native as N

    rng = np.random.default_rng(5)
    rows, M = 256, 2
    p, d = _layer(port, rng, rows, cols, 16)
    xs = rng.uniform(-2, 2, (M, cols)).astype(np.float32)
    res = rng.uniform(-1, 1, (M, rows)).astype(np.float32)
    eps = 1e-6
    y = torch.empty((M, rows), device="cuda")
    d.spmv_fused_into(torch.from_numpy(xs).cuda(), y, input=N.INPUT_RMSNORM, eps=eps,
                      residual=torch.from_numpy(res).cuda(), output_silu=True)
    got = y.cpu().numpy()
    for m in range(M):
        xn = (xs[m] / np.sqrt(np.mean(xs[m].astype(np.float64) ** 2) + eps)).astype(np.float32)
        pre = res[m] + port.spmv(p, xn)
        ok, err = close(got[m], pre / (1 + np.exp(-pre.astype(np.float64))))
        assert ok, (m, err)
    y2 = torch.empty((M, rows), device="cuda")
    d.spmv_fused_into(torch.from_numpy(xs).cuda(), y2, input=N.INPUT_SILU)
    got2 = y2.cpu().numpy()
    for m in range(M):
        xsil = (xs[m] / (1 + np.exp(-xs[m].astype(np.float64)))).astype(np.float32)
        ok, err = close(got2[m], port.spmv(p, xsil))
        assert ok, (m, err)


@pytest.mark.parametrize("cols", [512, 496])
def test_grouped_x_range(port, cols):
    """Huge / tiny / non-finite x give the reference's values, NaN / inf at
    the same positions (tiled: window scaling + exact fix-up; stream: f32)."""
    import torch

    rng = np.random.default_rng(9)
    rows = 64
    p, d = _layer(port, rng, rows, cols, 16)
    for kind in ("huge", "tiny", "inf", "nan"):
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        if kind == "huge":
            x *= 1e5
        elif kind == "tiny":
            x *= 1e-6
        elif kind == "inf":
            x[rng.integers(0, cols, 3)] = np.inf
        else:
            x[rng.integers(0, cols, 3)] = np.nan
        got = d.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        want = port.spmv(p, x)
        assert np.array_equal(np.isnan(got), np.isnan(want)), kind
        assert np.array_equal(np.isposinf(got), np.isposinf(want)), kind
        fin = np.isfinite(want)
        scale = np.abs(x[np.isfinite(x)]).max()
        ok, err = close(got[fin] / scale, want[fin] / scale)
        assert ok, (kind, err)


@pytest.mark.parametrize("M", [3, 9])
def test_grouped_many_tokens_wide(port, M):
    """4096 x 11008 (x of 11008 floats: two tokens per launch) and M > 4
    (token groups over several launches)."""
    import torch

    rng = np.random.default_rng(M)
    p, d = _layer(port, rng, 256, 11008, 16)  # tiled; the stream kernel's wide case is 4080 above
    xs = rng.uniform(-1, 1, (M, 11008)).astype(np.float32)
    y = d.spmv(torch.from_numpy(xs).cuda()).cpu().numpy()
    for m in range(M):
        ok, err = close(y[m], port.spmv(p, xs[m]))
        assert ok, (m, err)


def test_grouped_model_forward(port):
    """A model whose layers use the reference's default g_fine = 16 runs the
    fused forward (rmsnorm / silu / residual on the grouped path) and matches
    the oracle forward (model.cpp:118-202)."""
    from tests.test_gpu_verify import CFG, _close, build_model

    model, oracle_forward = build_model(port, plan=[["int4-2:4"] * 6], group=16)
    rng = np.random.default_rng(3)
    for M in (1, 6):
        tokens = rng.integers(0, CFG["vocab_size"], M).astype(np.int32)
        pos = rng.integers(0, CFG["max_positions"], M).astype(np.int32)
        vis = np.tril(np.ones((M, M), bool))
        got = model.forward(tokens, pos, vis).cpu().numpy()
        want = oracle_forward(tokens, pos, vis)
        assert _close(got, want) <= 1e-3, (M, _close(got, want))


@pytest.mark.parametrize("groups", ["g16", "g16/64"])
def test_grouped_unpack_bit_exact(port, groups):
    """unpack (packed.cpp:197-209) of a tiled g16 handle: values and keep mask."""
    rng = np.random.default_rng(13)
    rows, cols = 48, 256
    g = 16 if groups == "g16" else np.where(np.arange(rows) % 2 == 0, 16, 64).astype(np.uint32)
    p, d = _layer(port, rng, rows, cols, g)
    want_v, want_m = port.unpack(p)
    got_v, got_m = d.dequant()
    assert np.array_equal(got_v.cpu().numpy().view(np.uint32), want_v.view(np.uint32))
    assert np.array_equal(got_m, want_m)


def test_grouped_decode_loop(port):
    """The KV-cached decode loop (egt_decoder_*) over g16 layers (fused Q/K/V,
    rmsnorm / silu / residual on the 16-column-group kernels): the last
    step's logits against the oracle's full-prefix forward."""
    import torch

    from paper_2605_11582_b200.model import Decoder
    from tests.test_gpu_verify import CFG, build_model

    model, oracle_forward = build_model(port, plan=[["int4-2:4"] * 6], group=16)
    dec = Decoder(model, 40)
    toks = dec.generate([3, 1, 4, 1, 5], 8)
    n = len(toks) - 1
    want = oracle_forward(np.array(toks[:n], np.int32), np.arange(n, dtype=np.int32), np.tril(np.ones((n, n), bool)))
    logits = torch.empty(CFG["vocab_size"], device="cuda")
    dec.read(logits)
    err = np.abs(logits.cpu().numpy() - want[n - 1]) / (1 + np.abs(want[n - 1]))
    assert err.max() <= 1e-3, err.max()
