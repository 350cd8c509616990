"""The tcgen05 / TMEM many-token kernel (csrc/umma_spmm.cu) against the port's
f32 spmv (packed.cpp:211-220) / quant_dense_gemv (packed.cpp:266-281), token
by token: every format it takes (INT4 2:4, INT4 1:4 stored as 2:4, dense
INT4, FP16 2:4), 64- and 128-column scale groups, ragged rows / columns,
one and several token tiles, split-K, the fused residual / silu epilogue,
and the SASS evidence that the kernel runs on tcgen05 (UTCHMMA / LDTM)."""
import os
import subprocess

import numpy as np
import pytest

from tests.layers import close, make_f16, make_int4, to_product

pytestmark = pytest.mark.gpu


def _layer(port, rng, fmt, rows, cols, group=128):
    import paper_2605_11582_b200 as egt

    if fmt == "int4-dense":
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        q = port.quantize(w, np.full(rows, group, np.uint32))
        from paper_2605_11582_b200.packed import QuantizedMatrix

        qm = QuantizedMatrix(q.rows, q.cols, q.group_sizes, q.group_offsets, q.scales, q.zero_points, q.codes)
        return egt.DeviceMatrix.dense_i4(qm), (lambda x: port.quant_dense_gemv(q, x))
    n = 2 if fmt.endswith("2:4") else 1
    if fmt.startswith("int4"):
        p, _, _ = make_int4(rng, rows, cols, n, group, port)
    else:
        p, _, _ = make_f16(rng, rows, cols, n, port)
    return egt.DeviceMatrix.from_packed(to_product(p)), (lambda x: port.spmv(p, x))


@pytest.mark.parametrize("fmt", ["int4-2:4", "int4-1:4", "int4-dense", "fp16-2:4"])
@pytest.mark.parametrize("M", [9, 16, 17, 80, 130, 272])
def test_umma_products(port, fmt, M):
    import torch

    rng = np.random.default_rng(M + len(fmt))
    # ragged 128-row tile / k-quads; a 7B shape; several token tiles run on
    # tcgen05 for tall matrices (umma_eligible)
    rows, cols = {17: (400, 1408), 80: (4096, 4096)}.get(M, (8200, 640))
    d, ref = _layer(port, rng, fmt, rows, cols)
    xs = rng.uniform(-1, 1, (M, cols)).astype(np.float32)
    y = d.spmv(torch.from_numpy(xs).cuda()).cpu().numpy()
    for m in range(M):
        ok, err = close(y[m], ref(xs[m]))
        assert ok, (fmt, M, m, err)


@pytest.mark.parametrize("group", [64, 128])
def test_umma_group_sizes_and_split_k(port, group):
    """64 x 11008 at M = 40: few row tiles, so the plan splits K."""
    import torch

    rng = np.random.default_rng(group)
    d, ref = _layer(port, rng, "int4-2:4", 64, 11008, group)
    xs = rng.uniform(-1, 1, (40, 11008)).astype(np.float32)
    for _ in range(3):  # replays: the split-K counters reset themselves
        y = d.spmv(torch.from_numpy(xs).cuda()).cpu().numpy()
        for m in range(40):
            ok, err = close(y[m], ref(xs[m]))
            assert ok, (group, m, err)


def test_umma_fused_epilogue(port):
    """y = silu(res + x W^T) in the epilogue (model.cpp:186-190 glue)."""
    import torch

    rng = np.random.default_rng(3)
    rows, cols, M = 256, 1024, 48
    d, ref = _layer(port, rng, "int4-2:4", rows, cols)
    xs = rng.uniform(-1, 1, (M, cols)).astype(np.float32)
    res = rng.uniform(-1, 1, (M, rows)).astype(np.float32)
    y = torch.empty((M, rows), device="cuda")
    d.spmv_fused_into(torch.from_numpy(xs).cuda(), y, residual=torch.from_numpy(res).cuda(), output_silu=True)
    got = y.cpu().numpy()
    for m in range(M):
        pre = res[m] + ref(xs[m])
        want = pre / (1 + np.exp(-pre.astype(np.float64)))
        ok, err = close(got[m], want)
        assert ok, (m, err)


def test_umma_sass_is_tcgen05():
    """The built library carries the tcgen05 MMA, TMEM loads and bulk copies."""
    from paper_2605_11582_b200.native import LIB_PATH

    out = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True)
    sass = out.stdout
    if out.returncode != 0 or not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass and "LDTM" in sass and "UBLKCP" in sass and "UTMALDG" in sass


@pytest.mark.parametrize("fmt", ["int4-2:4", "fp16-2:4", "int4-dense"])
@pytest.mark.parametrize("M", [40, 272])
def test_umma_multi_segments(port, fmt, M):
    """egt_spmm_multi: Q, K, V in one tcgen05 launch (one x preparation, CTAs
    per segment) give each matrix's own product."""
    import torch

    from paper_2605_11582_b200.packed import spmm_multi

    rng = np.random.default_rng(M + 7)
    rows, cols = 384, 1024
    mats = [_layer(port, rng, fmt, rows, cols) for _ in range(3)]
    xs = rng.uniform(-1, 1, (M, cols)).astype(np.float32)
    x = torch.from_numpy(xs).cuda()
    ys = [torch.empty((M, rows), device="cuda") for _ in range(3)]
    spmm_multi([d for d, _ in mats], x, ys)
    for (d, ref), y in zip(mats, ys):
        got = y.cpu().numpy()
        for m in range(0, M, 7):
            ok, err = close(got[m], ref(xs[m]))
            assert ok, (fmt, M, m, err)


@pytest.mark.parametrize("M", [12, 80])
def test_umma_rmsnorm_input(port, M):
    """rmsnorm (model.cpp:57-67) folded into the tcgen05 x preparation, one
    matrix (egt_spmv_fused) and Q/K/V (egt_spmm_multi), including a row with
    an inf (the reference's rmsnorm then gives NaN there and 0 elsewhere)."""
    import torch

    from paper_2605_11582_b200 import native as N
    from paper_2605_11582_b200.packed import spmm_multi

    rng = np.random.default_rng(M + 3)
    rows, cols = 256, 1024
    mats = [_layer(port, rng, "int4-2:4", rows, cols) for _ in range(3)]
    xs = rng.uniform(-3, 3, (M, cols)).astype(np.float32)
    xs[1, 7] = np.inf
    eps = 1e-6
    xn = np.empty_like(xs)
    for m in range(M):
        inv = np.float32(1.0) / np.sqrt(np.float32(np.mean(xs[m].astype(np.float64) ** 2)) + np.float32(eps))
        xn[m] = xs[m] * inv
    x = torch.from_numpy(xs).cuda()
    y = torch.empty((M, rows), device="cuda")
    mats[0][0].spmv_fused_into(x, y, input=N.INPUT_RMSNORM, eps=eps)
    ys = [torch.empty((M, rows), device="cuda") for _ in range(3)]
    spmm_multi([d for d, _ in mats], x, ys, input=N.INPUT_RMSNORM, eps=eps)
    for got_all, (d, ref) in [(y, mats[0])] + list(zip(ys, mats)):
        got = got_all.cpu().numpy()
        for m in range(M):
            want = ref(xn[m])
            assert np.array_equal(np.isnan(got[m]), np.isnan(want)), m
            fin = np.isfinite(want)
            ok, err = close(got[m][fin], want[fin])
            assert ok, (M, m, err)


def test_spmm_multi_errors(port):
    """egt_spmm_multi's argument contract: 1..3 matrices sharing columns,
    identity or rmsnorm input, the reference-style EGT_EINVAL messages."""
    import torch

    import paper_2605_11582_b200 as egt
    from paper_2605_11582_b200 import native as N
    from paper_2605_11582_b200.packed import spmm_multi

    rng = np.random.default_rng(4)
    a, _ = _layer(port, rng, "int4-2:4", 128, 256)
    b, _ = _layer(port, rng, "int4-2:4", 128, 512)
    x = torch.zeros((20, 256), device="cuda")
    ys = [torch.empty((20, 128), device="cuda") for _ in range(4)]
    with pytest.raises(egt.InvalidArgument, match="1 to 3 matrices"):
        spmm_multi([a, a, a, a], x, ys)
    with pytest.raises(egt.InvalidArgument, match="share their columns"):
        spmm_multi([a, b], x, ys[:2])
    with pytest.raises(egt.InvalidArgument, match="none or rmsnorm"):
        spmm_multi([a, a], x, ys[:2], input=N.INPUT_SILU)


@pytest.mark.parametrize("M", [130, 272])
def test_umma_split_k_with_token_tiles(port, M):
    """Few row blocks, several token tiles: the planner splits K across a
    cluster per (row block, token tile) and the slices push their partial
    shares to each other (umma_spmm.cu push path)."""
    import torch

    rng = np.random.default_rng(M + 11)
    d, ref = _layer(port, rng, "int4-2:4", 256, 4096)
    xs = rng.uniform(-1, 1, (M, 4096)).astype(np.float32)
    res = rng.uniform(-1, 1, (M, 256)).astype(np.float32)
    y = torch.empty((M, 256), device="cuda")
    d.spmv_fused_into(torch.from_numpy(xs).cuda(), y, residual=torch.from_numpy(res).cuda())
    got = y.cpu().numpy()
    for m in range(M):
        ok, err = close(got[m], res[m] + ref(xs[m]))
        assert ok, (M, m, err)
