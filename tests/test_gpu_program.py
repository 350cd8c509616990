"""GPU parity of the persistent GEMV program kernel (csrc/program.cu) against
the oracle: every op's product equals the oracle's spmv (packed.cpp:211-220)
of the transformed input, within |got-want| <= 1e-3 (1+|want|)
(test_packed.cpp:279); the input transforms follow rmsnorm
(model.cpp:57-67, oracle/egt_oracle.c rmsnorm) and silu (model.cpp:80-84)."""
import os

import numpy as np
import pytest

from tests.layers import close, make_f16, make_int4, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def egt():
    import paper_2605_11582_b200 as egt

    return egt


@pytest.fixture(scope="module")
def torch():
    import torch

    torch.cuda.init()
    return torch


def _dev(egt, p):
    return egt.DeviceMatrix.from_packed(to_product(p))


def rmsnorm32(x):
    """oracle/egt_oracle.c rmsnorm (model.cpp:57-67): f32, left to right."""
    x = np.asarray(x, np.float32)
    ss = np.float32(0)
    for v in x:
        ss = np.float32(ss + np.float32(v * v))
    inv = np.float32(1.0) / np.sqrt(np.float32(ss / np.float32(x.size) + np.float32(1e-6)))
    return (x * inv).astype(np.float32)


def silu32(x):
    x = np.asarray(x, np.float32)
    return (x * (np.float32(1) / (np.float32(1) + np.exp(-x)))).astype(np.float32)


def _cuda(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def test_independent_mixed_formats(egt, port, torch):
    """Independent ops of every tiled format and several shapes in one launch."""
    from paper_2605_11582_b200.program import Op, Program

    rng = np.random.default_rng(5)
    layers = [make_int4(rng, 4096, 4096, 2, 128, port)[0],
              make_int4(rng, 1040, 2048, 1, 64, port)[0],
              make_int4(rng, 512, 13824, 2, 32, port)[0],      # 108 k-quads: two panels
              make_f16(rng, 784, 1536, 2, port)[0],
              make_f16(rng, 96, 4096, 1, port)[0],
              make_int4(rng, 11008, 4096, 2, 128, port)[0]]
    ds = [_dev(egt, p) for p in layers]
    assert all(d.path == "tiled-mma.sp" for d in ds)
    xs = [rng.uniform(-1, 1, p.cols).astype(np.float32) for p in layers]
    xt = [_cuda(torch, x) for x in xs]
    ys = [torch.full((p.rows,), float("nan"), device="cuda") for p in layers]
    prog = Program([Op(d, x, y) for d, x, y in zip(ds, xt, ys)])
    assert prog.info["grid"] >= 1 and prog.info["stages"] >= 2
    for rep in range(3):  # counters reset between launches
        for y in ys:
            y.fill_(float("nan"))
        prog.run()
        torch.cuda.synchronize()
        for p, x, y in zip(layers, xs, ys):
            ok, err = close(y.cpu().numpy(), port.spmv(p, x))
            assert ok, f"rep {rep} {p.rows}x{p.cols}: max rel err {err:.3e}"


def test_dense_int4_op(egt, port, torch):
    from paper_2605_11582_b200.program import Op, Program

    rng = np.random.default_rng(9)
    w = rng.uniform(-1, 1, (640, 2048)).astype(np.float32)
    q = egt.quantize_matrix(w, 64)
    d = egt.DeviceMatrix.dense_i4(q)
    assert d.path == "tiled-mma.sp"
    x = rng.uniform(-1, 1, 2048).astype(np.float32)
    y = torch.empty(640, device="cuda")
    Program([Op(d, _cuda(torch, x), y)]).run()
    want = d.spmv(_cuda(torch, x)).cpu().numpy()
    ok, err = close(y.cpu().numpy(), want)
    assert ok, err


def _decoder_chain(egt, port, torch, rng, d_model=1024, d_ff=2816, n_layers=2):
    """Attention-free decoder layers with the reference's glue
    (model.cpp:155-190): q = Wq rmsnorm(h); h += Wo q;
    f = Wff1 rmsnorm(h); h += Wff2 silu(f)."""
    from paper_2605_11582_b200.program import RMSNORM, SILU, Op

    h0 = rng.uniform(-1, 1, d_model).astype(np.float32)
    h = _cuda(torch, h0)
    ops, host = [], []
    for _ in range(n_layers):
        pq = make_int4(rng, d_model, d_model, 2, 128, port)[0]
        po = make_int4(rng, d_model, d_model, 2, 64, port)[0]
        p1 = make_int4(rng, d_ff, d_model, 2, 64, port)[0]
        p2 = make_int4(rng, d_model, d_ff, 1, 128, port)[0]
        q = torch.empty(d_model, device="cuda")
        f = torch.empty(d_ff, device="cuda")
        j = len(ops)
        ops.append(Op(_dev(egt, pq), h, q, input=RMSNORM, wait=j - 1))
        ops.append(Op(_dev(egt, po), q, h, residual=h, wait=j))
        ops.append(Op(_dev(egt, p1), h, f, input=RMSNORM, wait=j + 1))
        ops.append(Op(_dev(egt, p2), f, h, residual=h, input=SILU, wait=j + 2))
        host.append((pq, po, p1, p2))
    return h0, h, ops, host


def _decoder_oracle(port, h0, host):
    h = h0.copy()
    for pq, po, p1, p2 in host:
        q = port.spmv(pq, rmsnorm32(h))
        h = (h + port.spmv(po, q)).astype(np.float32)
        f = port.spmv(p1, rmsnorm32(h))
        h = (h + port.spmv(p2, silu32(f))).astype(np.float32)
    return h


def test_dependent_chain_transforms(egt, port, torch):
    """rmsnorm / silu input transforms, in-place residual, waits."""
    from paper_2605_11582_b200.program import Program

    rng = np.random.default_rng(17)
    h0, h, ops, host = _decoder_chain(egt, port, torch, rng)
    prog = Program(ops)
    want = _decoder_oracle(port, h0, host)
    for rep in range(3):
        h.copy_(_cuda(torch, h0))
        prog.run()
        torch.cuda.synchronize()
        ok, err = close(h.cpu().numpy(), want)
        assert ok, f"rep {rep}: max rel err {err:.3e}"


def test_small_grid_many_partials(egt, port, torch, monkeypatch):
    """A 7-CTA grid: row tiles split across CTAs and panels, reduced by the last
    arriver; also the 1-CTA grid (no partials across CTAs)."""
    from paper_2605_11582_b200.program import Op, Program

    rng = np.random.default_rng(23)
    layers = [make_int4(rng, 200, 13824, 2, 128, port)[0], make_int4(rng, 48, 4096, 1, 32, port)[0]]
    ds = [_dev(egt, p) for p in layers]
    xs = [rng.uniform(-1, 1, p.cols).astype(np.float32) for p in layers]
    for grid in ("7", "1", "333"):
        monkeypatch.setenv("EGT_PROGRAM_GRID", grid)
        ys = [torch.empty(p.rows, device="cuda") for p in layers]
        prog = Program([Op(d, _cuda(torch, x), y) for d, x, y in zip(ds, xs, ys)])
        for _ in range(2):
            prog.run()
            torch.cuda.synchronize()
            for p, x, y in zip(layers, xs, ys):
                ok, err = close(y.cpu().numpy(), port.spmv(p, x))
                assert ok, f"grid {grid} {p.rows}x{p.cols}: {err:.3e}"


def test_graph_capture_replay(egt, port, torch):
    from paper_2605_11582_b200.program import Program

    rng = np.random.default_rng(29)
    h0, h, ops, host = _decoder_chain(egt, port, torch, rng, n_layers=1)
    s = torch.cuda.Stream()
    prog = Program(ops, stream=s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            prog.run(s)
    want = _decoder_oracle(port, h0, host)
    for _ in range(3):
        h.copy_(_cuda(torch, h0))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        ok, err = close(h.cpu().numpy(), want)
        assert ok, err


def test_hazards_rejected(egt, port, torch):
    from paper_2605_11582_b200.native import InvalidArgument
    from paper_2605_11582_b200.program import Op, Program

    rng = np.random.default_rng(31)
    d = _dev(egt, make_int4(rng, 256, 256, 2, 32, port)[0])
    a, b, c = (torch.zeros(256, device="cuda") for _ in range(3))
    with pytest.raises(InvalidArgument, match="depends on op 0"):
        Program([Op(d, a, b), Op(d, b, c)])          # RAW without wait
    with pytest.raises(InvalidArgument, match="depends on op 0"):
        Program([Op(d, a, b), Op(d, c, a)])          # WAR without wait
    with pytest.raises(InvalidArgument, match="x overlaps y"):
        Program([Op(d, a, a)])
    with pytest.raises(InvalidArgument, match="input length"):
        Program([Op(d, torch.zeros(128, device="cuda"), b)])
    Program([Op(d, a, b), Op(d, b, c, wait=0)])      # ordered: accepted


@pytest.mark.parametrize("M", [1, 5])
@pytest.mark.parametrize("shape", [(1024, 2048), (256, 11008)])
def test_spmv_fused_transforms(egt, port, torch, M, shape):
    """egt_spmv_fused: rmsnorm / silu input transforms and the residual epilogue
    (in place) of the per-launch kernel equal the oracle's composition."""
    from paper_2605_11582_b200.native import INPUT_NONE, INPUT_RMSNORM, INPUT_SILU

    rng = np.random.default_rng(41 + M)
    rows, cols = shape
    p = make_int4(rng, rows, cols, 2, 64, port)[0]
    d = _dev(egt, p)
    xs = rng.uniform(-2, 2, (M, cols)).astype(np.float32)
    rs = rng.uniform(-1, 1, (M, rows)).astype(np.float32)
    for mode, f in ((INPUT_NONE, lambda v: v), (INPUT_RMSNORM, rmsnorm32), (INPUT_SILU, silu32)):
        x = _cuda(torch, xs)
        y = _cuda(torch, rs)  # residual in place
        d.spmv_fused_into(x if M > 1 else x[0], y if M > 1 else y[0], residual=y if M > 1 else y[0], input=mode)
        got = y.cpu().numpy()
        for m in range(M):
            want = rs[m] + port.spmv(p, f(xs[m]))
            ok, err = close(got[m], want)
            assert ok, f"mode {mode} token {m}: {err:.3e}"


def test_spmv_fused_output_silu(egt, port, torch):
    """EGT_SPMV_OUTPUT_SILU: y = silu(W rmsnorm(x)) -- the ff1 product of the
    decode step applying ff2's input transform once per element."""
    from paper_2605_11582_b200.native import INPUT_RMSNORM

    rng = np.random.default_rng(61)
    p = make_int4(rng, 2816, 1024, 2, 128, port)[0]
    d = _dev(egt, p)
    x = rng.uniform(-2, 2, 1024).astype(np.float32)
    y = torch.empty(2816, device="cuda")
    d.spmv_fused_into(_cuda(torch, x), y, input=INPUT_RMSNORM, output_silu=True)
    ok, err = close(y.cpu().numpy(), silu32(port.spmv(p, rmsnorm32(x))))
    assert ok, err


@pytest.mark.parametrize("input_", [0, 1])
def test_spmv_fused_multi_qkv(egt, port, torch, input_):
    """egt_spmv_fused_multi: three same-shape matrices over one x in one
    launch (the decode step's Q, K, V) equal three separate products."""
    from paper_2605_11582_b200.native import InvalidArgument
    from paper_2605_11582_b200.packed import spmv_fused_multi

    rng = np.random.default_rng(71 + input_)
    ps = [make_int4(rng, 1024, 2048, 2, 128, port)[0] for _ in range(3)]
    ds = [_dev(egt, p) for p in ps]
    x = rng.uniform(-2, 2, 2048).astype(np.float32)
    ys = [torch.full((1024,), float("nan"), device="cuda") for _ in range(3)]
    spmv_fused_multi(ds, _cuda(torch, x), ys, input=input_)
    xin = rmsnorm32(x) if input_ == 1 else x
    for p, y in zip(ps, ys):
        ok, err = close(y.cpu().numpy(), port.spmv(p, xin))
        assert ok, err
    other = _dev(egt, make_int4(rng, 512, 2048, 2, 128, port)[0])
    with pytest.raises(InvalidArgument, match="share shape"):
        spmv_fused_multi([ds[0], other], _cuda(torch, x), ys[:2])
