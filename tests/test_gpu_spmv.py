"""GPU parity: the sm_100a kernels (through the C-ABI) against the oracle on
identical seeded inputs.  Bit-exact for the device copy of the encoding
(dequantised values + recovered keep mask); |got-want| <= 1e-3 (1+|want|)
for products (the reference's own convention, test_packed.cpp:279)."""
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


def _check_product(egt, port, torch, p, rng, M=1, expect_path=None):
    d = _dev(egt, p)
    if expect_path:
        assert d.path == expect_path, d.path
    xs = rng.uniform(-1, 1, (M, p.cols)).astype(np.float32)
    x = torch.from_numpy(xs).cuda()
    y = d.spmv(x if M > 1 else x[0]).cpu().numpy().reshape(M, -1)
    for m in range(M):
        want = port.spmv(p, xs[m])
        ok, err = close(y[m], want)
        assert ok, f"token {m}: max rel err {err:.3e} ({d.format}, {d.path}, {p.rows}x{p.cols})"
    return d


@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_int4_2of4_g128_baseline_shapes(egt, port, torch, shape):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    p, _, _ = make_int4(rng, shape[0], shape[1], 2, 128, port)
    d = _check_product(egt, port, torch, p, rng, expect_path="tiled-mma.sp")
    assert d.format == "int4-2:4"
    assert d.algorithmic_bytes == port.footprint(p)["packed_bytes"]


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("group", [32, 64, 128, 256, "mixed"])
def test_int4_group_sizes(egt, port, torch, n, group):
    rng = np.random.default_rng(11 + n)
    rows, cols = 272, 1024
    g = np.where(rng.random(rows) < 0.5, 64, 128) if group == "mixed" else group
    p, _, _ = make_int4(rng, rows, cols, n, g, port)
    _check_product(egt, port, torch, p, rng, expect_path="tiled-mma.sp")


@pytest.mark.parametrize("n", [1, 2])
def test_int4_ragged_edges(egt, port, torch, n):
    """rows not a multiple of 16, cols a multiple of 32 but not of 128."""
    rng = np.random.default_rng(21)
    for rows, cols in ((1, 32), (17, 96), (33, 160), (250, 4000 - 4000 % 32)):
        p, _, _ = make_int4(rng, rows, cols, n, 32, port)
        _check_product(egt, port, torch, p, rng, expect_path="tiled-mma.sp")


@pytest.mark.parametrize("n", [1, 2])
def test_general_path_any_group(egt, port, torch, n):
    """Group sizes that do not sit on 32-column k-tiles, and cols % 32 != 0,
    run on the reference-order CUDA-core kernel."""
    rng = np.random.default_rng(31)
    for rows, cols, g in ((7, 36, 4), (64, 512, 16), (40, 200, 48), (3, 8, 8), (128, 1000, 100)):
        p, _, _ = make_int4(rng, rows, cols, n, g, port)
        # 16-column groups on 32-column k-tiles run tiled (two mma.sp per k-tile)
        path = "tiled-mma.sp" if g % 16 == 0 and cols % 32 == 0 else "general"
        _check_product(egt, port, torch, p, rng, expect_path=path)


@pytest.mark.parametrize("n", [1, 2])
def test_sparse_fp16(egt, port, torch, n):
    rng = np.random.default_rng(41)
    for rows, cols in ((4096, 4096), (100, 96)):
        p, _, _ = make_f16(rng, rows, cols, n, port)
        d = _check_product(egt, port, torch, p, rng, expect_path="tiled-mma.sp")
        assert d.format == f"fp16-{n}:4"
    p, _, _ = make_f16(rng, 9, 36, n, port)
    _check_product(egt, port, torch, p, rng, expect_path="general")


def test_dense_int4(egt, port, torch):
    """quant_dense_gemv semantics (packed.cpp:266-281)."""
    rng = np.random.default_rng(51)
    for rows, cols, g, path in ((4096, 4096, 128, "tiled-mma.sp"), (48, 96, 32, "tiled-mma.sp"),
                                (20, 40, 8, "general")):
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        q = egt.quantize_matrix(w, g)
        d = egt.DeviceMatrix.dense_i4(q)
        assert d.path == path and d.format == "int4-dense"
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        y = d.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        from oracle.oracle import Quantized

        qo = Quantized(rows, cols, q.group_sizes, q.group_offsets, q.scales, q.zero_points, q.codes)
        ok, err = close(y, port.quant_dense_gemv(qo, x))
        assert ok, err
        vals, bits = d.dequant()
        assert np.array_equal(vals.cpu().numpy().view(np.uint32), port.dequantize(qo).view(np.uint32))
        assert np.unpackbits(bits, bitorder="little")[: rows * cols].all()


@pytest.mark.parametrize("kind", ["int4-2", "int4-1", "fp16-2", "fp16-1", "int4-general"])
def test_dequant_bit_exact(egt, port, torch, kind):
    """The device copy of the encoding reproduces the reference's unpack bit
    for bit: values (decode_value in f32) and the recovered keep mask."""
    rng = np.random.default_rng(61)
    for rows, cols in ((64, 512), (37, 160), (16, 32)):
        if kind.startswith("int4-general"):
            p, mask, _ = make_int4(rng, rows, cols + 4, 2, 12, port)
        elif kind.startswith("int4"):
            p, mask, _ = make_int4(rng, rows, cols, int(kind[-1]), 32, port)
        else:
            p, mask, _ = make_f16(rng, rows, cols, int(kind[-1]), port)
        want_v, want_m = port.unpack(p)
        got_v, got_m = _dev(egt, p).dequant()
        assert np.array_equal(got_v.cpu().numpy().view(np.uint32), want_v.view(np.uint32))
        assert np.array_equal(got_m, want_m)
        assert np.array_equal(got_m, mask)


@pytest.mark.parametrize("M", [2, 3, 4, 5, 8, 9, 16, 33])
def test_multi_token(egt, port, torch, M):
    """M-row products (the verify pass's skinny SpGEMM) per token vs oracle."""
    rng = np.random.default_rng(71 + M)
    p, _, _ = make_int4(rng, 528, 768, 2, 128, port)
    _check_product(egt, port, torch, p, rng, M=M)
    p, _, _ = make_int4(rng, 130, 256, 1, 64, port)
    _check_product(egt, port, torch, p, rng, M=M)


def test_row_shards_zero_copy(egt, port, torch):
    rng = np.random.default_rng(81)
    p, _, _ = make_int4(rng, 1024, 2048, 2, 128, port)
    d = _dev(egt, p)
    x = rng.uniform(-1, 1, p.cols).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    full = d.spmv(xt).cpu().numpy()
    for G in (2, 4, 8):
        per = p.rows // G
        parts = [d.slice_rows(i * per, (i + 1) * per).spmv(xt).cpu().numpy() for i in range(G)]
        assert close(np.concatenate(parts), full, 1e-5)[0]  # split-K plans may differ per shard
    tail = d.slice_rows(1008, 1024).spmv(xt).cpu().numpy()
    assert close(tail, full[1008:], 1e-5)[0]
    with pytest.raises(egt.InvalidArgument):
        d.slice_rows(8, 40)


def test_host_drop_in_and_errors(egt, port, torch):
    rng = np.random.default_rng(91)
    p, _, _ = make_int4(rng, 300, 640, 2, 128, port)
    x = rng.uniform(-1, 1, 640).astype(np.float32)
    y = egt.spmv(to_product(p), x)
    assert close(y, port.spmv(p, x))[0]
    d = _dev(egt, p)
    assert np.array_equal(d.spmv_host(x), d.spmv(torch.from_numpy(x).cuda()).cpu().numpy())
    with pytest.raises(egt.InvalidArgument, match="input length differs from columns"):
        d.spmv_host(np.ones(641, np.float32))
    bad = to_product(p)
    bad.index_words = bad.index_words.copy()
    first = (int(bad.index_words[0]) >> 14) & 3
    bad.index_words[0] = (int(bad.index_words[0]) & 0x0FFF) | (first << 14) | (first << 12)
    with pytest.raises(egt.FormatError, match="offsets"):
        egt.DeviceMatrix.from_packed(bad)
    short = to_product(p)
    short.value_bytes = short.value_bytes[:-1]
    with pytest.raises(egt.FormatError, match="value byte count"):
        egt.DeviceMatrix.from_packed(short)


def test_empty_shapes(egt, port, torch):
    rng = np.random.default_rng(101)
    p, _, _ = make_int4(rng, 0, 64, 2, 32, port)
    d = _dev(egt, p)
    assert d.spmv_host(np.zeros(64, np.float32)).size == 0
    p, _, _ = make_int4(rng, 5, 0, 2, 32, port)
    d = _dev(egt, p)
    assert np.array_equal(d.spmv_host(np.zeros(0, np.float32)), np.zeros(5, np.float32))


def test_graph_replay_chain(egt, port, torch):
    """A CUDA-graph-captured chain with PDL (y of one GEMV feeds the next)
    equals eager execution, replayed several times (split-K counters reset)."""
    rng = np.random.default_rng(111)
    layers = [make_int4(rng, 4096, 4096, 2, 128, port)[0] for _ in range(3)]
    ds = [_dev(egt, p) for p in layers]
    x0 = torch.from_numpy(rng.uniform(-1, 1, 4096).astype(np.float32)).cuda()
    bufs = [torch.empty(4096, device="cuda") for _ in range(3)]

    def chain(x):
        for d, b in zip(ds, bufs):
            d.spmv_into(x, b)
            x = b
        return x

    eager = chain(x0).clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        chain(x0)  # warm-up allocates the workspace outside capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            chain(x0)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(bufs[-1], eager)
    want = x0.cpu().numpy()
    for p in layers:
        want = port.spmv(p, want)
    scale = float(np.sqrt(np.mean(want.astype(np.float64) ** 2)))  # chained magnitudes grow ~30x/layer
    assert close(eager.cpu().numpy() / scale, want / scale)[0]


def test_effective_matrix_probe(egt, port, torch, tmp_path):
    """X = I recovers the matrix the tensor cores actually multiply by; it
    must equal the reference's unpack exactly (small integers x scale 1)."""
    import json
    import os

    rng = np.random.default_rng(121)
    for n in (2, 1):
        rows, cols = 16, 128
        p, _, _ = make_int4(rng, rows, cols, n, 128, port)
        d = _dev(egt, p)
        eye = torch.eye(cols, dtype=torch.float32, device="cuda")
        w_eff = d.spmv(eye).cpu().numpy().T  # [rows x cols]
        want, _ = port.unpack(p)
        if not np.allclose(w_eff, want, rtol=1e-5, atol=1e-6):
            out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
            os.makedirs(out, exist_ok=True)
            with open(os.path.join(out, f"probe_n{n}.json"), "w") as f:
                json.dump({"w_eff": w_eff.tolist(), "want": want.tolist()}, f)
        assert np.allclose(w_eff, want, rtol=1e-5, atol=1e-6), f"n={n}: tensor-core layout mismatch"


def test_sharded_spmv_nccl_single_rank(egt, port, torch):
    """ShardedSpmv over an NCCL group (world 1 on one GPU): local shard
    product + all-gather equals the unsharded product."""
    import os

    import torch.distributed as dist

    from paper_2605_11582_b200.parallel import ShardedSpmv

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(131)
        p, _, _ = make_int4(rng, 640, 1024, 2, 128, port)
        d = _dev(egt, p)
        sh = ShardedSpmv(d)
        x = torch.from_numpy(rng.uniform(-1, 1, 1024).astype(np.float32)).cuda()
        assert torch.equal(sh(x), d.spmv(x))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [9, 16, 17, 33, 80])
def test_multi_token_wide(egt, port, torch, M):
    """M-row products on a 4096-wide layer (the 7B verify pass): the planner
    must find a (multi-wave) plan when one wave cannot hold the x fragments."""
    rng = np.random.default_rng(171 + M)
    p, _, _ = make_int4(rng, 1040, 4096, 2, 128, port)
    _check_product(egt, port, torch, p, rng, M=M)


@pytest.mark.parametrize("kind", ["int4-1:4-g64", "int4-2:4-g32", "fp16-2:4", "fp16-1:4"])
@pytest.mark.parametrize("M", [17, 40, 272])
def test_many_token_formats(egt, port, torch, kind, M):
    """The many-token kernel (spmm_wide.cu, M > 16) for every tiled format."""
    rng = np.random.default_rng(191 + M + len(kind))
    if kind.startswith("int4"):
        n = 1 if "1:4" in kind else 2
        p, _, _ = make_int4(rng, 272, 1536, n, int(kind.split("-g")[1]), port)
    else:
        p, _, _ = make_f16(rng, 272, 1536, 1 if "1:4" in kind else 2, port)
    _check_product(egt, port, torch, p, rng, M=M)


@pytest.mark.parametrize("M", [18, 64])
def test_many_token_dense_int4(egt, port, torch, M):
    rng = np.random.default_rng(301 + M)
    w = rng.uniform(-1, 1, (400, 2048)).astype(np.float32)
    q = egt.quantize_matrix(w, 64)
    d = egt.DeviceMatrix.dense_i4(q)
    xs = rng.uniform(-1, 1, (M, 2048)).astype(np.float32)
    y = d.spmv(torch.from_numpy(xs).cuda()).cpu().numpy()
    qo = port.quantize(w, np.full(400, 64, np.uint32), None)
    for m in (0, M // 2, M - 1):
        ok, err = close(y[m], port.quant_dense_gemv(qo, xs[m]))
        assert ok, err


@pytest.mark.parametrize("shape", [(5120, 13824), (8192, 28672)])
def test_baseline_sharded_shapes_full_size(egt, port, torch, shape):
    """BASELINE config[4] at full size: the unsharded product against the
    oracle, and the 2/4/8-way row shards (parallel.RowShardPlan) reassembled
    against the unsharded product (the all-gather is a concatenation)."""
    from paper_2605_11582_b200.parallel import RowShardPlan

    rows, cols = shape
    rng = np.random.default_rng(rows)
    p, _, _ = make_int4(rng, rows, cols, 2, 128, port)
    d = _dev(egt, p)
    x = rng.uniform(-1, 1, cols).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    full = d.spmv(xt).cpu().numpy()
    ok, err = close(full, port.spmv(p, x))
    assert ok, err
    for G in (2, 4, 8):
        plan = RowShardPlan.make(rows, G)
        parts = [d.slice_rows(r0, r1).spmv(xt).cpu().numpy() for r0, r1 in plan.bounds]
        ok, err = close(np.concatenate(parts), full, 1e-5)
        assert ok, (G, err)


@pytest.mark.parametrize("M", [17, 80])
def test_many_token_fused_epilogue(egt, port, torch, M):
    """The many-token kernel's epilogue glue (the verify forward's
    x += o Wo^T and silu(b ff1^T), model.cpp:186-190): y = silu(res + X W^T)
    and y = y + X W^T in place, against the plain product."""
    rng = np.random.default_rng(300 + M)
    p, _, _ = make_int4(rng, 272, 1536, 2, 128, port)
    d = _dev(egt, p)
    x = torch.from_numpy(rng.uniform(-1, 1, (M, p.cols)).astype(np.float32)).cuda()
    res = torch.from_numpy(rng.uniform(-1, 1, (M, p.rows)).astype(np.float32)).cuda()
    plain = d.spmv(x)
    y = torch.empty_like(res)
    d.spmv_fused_into(x, y, residual=res, output_silu=True)
    want = res + plain
    want = want * torch.sigmoid(want)
    assert torch.allclose(y, want, rtol=1e-6, atol=1e-6)
    acc = res.clone()
    d.spmv_fused_into(x, acc, residual=acc)
    assert torch.equal(acc, res + plain)


def test_gemv_f32_dense_baseline(egt, torch):
    """The dense-FP arm (egt_gemv_f32) against a float64 product."""
    rng = np.random.default_rng(55)
    for rows, cols in [(7, 13), (300, 1024)]:
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        y = egt.gemv_f32(torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda()).cpu().numpy()
        want = w.astype(np.float64) @ x.astype(np.float64)
        assert np.max(np.abs(y - want) / (1 + np.abs(want))) < 1e-5


def test_bench_spmv_harness(egt, torch):
    """bench_spmv / bench_csv (packed.cpp:310-393) on the device: the
    reference's CSV layout, variant order and analytic bytes (checked against
    the unmodified reference harness when oracle/_ref is built), its errors."""
    import os

    csv = egt.bench_spmv([(256, 512)], reps=3, seed=11)
    lines = csv.strip().split("\n")
    assert lines[0] == "variant,rows,cols,pattern,median_ns,p95_ns,bytes"
    rows = [l.split(",") for l in lines[1:]]
    assert [(r[0], r[3]) for r in rows] == [("dense-fp", "dense"), ("quant-dense", "dense"),
                                            ("packed-2:4", "2:4"), ("packed-1:4", "1:4")]
    assert all(int(r[4]) > 0 and int(r[5]) >= int(r[4]) for r in rows)
    ref_lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                           "libegt_ref.so")
    if os.path.exists(ref_lib):
        from oracle.oracle import Oracle

        _, _, ref_bytes = Oracle("reference").ref_bench_spmv(256, 512, 1, 11)
        assert [int(r[6]) for r in rows] == ref_bytes
    with pytest.raises(egt.InvalidArgument, match="repetitions must be positive"):
        egt.bench_spmv([(16, 64)], reps=0)
    with pytest.raises(egt.InvalidArgument, match="multiple of 4"):
        egt.bench_spmv([(16, 66)], reps=1)
