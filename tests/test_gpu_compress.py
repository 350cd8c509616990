"""GPU compression: importance_scores, prune_nm and
quantize_matrix + pack on the device, byte-identical to the oracle port
(itself pinned to the unmodified reference: tests/test_oracle_golden.py)."""
import numpy as np
import pytest

from oracle.oracle import random_nm_mask

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


def _cuda(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("shape", [(7, 13), (64, 256), (300, 1030)])
def test_importance_bit_exact(egt, port, torch, shape):
    rng = np.random.default_rng(shape[0])
    w = rng.normal(size=shape).astype(np.float32)
    xn = rng.uniform(0, 3, shape[1]).astype(np.float32)
    g = np.abs(rng.normal(size=shape)).astype(np.float32)
    got = egt.gpu_importance(_cuda(torch, w), _cuda(torch, xn), _cuda(torch, g)).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), port.importance(w, xn, g).view(np.uint32))


@pytest.mark.parametrize("shape", [(5, 13), (33, 130), (256, 4096)])
@pytest.mark.parametrize("n", [1, 2, 3])
def test_prune_nm_bit_exact(egt, port, torch, shape, n):
    """Ties (scores rounded to 0.5), zero and negative scores, a short last group."""
    rng = np.random.default_rng(shape[1] + n)
    s = (np.round(rng.normal(size=shape) * 2) / 2).astype(np.float32)
    got = egt.gpu_prune_nm(_cuda(torch, s), n).cpu().numpy()
    assert np.array_equal(got, port.prune_nm(s, n))


def test_prune_nm_errors(egt, torch):
    s = torch.ones((4, 8), device="cuda")
    with pytest.raises(egt.InvalidArgument, match="group width must be 4"):
        egt.gpu_prune_nm(s, 2, m=8)
    with pytest.raises(egt.InvalidArgument, match="keep count"):
        egt.gpu_prune_nm(s, 4)


def _host(port, w, mask, n, gs):
    rows, cols = w.shape
    q = port.quantize(w, gs, mask)
    return port.pack_int4(mask, rows, cols, q, n)


CASES = [  # rows, cols, n, group sizes (int or per-row list)
    (16, 128, 2, 128),
    (48, 640, 2, 100),        # ragged last group
    (40, 1024, 1, 64),
    (33, 512, 2, [64, 128, 512, 1000] * 8 + [32]),  # per-row (adaptive) group sizes, g > cols
    (257, 4096, 2, 128),
    (129, 2048, 1, 128),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}-n{c[2]}" for c in CASES])
def test_quantize_pack_byte_exact(egt, port, torch, case):
    rows, cols, n, g = case
    rng = np.random.default_rng(rows * 7 + cols)
    w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
    w[0, :8] = 0.0  # flat / zero groups
    mask = random_nm_mask(rng, rows, cols, n)
    gs = np.broadcast_to(np.asarray(g, np.uint32), (rows,)).copy()
    want = _host(port, w, mask, n, gs)
    d, raw = egt.gpu_quantize_pack(_cuda(torch, w), _cuda(torch, mask), n, gs)
    assert np.array_equal(raw["index_words"].cpu().numpy().view(np.uint16), want.index_words)
    assert np.array_equal(raw["value_bytes"].cpu().numpy(), want.value_bytes)
    assert np.array_equal(raw["group_offsets"].cpu().numpy().view(np.uint32), want.group_offsets)
    assert np.array_equal(raw["scales"].cpu().numpy().view(np.uint32), want.scales.view(np.uint32))
    assert np.array_equal(raw["zero_points"].cpu().numpy(), want.zero_points)
    # the device matrix equals the one uploaded from the host arrays
    from tests.layers import to_product

    h = egt.DeviceMatrix.from_packed(to_product(want))
    x = torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda()
    assert torch.equal(d.spmv(x), h.spmv(x))
    wd, md = d.dequant()
    wh, mh = h.dequant()
    assert torch.equal(wd, wh) and np.array_equal(md, mh)


def test_quantize_pack_full_size(egt, port, torch):
    """11008 x 4096 (the 7B up-projection), byte-exact."""
    rng = np.random.default_rng(11008)
    w = rng.uniform(-1, 1, (11008, 4096)).astype(np.float32)
    mask = random_nm_mask(rng, 11008, 4096, 2)
    gs = np.full(11008, 128, np.uint32)
    want = _host(port, w, mask, 2, gs)
    _, raw = egt.gpu_quantize_pack(_cuda(torch, w), _cuda(torch, mask), 2, gs, want_matrix=False)
    assert np.array_equal(raw["index_words"].cpu().numpy().view(np.uint16), want.index_words)
    assert np.array_equal(raw["value_bytes"].cpu().numpy(), want.value_bytes)
    assert np.array_equal(raw["scales"].cpu().numpy(), want.scales)
    assert np.array_equal(raw["zero_points"].cpu().numpy(), want.zero_points)


def test_pipeline_importance_prune_pack(egt, port, torch):
    """importance -> prune_nm(2:4) -> quantize + pack on the device, against
    the oracle running the same three steps, then the product."""
    from tests.layers import close

    rng = np.random.default_rng(3)
    rows, cols = 272, 1536
    w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
    xn = rng.uniform(0.5, 2, cols).astype(np.float32)
    ga = np.abs(rng.normal(size=(rows, cols))).astype(np.float32)
    s_dev = egt.gpu_importance(_cuda(torch, w), _cuda(torch, xn), _cuda(torch, ga))
    m_dev = egt.gpu_prune_nm(s_dev, 2)
    d, raw = egt.gpu_quantize_pack(_cuda(torch, w), m_dev, 2, 128)
    mask = port.prune_nm(port.importance(w, xn, ga), 2)
    assert np.array_equal(m_dev.cpu().numpy(), mask)
    want = _host(port, w, mask, 2, np.full(rows, 128, np.uint32))
    assert np.array_equal(raw["value_bytes"].cpu().numpy(), want.value_bytes)
    x = rng.uniform(-1, 1, cols).astype(np.float32)
    ok, err = close(d.spmv(_cuda(torch, x)).cpu().numpy(), port.spmv(want, x))
    assert ok, err


def test_quantize_pack_errors_match_host(egt, port, torch):
    rng = np.random.default_rng(4)
    w = rng.uniform(-1, 1, (8, 64)).astype(np.float32)
    b = np.zeros((8, 64), bool)
    b[:, 0::2] = True
    b[5, 20:24] = [True, True, True, False]  # row 5, column 20 keeps 3
    mask = np.packbits(b.reshape(-1), bitorder="little")
    with pytest.raises(egt.InvalidArgument) as gpu_err:
        egt.gpu_quantize_pack(_cuda(torch, w), _cuda(torch, mask), 2, 64)
    q = egt.quantize_matrix(w, 64, mask)
    with pytest.raises(egt.InvalidArgument) as host_err:
        egt.pack(mask, q, 2)
    assert str(gpu_err.value) == str(host_err.value)
    assert "row 5, column 20 keeps 3 entries (want 2)" in str(gpu_err.value)
    with pytest.raises(egt.InvalidArgument, match="multiple of the group width"):
        egt.gpu_quantize_pack(_cuda(torch, w[:, :62].copy()), _cuda(torch, mask), 2, 64)
    with pytest.raises(egt.InvalidArgument, match="zero group size"):
        egt.gpu_quantize_pack(_cuda(torch, w), _cuda(torch, mask), 2, 0)
