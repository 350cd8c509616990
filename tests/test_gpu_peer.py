"""Row-sharded SparseGemv with the all-gather fused into the product kernel
(include/egt_b200.h egt_spmv_allgather).  Ranks are simulated on
the one GPU (their buffers all in its HBM; the kernels of the ranks run one
after another with EGT_PEER_NOWAIT, then each rank's wait), plus a real
two-process run over CUDA IPC on the same device.  Every rank's gathered y
must equal the concatenation of the shard products bit for bit (the fused
kernel is the same arithmetic), and the oracle within 1e-3 (1+|want|)."""
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


def _layer(egt, port, rng, kind, rows, cols):
    if kind == "fp16-2:4":
        p, _, _ = make_f16(rng, rows, cols, 2, port)
    else:
        p, _, _ = make_int4(rng, rows, cols, 1 if kind == "int4-1:4" else 2, 128, port)
    return p, egt.DeviceMatrix.from_packed(to_product(p))


def _run_local(torch, d, groups, plan, x, M):
    shards = [d.slice_rows(r0, r1) for r0, r1 in plan.bounds]
    for g, sh, (r0, _) in zip(groups, shards, plan.bounds):
        g.spmv(sh, x, r0, d.rows, nowait=True)
    for g in groups:
        g.wait()
    torch.cuda.synchronize()
    want = torch.cat([sh.spmv(x) for sh in shards], dim=-1)
    shape = (d.rows,) if M == 1 else (M, d.rows)
    return [g.y(shape).clone() for g in groups], want


@pytest.mark.parametrize("kind", ["int4-2:4", "int4-1:4", "fp16-2:4"])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M", [1, 4])
def test_fused_allgather_local_ranks(egt, port, torch, kind, world, M):
    from paper_2605_11582_b200.parallel import PeerGroup, RowShardPlan

    rng = np.random.default_rng(7 + world + 10 * M)
    p, d = _layer(egt, port, rng, kind, 656, 1536)
    plan = RowShardPlan.make(d.rows, world)
    groups = PeerGroup.local_ranks(world, M * d.rows)
    for rep in range(3):  # the arrival counters keep counting across calls
        xs = rng.uniform(-1, 1, (M, d.cols)).astype(np.float32)
        x = torch.from_numpy(xs).cuda()
        x = x[0] if M == 1 else x
        ys, want = _run_local(torch, d, groups, plan, x, M)
        for r, y in enumerate(ys):
            assert torch.equal(y, want), (rep, r)
        got = ys[0].cpu().numpy().reshape(M, -1)
        for m in range(M):
            ok, err = close(got[m], port.spmv(p, xs[m]))
            assert ok, err
    for g in groups:
        g.check()


def test_fused_allgather_in_kernel_wait_and_graph(egt, port, torch):
    """world 1: the kernel's own last CTA signals and waits; a CUDA graph of
    the call replays (device-side sequence numbers)."""
    from paper_2605_11582_b200.parallel import PeerGroup

    rng = np.random.default_rng(5)
    p, d = _layer(egt, port, rng, "int4-2:4", 1024, 2048)
    (g,) = PeerGroup.local_ranks(1, d.rows)
    x = torch.from_numpy(rng.uniform(-1, 1, d.cols).astype(np.float32)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g.spmv(d, x, 0, d.rows)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.spmv(d, x, 0, d.rows)
    for _ in range(5):
        x.copy_(torch.from_numpy(rng.uniform(-1, 1, d.cols).astype(np.float32)))
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(g.y((d.rows,)), d.spmv(x))
    g.check()


def test_fused_allgather_missing_peer_times_out(egt, port, torch):
    """A rank whose peer never runs gives up after the bounded wait and
    reports it (no hang)."""
    from paper_2605_11582_b200.parallel import PeerGroup, RowShardPlan

    rng = np.random.default_rng(6)
    _, d = _layer(egt, port, rng, "int4-2:4", 256, 512)
    plan = RowShardPlan.make(d.rows, 2)
    g0, _g1 = PeerGroup.local_ranks(2, d.rows)
    x = torch.from_numpy(rng.uniform(-1, 1, d.cols).astype(np.float32)).cuda()
    g0.spmv(d.slice_rows(*plan.bounds[0]), x, 0, d.rows)
    with pytest.raises(egt.EgtError, match="timed out"):
        g0.check()


def test_fused_allgather_errors(egt, port, torch):
    from paper_2605_11582_b200.parallel import PeerGroup

    rng = np.random.default_rng(8)
    _, d = _layer(egt, port, rng, "int4-2:4", 256, 512)
    (g,) = PeerGroup.local_ranks(1, d.rows)
    x = torch.zeros(d.cols, device="cuda")
    with pytest.raises(egt.InvalidArgument, match="stride"):
        g.spmv(d, x, 16, d.rows)
    with pytest.raises(egt.InvalidArgument, match="input length differs from columns"):
        g.spmv(d, torch.zeros((2, d.cols - 4), device="cuda"), 0, d.rows)


@pytest.mark.parametrize("shape", [(8192, 28672), (5120, 13824)])
def test_fused_allgather_baseline_shapes(egt, port, torch, shape):
    """BASELINE config[4] shapes, 8 simulated ranks, against the oracle."""
    from paper_2605_11582_b200.parallel import PeerGroup, RowShardPlan

    rows, cols = shape
    rng = np.random.default_rng(rows + 1)
    p, d = _layer(egt, port, rng, "int4-2:4", rows, cols)
    plan = RowShardPlan.make(rows, 8)
    groups = PeerGroup.local_ranks(8, rows)
    xs = rng.uniform(-1, 1, cols).astype(np.float32)
    ys, want = _run_local(torch, d, groups, plan, torch.from_numpy(xs).cuda(), 1)
    assert all(torch.equal(y, want) for y in ys)
    ok, err = close(ys[3].cpu().numpy(), port.spmv(p, xs))
    assert ok, err


def _ipc_worker(rank, world, port_no, q):
    import torch
    import torch.distributed as dist

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port_no)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2605_11582_b200 as egt
        from oracle.oracle import Oracle
        from paper_2605_11582_b200.parallel import FusedShardedSpmv

        port = Oracle("port")
        rng = np.random.default_rng(2024)  # same layer on every rank
        p, _, _ = make_int4(rng, 1040, 2048, 2, 128, port)
        d = egt.DeviceMatrix.from_packed(to_product(p))
        sh = FusedShardedSpmv(d)
        ok = True
        for _ in range(3):
            x = torch.from_numpy(rng.uniform(-1, 1, d.cols).astype(np.float32)).cuda()
            dist.barrier()
            y = sh(x).clone()
            torch.cuda.synchronize()
            dist.barrier()  # every rank's slice landed before anyone rewrites
            ok &= bool(torch.equal(y, d.spmv(x)))
        sh.peers.check()
        q.put((rank, ok, ""))
    except Exception as e:  # reported to the parent
        q.put((rank, False, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_fused_allgather_two_processes_ipc(egt, torch):
    """Two ranks in two processes on one GPU: buffers exchanged as CUDA IPC
    handles over gloo, each kernel stores into the other's buffer."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    from tests.test_parallel_gloo import _free_port

    port_no = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def test_fused_allgather_empty_shards(egt, port, torch):
    """More ranks than row tiles: empty shards still signal, so every rank's
    wait completes and the gathered y is whole."""
    from paper_2605_11582_b200.parallel import PeerGroup, RowShardPlan

    rng = np.random.default_rng(9)
    p, d = _layer(egt, port, rng, "int4-2:4", 32, 256)
    plan = RowShardPlan.make(d.rows, 4)
    assert any(r1 == r0 for r0, r1 in plan.bounds)
    groups = PeerGroup.local_ranks(4, d.rows)
    xs = rng.uniform(-1, 1, d.cols).astype(np.float32)
    ys, want = _run_local(torch, d, groups, plan, torch.from_numpy(xs).cuda(), 1)
    assert all(torch.equal(y, want) for y in ys)
    for g in groups:
        g.check()
