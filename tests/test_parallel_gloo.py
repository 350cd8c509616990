"""Multi-process (world_size 2, gloo, CPU) coverage of the row-sharded path:
shard plans and the y-slice all-gather.  Each rank computes its rows of the
product with the oracle (the CUDA kernel is covered by the GPU tests) and the
gathered result must equal the single-process product bit for bit: shards do
not change any row's accumulation order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2605_11582_b200.parallel import RowShardPlan


def test_shard_plan_properties():
    for rows in (1, 15, 16, 100, 4096, 5120, 8192, 11008):
        for world in (1, 2, 3, 4, 8):
            p = RowShardPlan.make(rows, world)
            assert p.bounds[0][0] == 0 and p.bounds[-1][1] == rows
            for (a0, a1), (b0, b1) in zip(p.bounds, p.bounds[1:]):
                assert a1 == b0
            for r0, r1 in p.bounds:
                assert (r0 % 16 == 0 or r0 == rows) and (r1 % 16 == 0 or r1 == rows)
            sizes = [r1 - r0 for r0, r1 in p.bounds]
            assert max(sizes) - min(sizes) <= 32 or rows < 16 * world  # one tile + the ragged end
    # the BASELINE sharded shapes split evenly
    assert [b[1] - b[0] for b in RowShardPlan.make(8192, 8).bounds] == [1024] * 8
    assert [b[1] - b[0] for b in RowShardPlan.make(5120, 8).bounds] == [640] * 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from oracle.oracle import Oracle, Packed, mask_from_bool, random_nm_mask  # noqa: F401
    from paper_2605_11582_b200.parallel import RowShardPlan, gather_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_o = Oracle("port")
        rng = np.random.default_rng(77)  # same inputs on every rank
        rows, cols = 136, 256
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        mask = random_nm_mask(rng, rows, cols, 2)
        qm = port_o.quantize(w, np.full(rows, 128, np.uint32), mask)
        p = port_o.pack_int4(mask, rows, cols, qm, 2)
        X = rng.uniform(-1, 1, (3, cols)).astype(np.float32)
        full = np.stack([port_o.spmv(p, x) for x in X])
        plan = RowShardPlan.make(rows, world)
        r0, r1 = plan.local(rank)
        # this rank's rows: the oracle over the row sub-range of the stream
        row_nnz = cols // 2
        shard = Packed(2, 4, r1 - r0, cols, 1, p.index_words[r0 * row_nnz // 8: r1 * row_nnz // 8],
                       p.value_bytes[r0 * row_nnz // 2: r1 * row_nnz // 2], p.group_sizes[r0:r1],
                       p.group_offsets[r0: r1 + 1] - p.group_offsets[r0],
                       p.scales[p.group_offsets[r0]: p.group_offsets[r1]],
                       p.zero_points[p.group_offsets[r0]: p.group_offsets[r1]])
        y_local = torch.from_numpy(np.stack([port_o.spmv(shard, x) for x in X]))
        y = gather_rows(y_local, plan).numpy()
        y1 = gather_rows(y_local[0].clone(), plan).numpy()
        q.put((rank, bool(np.array_equal(y, full)), bool(np.array_equal(y1, full[0]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_allgather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok and ok1 for _, ok, ok1 in results), results


def _handle_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2605_11582_b200.parallel import exchange_handles

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank + 1] * 32 + list(range(32)))  # a 64-byte CUDA IPC handle stand-in
        got = exchange_handles(mine)
        q.put((rank, got == [bytes([r + 1] * 32 + list(range(32))) for r in range(world)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_peer_handle_exchange_gloo(world):
    """The fused all-gather's setup step: every rank's peer-buffer handle,
    in rank order, on every rank (parallel.exchange_handles)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handle_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert all(ok for _, ok in results), results
