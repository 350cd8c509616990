"""us/call of a row-shard product: independent, dependent, and with the fused
all-gather epilogue (world 1 / simulated ranks), same weights, CUDA graphs."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.parallel import PeerGroup  # noqa: E402


def timed(fn, n=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


out = {}
for rows, cols in [(5120, 13824), (8192, 28672), (4096, 4096)]:
    p = bench.host_layer(np.random.default_rng(rows), rows, cols)
    copies = max(2, -(-2 * 126 * 2**20 // bench.shape_bytes(p)))
    ds = [egt.DeviceMatrix.from_packed(p) for _ in range(copies)]
    x = torch.rand(cols, device="cuda")
    y = torch.empty(rows, device="cuda")
    (g,) = PeerGroup.local_ranks(1, rows)
    r = {}
    r["indep"] = timed(lambda s: [d.spmv_into(x, y, s, independent=True) for d in ds]) / copies
    r["dep"] = timed(lambda s: [d.spmv_into(x, y, s) for d in ds]) / copies
    r["fused_w1"] = timed(lambda s: [g.spmv(d, x, 0, rows, s) for d in ds]) / copies
    r["fused_w1_indep"] = timed(lambda s: [g.spmv(d, x, 0, rows, s, independent=True) for d in ds]) / copies
    out[f"{rows}x{cols}"] = {k: round(v, 3) for k, v in r.items()}
print(json.dumps(out))
