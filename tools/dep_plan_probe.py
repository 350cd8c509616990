"""Dependent-launch us/call of one shape under forced tiled plans
(RB,S,nw,NST,CH; 'auto' = the planner): copies of the layer in a CUDA graph,
each call waiting for its predecessor, x static (no chaining)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.native import lib  # noqa: E402

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x4096").split("x"))
plans = sys.argv[2:] or ["auto"]
rng = np.random.default_rng(1)
p = bench.host_layer(rng, *shape)
copies = max(4, (512 << 20) // (shape[0] * shape[1] // 2))
mats = [egt.DeviceMatrix.from_packed(p) for _ in range(copies)]
x = torch.from_numpy(rng.uniform(-1, 1, shape[1]).astype(np.float32)).cuda()
ys = [torch.empty(shape[0], device="cuda") for _ in mats]
s = torch.cuda.Stream()
for pl in plans:
    if pl == "auto":
        lib().egt_tune_force_plan(0, 0, 0, 0, 0)
    else:
        f = [int(v) for v in pl.split(",")] + [0, 0]
        lib().egt_tune_force_plan(f[0], f[1], f[2], f[3], f[4])
    with torch.cuda.stream(s):
        for d, y in zip(mats, ys):
            d.spmv_into(x, y, s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for d, y in zip(mats, ys):
                d.spmv_into(x, y, s)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            g.replay()
        e1.record(s)
        e1.synchronize()
    print(f"{shape} plan {pl}: {1e3 * e0.elapsed_time(e1) / (10 * len(mats)):.3f} us/call", flush=True)
lib().egt_tune_force_plan(0, 0, 0, 0, 0)
