import sys, os
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2605_11582_b200 as egt
from paper_2605_11582_b200.native import lib
import ctypes as C
import bench
rng = np.random.default_rng(0)
for shape in [(4096, 4096), (11008, 4096), (4096, 11008)]:
    p = bench.host_layer(rng, *shape)
    d = egt.DeviceMatrix.from_packed(p)
    for M in (1, 2, 4, 8):
        x = torch.from_numpy(rng.uniform(-1, 1, (M, shape[1])).astype(np.float32)).cuda()
        y = torch.empty((M, shape[0]), device="cuda")
        for _ in range(3): d.spmv_into(x if M > 1 else x[0], y if M > 1 else y[0])
        torch.cuda.synchronize()
        info = d.plan_info(M) if hasattr(d, "plan_info") else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): d.spmv_into(x if M > 1 else x[0], y if M > 1 else y[0])
        e1.record(); e1.synchronize()
        print(shape, M, round(e0.elapsed_time(e1) * 1e3 / 50, 2), "us", info)
