"""One many-token product (spmm_wide.cu) for ncu: 4096x4096 INT4 2:4, M tokens."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 80
rows, cols = (int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "4096x4096").split("x"))
p = bench.host_layer(np.random.default_rng(1), rows, cols)
d = egt.DeviceMatrix.from_packed(p)
x = torch.rand((M, cols), device="cuda")
y = torch.empty((M, rows), device="cuda")
for _ in range(3):
    d.spmv_into(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    d.spmv_into(x, y)
e1.record()
e1.synchronize()
print(f"{rows}x{cols} M={M}: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us")
