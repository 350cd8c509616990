"""One SparseGemv shape under a forced plan, launched a few times (for ncu)."""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_11582_b200 as egt  # noqa: E402
from bench import host_layer  # noqa: E402
from paper_2605_11582_b200 import native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="4096x4096")
ap.add_argument("--plan", default="")  # RB,S,nw
ap.add_argument("--launches", type=int, default=4)
ap.add_argument("--indep", action="store_true")
a = ap.parse_args()
rows, cols = map(int, a.shape.split("x"))
rng = np.random.default_rng(3)
p = host_layer(rng, rows, cols)
layers = [egt.DeviceMatrix.from_packed(p) for _ in range(4)]
x = torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda()
y = torch.empty(rows, device="cuda")
if a.plan:
    rb, s, nw = map(int, a.plan.split(","))
    native.lib().egt_tune_force_plan(rb, s, nw, 0, 0)
for i in range(a.launches):
    layers[i % 4].spmv_into(x, y, independent=a.indep)
torch.cuda.synchronize()
print("ok", float(y.norm()))
