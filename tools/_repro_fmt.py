import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_2605_11582_b200 as egt
rng = np.random.default_rng(3)
for kind in ["int4-dense", "fp16-2:4", "int4-2:4"]:
    host = bench.decode_host_layers(rng, [kind])
    for (k, rows, cols), a in host.items():
        d = egt.DeviceMatrix.dense_i4(a) if k == "int4-dense" else egt.DeviceMatrix.from_packed(a)
        for M in (64, 80, 272):
            x = torch.from_numpy(rng.uniform(-1, 1, (M, cols)).astype(np.float32)).cuda()
            y = d.spmv(x); torch.cuda.synchronize()
            r = d.spmv(x[M - 1]); torch.cuda.synchronize()
            print(k, rows, cols, M, float(((y[M - 1] - r).abs() / (1 + r.abs())).max()), flush=True)
