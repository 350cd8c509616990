import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_2605_11582_b200 as egt
rng = np.random.default_rng(3)
rows, cols = (int(v) for v in sys.argv[1].split("x"))
p = bench.host_layer(rng, rows, cols)
d = egt.DeviceMatrix.from_packed(p)
for M in [int(v) for v in sys.argv[2].split(",")]:
    x = torch.from_numpy(rng.uniform(-1, 1, (M, cols)).astype(np.float32)).cuda()
    y = d.spmv(x)
    torch.cuda.synchronize()
    ref = torch.stack([d.spmv(x[m]) for m in range(M)])
    print(rows, cols, M, "ok", float(((y - ref).abs() / (1 + ref.abs())).max()), flush=True)
