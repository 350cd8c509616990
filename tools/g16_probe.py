import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2605_11582_b200 as egt
import bench
rng = np.random.default_rng(0)
p = bench.format_layer(rng, "int4-2:4-g16", 4096, 4096)
d = egt.DeviceMatrix.from_packed(p)
x = torch.from_numpy(rng.uniform(-1, 1, 4096).astype(np.float32)).cuda()
y = torch.empty(4096, device="cuda")
for _ in range(3):
    d.spmv_into(x, y)
torch.cuda.synchronize()
print(d.path, d.algorithmic_bytes)
