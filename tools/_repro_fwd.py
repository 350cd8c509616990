import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
import paper_2605_11582_b200 as egt
from paper_2605_11582_b200.model import DeviceModel
rng = np.random.default_rng(3)
kind = sys.argv[1] if len(sys.argv) > 1 else "int4-2:4"
cfg = dict(vocab_size=1000, d_model=4096, n_layers=1, n_heads=32, d_ff=11008, max_positions=4096)
host = bench.decode_host_layers(rng, [kind])
layers = []
for rows, cols in bench.LAYER_SHAPES:
    a = host[(kind, rows, cols)]
    layers.append(egt.DeviceMatrix.dense_i4(a) if kind == "int4-dense" else egt.DeviceMatrix.from_packed(a))
hw = rng.uniform(-0.01, 0.01, (1000, 4096)).astype(np.float32)
hkeep = np.zeros((1000, 1024, 4), bool); hkeep[:, :, :2] = True
hmask = np.packbits(hkeep.reshape(-1), bitorder="little")
head = egt.DeviceMatrix.from_packed(egt.pack(hmask, egt.quantize_matrix(hw, 128, hmask), 2))
model = DeviceModel(cfg, rng.uniform(-0.01, 0.01, (1000, 4096)).astype(np.float32), layers, head)
for M in [int(v) for v in sys.argv[2].split(",")]:
    vis = np.tril(np.ones((M, M), bool))
    out = model.forward(np.arange(M, dtype=np.int32) % 1000, np.arange(M, dtype=np.int32), vis)
    torch.cuda.synchronize()
    print(kind, M, "ok", float(out.abs().max()), flush=True)
