"""One decode step on the 7B-shaped int4-2:4 stack after warm-up (for an ncu
launch list of the step's kernels): EGT_BENCH_NO_VERIFY style setup."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.model import Decoder, DeviceModel  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
rng = np.random.default_rng(7)
cfg = dict(bench.DECODE_CFG, n_layers=L)
host = bench.decode_host_layers(rng, ["int4-2:4"])
layers = [egt.DeviceMatrix.from_packed(host[("int4-2:4", r, c)]) for _ in range(L) for r, c in bench.LAYER_SHAPES]
hw = rng.uniform(-0.01, 0.01, (cfg["vocab_size"], 4096)).astype(np.float32)
keep = np.zeros((cfg["vocab_size"], 1024, 4), bool)
keep[:, :, :2] = True
mask = np.packbits(keep.reshape(-1), bitorder="little")
head = egt.DeviceMatrix.from_packed(egt.pack(mask, egt.quantize_matrix(hw, 128, mask), 2))
model = DeviceModel(cfg, rng.uniform(-0.01, 0.01, (cfg["vocab_size"], 4096)).astype(np.float32), layers, head)
dec = Decoder(model, 128)
dec.start(list(range(16)))
dec.step(20)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
dec.step(1)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
