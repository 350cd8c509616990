import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from tests.layers import close, make_f16, make_int4, to_product
from oracle.oracle import Oracle
import paper_2605_11582_b200 as egt
from paper_2605_11582_b200.program import Op, Program
port = Oracle("port")
rng = np.random.default_rng(5)
layers = [make_int4(rng, 4096, 4096, 2, 128, port)[0],
          make_int4(rng, 1040, 2048, 1, 64, port)[0],
          make_int4(rng, 512, 13824, 2, 32, port)[0],
          make_f16(rng, 784, 1536, 2, port)[0],
          make_f16(rng, 96, 4096, 1, port)[0],
          make_int4(rng, 11008, 4096, 2, 128, port)[0]]
sel = [int(v) for v in os.environ.get("SEL", "0,1,2,3,4,5").split(",")]
layers = [layers[i] for i in sel]
ds = [egt.DeviceMatrix.from_packed(to_product(p)) for p in layers]
xs = [rng.uniform(-1, 1, p.cols).astype(np.float32) for p in layers]
ys = [torch.full((p.rows,), float("nan"), device="cuda") for p in layers]
prog = Program([Op(d, torch.from_numpy(x).cuda(), y) for d, x, y in zip(ds, xs, ys)])
prog.run(); torch.cuda.synchronize()
print(os.environ.get("TAG", ""), sel, prog.info["stages"], [round(close(y.cpu().numpy(), port.spmv(p, x))[1], 6) for p, x, y in zip(layers, xs, ys)])
