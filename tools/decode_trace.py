"""Per-product timeline of one KV-cached decode step (EGT_TILED_TRACE):
for each SparseGemv launch of the step graph, when it started, passed its PDL
wait, finished staging x and computing, and when its last CTA exited, grouped
by role in the layer.  python tools/decode_trace.py [layers]"""
import ctypes as C
import os
import sys

os.environ["EGT_TILED_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.model import Decoder, DeviceModel  # noqa: E402
from paper_2605_11582_b200.native import lib  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
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
n_per = 4 * L + 1  # fused QKV, O, ff1, ff2 per layer + head
buf = (C.c_ulonglong * (8 * 4096))()
lib().egt_tune_read_trace(buf, 8 * 4096, 1)  # reset before the decoder's warm-up + capture
dec = Decoder(model, 128)
dec.start(list(range(16)))
dec.step(30)
torch.cuda.synchronize()
lib().egt_tune_read_trace(buf, 8 * 4096, 1)
dec.step(1)
torch.cuda.synchronize()
lib().egt_tune_read_trace(buf, 8 * 4096, 0)
t = np.frombuffer(buf, np.uint64).reshape(4096, 8).astype(np.int64)
# launch_tiled slots: eager warm-up step = 0 .. n_per-1, captured graph = n_per .. 2 n_per - 1
sl = t[n_per:2 * n_per]
base = sl[:, 0].min()
roles = ["qkv", "o", "ff1", "ff2"]
stats = {r: [] for r in roles + ["head"]}
prev_exit = None
rows = []
for j in range(n_per):
    role = "head" if j == n_per - 1 else roles[j % 4]
    r = sl[j]
    gap = (r[1] - prev_exit) if prev_exit is not None else 0
    stats[role].append((r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], gap, r[4] - (prev_exit or r[0])))
    prev_exit = r[4]
span = sl[:, 4].max() - base
print(f"{L} layers: step span {span / 1e3:.1f} us (first product start -> last exit)")
print("role  start->wait  stage  compute  epi->exit  prev_exit->wait  prev_exit->exit (median ns)")
for role, v in stats.items():
    a = np.median(np.array(v), axis=0)
    print(f"{role:5s} {a[0]:10.0f} {a[1]:7.0f} {a[2]:8.0f} {a[3]:9.0f} {a[4]:14.0f} {a[5]:14.0f}")
