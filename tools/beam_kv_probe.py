"""One KV-cached constrained beam decode on a small 7B-width stack (4
layers) for an ncu launch list: where a KV step's time goes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.model import DeviceModel, Trie  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kv = (sys.argv[2] if len(sys.argv) > 2 else "kv") == "kv"
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
token, parent, payload, frontier = [1], [0], [-1], [0]
for _ in range(4):
    nxt = []
    for nd in frontier:
        for dg in range(8):
            token.append(4 + dg)
            parent.append(nd)
            payload.append(-1)
            nxt.append(len(token) - 1)
    frontier = nxt
for i, nd in enumerate(frontier):
    payload[nd] = i
trie = Trie(np.array(token, np.uint32), np.array(parent, np.uint32), np.array(payload, np.int64))
prompt = rng.integers(0, cfg["vocab_size"], 16).astype(np.int32)
for _ in range(2):
    model.decode(trie, prompt, beam_size=4, mode="autoregressive", kv_cache=kv)
torch.cuda.synchronize()
t0 = time.perf_counter()
out, st = model.decode(trie, prompt, beam_size=4, mode="autoregressive", kv_cache=kv)
torch.cuda.synchronize()
print(f"L={L} kv={kv}: {1e3 * (time.perf_counter() - t0):.2f} ms, {st}", flush=True)
