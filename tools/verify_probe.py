"""One prefix-tree verification forward (M = prompt + tree nodes) over the
7B-shaped stack, for profiling (ncu launch list) and timing."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.model import DeviceModel  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    layers_n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    rng = np.random.default_rng(7)
    cfg = dict(bench.DECODE_CFG, n_layers=layers_n)
    host = bench.decode_host_layers(rng, ["int4-2:4"])
    layers = [egt.DeviceMatrix.from_packed(host[("int4-2:4", r, c)]) for _ in range(layers_n) for r, c in bench.LAYER_SHAPES]
    hw = rng.uniform(-0.01, 0.01, (cfg["vocab_size"], 4096)).astype(np.float32)
    keep = np.zeros((cfg["vocab_size"], 1024, 4), bool)
    keep[:, :, :2] = True
    mask = np.packbits(keep.reshape(-1), bitorder="little")
    head = egt.DeviceMatrix.from_packed(egt.pack(mask, egt.quantize_matrix(hw, 128, mask), 2))
    model = DeviceModel(cfg, rng.uniform(-0.01, 0.01, (cfg["vocab_size"], 4096)).astype(np.float32), layers, head)
    vis = np.tril(np.ones((M, M), bool))
    toks = rng.integers(0, cfg["vocab_size"], M).astype(np.int32)
    pos = np.arange(M, dtype=np.int32)
    model.forward(toks, pos, vis)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model.forward(toks, pos, vis)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"M={M} layers={layers_n}: median {ts[len(ts) // 2]:.2f} ms (min {ts[0]:.2f}, max {ts[-1]:.2f})", flush=True)


if __name__ == "__main__":
    main()
