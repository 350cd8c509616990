"""Micro-experiments for the program kernel: single-op programs of each shape
and programs of n copies of one shape (independent ops)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.program import Op, Program  # noqa: E402
from tools.prog_probe import timeit  # noqa: E402


def main():
    rng = np.random.default_rng(1)
    stream = torch.cuda.Stream()
    out = {}
    shapes = [(4096, 4096), (11008, 4096), (4096, 11008)]
    ns = (1, 4, 24)
    reps = 30
    if len(sys.argv) > 1:  # e.g. 11008x4096:24 (profiling: one config, few launches)
        sh, n = sys.argv[1].split(":")
        shapes = [tuple(int(v) for v in sh.split("x"))]
        ns = (int(n),)
        reps = 1
    for shape in shapes:
        p = bench.host_layer(rng, *shape)
        b = bench.shape_bytes(p)
        copies = [egt.DeviceMatrix.from_packed(p, stream) for _ in range(24)]
        x = torch.from_numpy(rng.uniform(-1, 1, shape[1]).astype(np.float32)).cuda()
        for n in ns:
            ys = [torch.empty(shape[0], device="cuda") for _ in range(n)]
            prog = Program([Op(copies[i], x, ys[i]) for i in range(n)], stream)
            ms = timeit(lambda: prog.run(stream), reps, stream)
            out[f"{shape[0]}x{shape[1]} n={n}"] = {"us_per_op": round(1e3 * ms / n, 2),
                                                   "GBps": round(n * b / ms / 1e6, 1)}
        del copies
    print(json.dumps(out))


if __name__ == "__main__":
    main()
