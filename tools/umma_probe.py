"""Per-call time of the many-token products at the 7B verify shapes (M = 80
and 272): the tcgen05 kernel (default) or, with EGT_NO_UMMA=1, the legacy
mma.sp kernel.  Prints one JSON line per (shape, M)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_11582_b200 as egt  # noqa: E402

rng = np.random.default_rng(0)
out = []
for rows, cols in [(4096, 4096), (11008, 4096), (4096, 11008), (32000, 4096)]:
    w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
    pats = np.array([[1, 1, 0, 0], [1, 0, 1, 0], [0, 1, 0, 1], [0, 0, 1, 1]], bool)
    keep = pats[rng.integers(0, 4, (rows, cols // 4))].reshape(rows, cols)
    mask = np.packbits(keep.reshape(-1), bitorder="little")
    p = egt.pack(mask, egt.quantize_matrix(w, 128, mask), 2)
    copies = max(2, min(8, (256 << 20) // (rows * cols // 2)))
    mats = [egt.DeviceMatrix.from_packed(p) for _ in range(copies)]
    for M in [int(v) for v in os.environ.get("UMMA_PROBE_M", "80,272").split(",")]:
        x = torch.from_numpy(rng.uniform(-1, 1, (M, cols)).astype(np.float32)).cuda()
        ys = [torch.empty((M, rows), device="cuda") for _ in mats]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for d, y in zip(mats, ys):  # plans and workspaces before the capture
                d.spmv_into(x, y, st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for d, y in zip(mats, ys):
                d.spmv_into(x, y, st)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        reps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        e1.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (reps * len(mats))
        flops = 2.0 * rows * cols / 2 * M
        r = {"shape": f"{rows}x{cols}", "M": M, "us": round(us, 2), "useful_TFLOPS": round(flops / us / 1e6, 1),
             "kernel": "legacy mma.sp" if os.environ.get("EGT_NO_UMMA") else "tcgen05"}
        print(json.dumps(r), flush=True)
