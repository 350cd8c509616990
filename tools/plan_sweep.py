"""Measure the tiled SpGEMV launch plans (RB row tiles/CTA, S K-splits, nw
consumer warps) for the sweep shapes on the GPU and print µs/call per plan.
Rotates over enough distinct weight copies to exceed L2; CUDA-graph replay
with PDL, like bench.py.  Usage: python tools/plan_sweep.py [--shapes ...]"""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_11582_b200 as egt  # noqa: E402
from bench import host_layer, shape_bytes  # noqa: E402
from paper_2605_11582_b200 import native  # noqa: E402


def time_plan(layers, x, ys, stream, reps=20, indep=False):
    for d, y in zip(layers, ys):  # warm-up (plans + workspace)
        d.spmv_into(x, y, stream, independent=indep)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for d, y in zip(layers, ys):
                d.spmv_into(x, y, stream, independent=indep)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):  # replay() runs on the current stream
        for _ in range(3):
            g.replay()
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    e1.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (reps * len(layers))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,11008x4096,4096x11008")
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--indep", action="store_true", help="EGT_SPMV_INDEPENDENT launches")
    ap.add_argument("--quick", action="store_true", help="dependent sweep over S in {1, 2} only")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "plan_sweep.json"))
    args = ap.parse_args()
    rng = np.random.default_rng(7)
    stream = torch.cuda.Stream()
    L = native.lib()
    results = {}
    for spec in args.shapes.split(","):
        rows, cols = map(int, spec.split("x"))
        p = host_layer(rng, rows, cols) if args.n == 2 else None
        copies = max(8, math.ceil(300e6 / shape_bytes(p)))
        layers = [egt.DeviceMatrix.from_packed(p, stream) for _ in range(copies)]
        x = torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda()
        ys = [torch.empty(rows, device="cuda") for _ in range(copies)]
        RT, KQ = (rows + 15) // 16, (cols + 127) // 128
        res = []
        L.egt_tune_force_plan(0, 0, 0, 0, 0)
        t = time_plan(layers, x, ys, stream, indep=args.indep)
        res.append({"plan": "auto", "us": t, "GBps": shape_bytes(p) / t / 1e3})
        for S in ((1, 2, 3, 4) if args.indep else ((1, 2) if args.quick else (1, 2, 3, 4, 6, 8))):
            if S > KQ:
                continue
            for ctas in ((48, 96, 148, 256) if args.indep else (74, 128, 148, 296)):
                RB = max(1, math.ceil(RT * S / ctas))
                for nw, ch in (((4, 0), (6, 0), (8, 0), (8, 16), (12, 0), (12, 24), (16, 0)) if args.indep else ((4, 0), (8, 0), (12, 0), (12, 24))):
                    L.egt_tune_force_plan(RB, S, nw, 0, ch)
                    try:
                        t = time_plan(layers, x, ys, stream, indep=args.indep)
                    except Exception as e:  # noqa: BLE001
                        res.append({"plan": [RB, S, nw, ch], "error": str(e)})
                        continue
                    res.append({"plan": [RB, S, nw, ch], "grid": math.ceil(RT / RB) * S, "us": round(t, 3),
                                "GBps": round(shape_bytes(p) / t / 1e3, 1)})
        L.egt_tune_force_plan(0, 0, 0, 0, 0)
        res.sort(key=lambda r: r.get("us", 1e9))
        results[spec] = res
        print(spec, json.dumps(res[:8]), flush=True)
        del layers
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
