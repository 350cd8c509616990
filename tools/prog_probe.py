"""Timing probe for the persistent program kernel: the 7B layer sweep as one
program of independent ops, and as a decode-like dependent chain.

    python tools/prog_probe.py [--layers 32] [--reps 50]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.program import RMSNORM, SILU, Op, Program  # noqa: E402


def timeit(fn, reps, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    rng = np.random.default_rng(2605)
    host = {s: bench.host_layer(rng, *s) for s in sorted(set(bench.LAYER_SHAPES))}
    stream = torch.cuda.Stream()
    layers = [egt.DeviceMatrix.from_packed(host[s], stream) for _ in range(args.layers) for s in bench.LAYER_SHAPES]
    torch.cuda.synchronize()
    step_bytes = sum(bench.shape_bytes(host[s]) for s in bench.LAYER_SHAPES) * args.layers
    out = {"layers": args.layers, "bytes_per_step": step_bytes}

    # independent sweep: every op reads the step input for its width
    xs = {c: torch.from_numpy(rng.uniform(-1, 1, c).astype(np.float32)).cuda() for c in (4096, 11008)}
    ys = [torch.empty(d.rows, device="cuda") for d in layers]
    prog = Program([Op(d, xs[d.cols], y) for d, y in zip(layers, ys)], stream)
    out["program_info"] = prog.info
    ms = timeit(lambda: prog.run(stream), args.reps, stream)
    out["indep_ms"] = ms
    out["indep_GBps"] = step_bytes / ms / 1e6
    # spot parity vs the per-launch kernel
    ref = [layers[i].spmv(xs[layers[i].cols]) for i in (0, 4, 5)]
    out["indep_vs_spmv_max_rel"] = max(float(((ys[i] - r).abs() / (1 + r.abs())).max())
                                       for i, r in zip((0, 4, 5), ref))

    # decode-like chain: q,k,v = W rmsnorm(h) (wait on previous layer);
    # h += Wo v (wait on v); f = Wff1 rmsnorm(h); h += Wff2 silu(f)
    h = torch.from_numpy(rng.uniform(-1, 1, 4096).astype(np.float32)).cuda()
    q = torch.empty(4096, device="cuda")
    k = torch.empty(4096, device="cuda")
    v = torch.empty(4096, device="cuda")
    f = torch.empty(11008, device="cuda")
    ops = []
    for L in range(args.layers):
        wq, wk, wv, wo, w1, w2 = layers[6 * L: 6 * L + 6]
        j = len(ops)
        ops += [Op(wq, h, q, input=RMSNORM, wait=j - 1), Op(wk, h, k, input=RMSNORM, wait=j - 1),
                Op(wv, h, v, input=RMSNORM, wait=j - 1), Op(wo, v, h, residual=h, wait=j + 2),
                Op(w1, h, f, input=RMSNORM, wait=j + 3), Op(w2, f, h, residual=h, input=SILU, wait=j + 4)]
    chain = Program(ops, stream)
    h0 = h.clone()

    def run_chain():
        chain.run(stream)

    ms = timeit(run_chain, args.reps, stream)
    out["chain_ms"] = ms
    out["chain_GBps"] = step_bytes / ms / 1e6
    out["chain_finite"] = bool(torch.isfinite(h).all())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
