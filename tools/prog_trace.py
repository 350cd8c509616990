"""CTA-0 timeline of the program kernel (EGT_PROGRAM_TRACE): per ring chunk the
producer issue clock, the consumer data-ready and done clocks and the
epilogue segment clock.  Prints gaps statistics in SM cycles.

    EGT_PROGRAM_TRACE=1 python tools/prog_trace.py [shape:n]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["EGT_PROGRAM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.native import check, lib  # noqa: E402
from paper_2605_11582_b200.program import Op, Program  # noqa: E402


def main():
    spec = sys.argv[1] if len(sys.argv) > 1 else "11008x4096:24"
    rng = np.random.default_rng(1)
    if spec.startswith("chain"):  # decode-like dependent chain over L layers
        from paper_2605_11582_b200.program import RMSNORM, SILU
        L = int(spec.split(":")[1]) if ":" in spec else 4
        host = {s: bench.host_layer(rng, *s) for s in sorted(set(bench.LAYER_SHAPES))}
        layers = [egt.DeviceMatrix.from_packed(host[s]) for _ in range(L) for s in bench.LAYER_SHAPES]
        h = torch.from_numpy(rng.uniform(-1, 1, 4096).astype(np.float32)).cuda()
        q, k, v = (torch.empty(4096, device="cuda") for _ in range(3))
        f = torch.empty(11008, device="cuda")
        ops = []
        for i in range(L):
            wq, wk, wv, wo, w1, w2 = layers[6 * i: 6 * i + 6]
            j = len(ops)
            ops += [Op(wq, h, q, input=RMSNORM, wait=j - 1), Op(wk, h, k, input=RMSNORM, wait=j - 1),
                    Op(wv, h, v, input=RMSNORM, wait=j - 1), Op(wo, v, h, residual=h, wait=j + 2),
                    Op(w1, h, f, input=RMSNORM, wait=j + 3), Op(w2, f, h, residual=h, input=SILU, wait=j + 4)]
        prog = Program(ops)
    else:
        sh, n = spec.split(":")
        rows, cols = (int(v) for v in sh.split("x"))
        n = int(n)
        p = bench.host_layer(rng, rows, cols)
        ds = [egt.DeviceMatrix.from_packed(p) for _ in range(n)]
        x = torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda()
        ys = [torch.empty(rows, device="cuda") for _ in range(n)]
        prog = Program([Op(d, x, y) for d, y in zip(ds, ys)])
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    N = 4096
    buf = (C.c_longlong * (8 * N))()
    check(lib().egt_program_debug_trace(prog._h, buf, 8 * N))
    t = np.frombuffer(buf, dtype=np.int64).reshape(8, N)
    nq = int((t[0] > 0).sum())
    nc = int((t[1] > 0).sum())
    t0 = t[0, 0]
    iss, rdy, done, epi = (t[i, :max(nq, nc)] - t0 for i in range(4))
    print(f"chunks: producer {nq}, consumer {nc}, epilogue {(t[3] > 0).sum()}; info {prog.info}")
    print(f"span (cycles): issue last {iss[nq-1]}, consumer done last {done[nc-1]}")
    lat = rdy[:nc] - iss[:nc]
    comp = done[:nc] - rdy[:nc]
    gap = rdy[1:nc] - done[:nc - 1]
    for name, v in (("issue->ready", lat), ("ready->done (compute)", comp), ("done->next ready", gap),
                    ("issue interval", np.diff(iss[:nq]))):
        print(f"{name:24s} median {np.median(v):8.0f}  p10 {np.percentile(v, 10):8.0f}  p90 {np.percentile(v, 90):8.0f}")
    nops = prog.info["n_ops"]
    print("per op: consumer start, wait passed, staged, epilogue done-arrive (cycles from first issue)")
    for j in range(min(nops, 40)):
        w = t[5, j] - t0 if t[5, j] else -1
        print(j, t[4, j] - t0, w, t[6, j] - t0 if t[6, j] else -1, t[7, j] - t0)
    print("first 60 chunks: issue, ready, done; epilogue")
    for i in range(min(60, nc)):
        print(i, iss[i], rdy[i], done[i], epi[i] if i < len(epi) else "")


if __name__ == "__main__":
    main()
