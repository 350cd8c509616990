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
    sh, n = spec.split(":")
    rows, cols = (int(v) for v in sh.split("x"))
    n = int(n)
    rng = np.random.default_rng(1)
    p = bench.host_layer(rng, rows, cols)
    ds = [egt.DeviceMatrix.from_packed(p) for _ in range(n)]
    x = torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda()
    ys = [torch.empty(rows, device="cuda") for _ in range(n)]
    prog = Program([Op(d, x, y) for d, y in zip(ds, ys)])
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    N = 4096
    buf = (C.c_longlong * (4 * N))()
    check(lib().egt_program_debug_trace(prog._h, buf, 4 * N))
    t = np.frombuffer(buf, dtype=np.int64).reshape(4, N)
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
    print("first 40 chunks: issue, ready, done")
    for i in range(min(40, nc)):
        print(i, iss[i], rdy[i], done[i])


if __name__ == "__main__":
    main()
