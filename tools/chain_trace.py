"""Timeline of a dependent chain of SparseGemv launches (EGT_TILED_TRACE):
per launch, relative to the previous launch's last CTA exit, when CTA 0
started, passed the PDL wait, finished staging x and computing, and when the
last CTA exited.  python tools/chain_trace.py [shape] [n] [indep]"""
import ctypes as C
import os
import sys

os.environ["EGT_TILED_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.native import lib  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "4096x4096"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12  # (U(-1,1) weights overflow f32 after ~25 launches)
rows, cols = map(int, shape.split("x"))
rng = np.random.default_rng(1)
# U(-1, 1) weights: activations grow along the chain (model-scale weights
# shrink them below 2^-9 after a few launches and measure the x-range restage)
p = bench.host_layer(rng, rows, cols)
ds = [egt.DeviceMatrix.from_packed(p) for _ in range(n)]
assert rows == cols, "chain needs square layers"
bufs = [torch.from_numpy(rng.uniform(-1, 1, cols).astype(np.float32)).cuda() for _ in range(2)]
s = torch.cuda.Stream()


indep = len(sys.argv) > 3 and sys.argv[3] == "indep"
for arg in sys.argv[3:]:
    if arg.startswith("plan="):  # RB,S,nw[,NST,CH]
        f = [int(v) for v in arg[5:].split(",")] + [0, 0]
        lib().egt_tune_force_plan(f[0], f[1], f[2], f[3], f[4])
ys = [torch.empty(rows, device="cuda") for _ in range(n)]


def chain():
    for i, d in enumerate(ds):
        if indep:  # every product reads the same x: EGT_SPMV_INDEPENDENT launches
            d.spmv_into(bufs[0], ys[i], s, independent=True)
        else:
            d.spmv_into(bufs[i % 2], bufs[(i + 1) % 2], s)


with torch.cuda.stream(s):
    chain()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        chain()
    for _ in range(3):
        g.replay()
    s.synchronize()
    buf = (C.c_ulonglong * (8 * 4096))()
    lib().egt_tune_read_trace(buf, 8 * 4096, 1)  # reset
    g.replay()
    s.synchronize()
lib().egt_tune_read_trace(buf, 8 * 4096, 0)
t = np.frombuffer(buf, np.uint64).reshape(4096, 8).astype(np.int64)
# the graph's launches used slots n .. 2n-1 (the eager chain used 0 .. n-1)
sl = t[n:2 * n]
first = (~sl[:, 5].astype(np.uint64)).astype(np.int64)
base = first.min()
print(f"{shape} x{n} dependent chain, ns relative to the first CTA start of launch 0")
print(" i  first_start  cta0_start  waited  staged  computed  last_exit | exit->next_wait")
for i in range(n):
    r = sl[i] - base
    nxt = (sl[i + 1, 1] - sl[i, 4]) if i + 1 < n else 0
    print(f"{i:2d} {first[i]-base:10d} {r[0]:10d} {r[1]:8d} {r[2]:8d} {r[3]:8d} {r[4]:9d} | {nxt:6d}")
per = (sl[n - 1, 4] - sl[0, 4]) / (n - 1)
if sl[:, 6].any():
    print(f"first touch of x: {np.median(sl[:, 6] - sl[:, 1]):.0f} ns, then staging {np.median(sl[:, 2] - sl[:, 6]):.0f} ns")
print(f"per launch (exit to exit): {per:.0f} ns; stage {np.median(sl[:, 2]-sl[:, 1]):.0f} ns, compute {np.median(sl[:, 3]-sl[:, 2]):.0f} ns, "
      f"epilogue->last exit {np.median(sl[:, 4]-sl[:, 3]):.0f} ns, exit->next wait {np.median(sl[1:, 1]-sl[:-1, 4]):.0f} ns")
