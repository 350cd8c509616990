"""Timeline of one tcgen05 many-token product, CTA (0,0,0) (EGT_UMMA_TRACE=1):
producer x/raw issue, MMA issue, dequant done, epilogue round done (us from
the CTA start)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ.setdefault("EGT_UMMA_TRACE", "1")
sys.path.insert(0, ".")
import paper_2605_11582_b200 as egt  # noqa: E402
from paper_2605_11582_b200.native import lib  # noqa: E402

rows, cols, M = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 80))]
rng = np.random.default_rng(0)
w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
pats = np.array([[1, 1, 0, 0], [1, 0, 1, 0], [0, 1, 0, 1], [0, 0, 1, 1]], bool)
keep = pats[rng.integers(0, 4, (rows, cols // 4))].reshape(rows, cols)
mask = np.packbits(keep.reshape(-1), bitorder="little")
d = egt.DeviceMatrix.from_packed(egt.pack(mask, egt.quantize_matrix(w, 128, mask), 2))
x = torch.from_numpy(rng.uniform(-1, 1, (M, cols)).astype(np.float32)).cuda()
y = d.spmv(x)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 1024)()
lib().egt_tune_read_trace(buf, 1024, 1)
y = d.spmv(x)
torch.cuda.synchronize()
lib().egt_tune_read_trace(buf, 1024, 1)
t = np.array(buf[:], dtype=np.int64)
t0 = t[0]


def us(v):
    return "-" if v == 0 else f"{(v - t0) / 1e3:.2f}"


print(f"{rows}x{cols} M={M}: alloc done {us(t[1])}")
for st in range(0, 36):
    if t[8 + st] == 0 and t[80 + st] == 0:
        break
    print(f"stage {st:2d}: x {us(t[8 + st]):>6} | deq2 a_empty {us(t[640 + st]):>6} raw {us(t[720 + st]):>6} "
          f"done {us(t[160 + st]):>6} | deq9 done {us(t[480 + st]):>6} | mma tm_empty {us(t[560 + st]):>6} "
          f"a_full {us(t[400 + st]):>6} issued {us(t[80 + st]):>6}")
print(f"outputs done {us(t[2])}, teardown barrier {us(t[3])}, cluster barrier {us(t[4])}, loads {us(t[7])}, leader sum {us(t[5])}, "
      f"end {us(t[6])}")
print("epilogue warps: rounds done", [us(v) for v in t[800:808]], "\n  past bar", [us(v) for v in t[810:818]],
      "\n  partials", [us(v) for v in t[840:848]],
      "\n  outputs", [us(v) for v in t[820:828]])
print("reduce pass starts", us(t[900]), us(t[901]))
print("tail iterations:", [us(v) for v in t[860:880] if v])
print("MMA loop cycles per k-quad (waits, MMAs + round commits, slot commits, total):")
for i in range(8):
    print("  k-quad", 2 + i, [int(v) for v in t[900 + 8 * i:904 + 8 * i]])
print("raw issued:", [us(v) for v in t[320:340] if v])
print("epilogue rounds:", [us(v) for v in t[240:280] if v])
