"""Error table of the x-range paths (diagnostic, profiles/xrange_r02.txt):
per format x M x input family the device product against the port's f32
spmv under the plain metric max |d|/(1+|want|) ("strict"), under the test's
cancellation-aware metric ("test"), and the reference's OWN f32 result
against float64 under the plain metric ("ref-vs-f64")."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.oracle import Oracle  # noqa: E402
from tests.test_gpu_xrange import FORMATS, KINDS, _abs_sum, _compare, _layer, _ref_noise, _xs  # noqa: E402

port = Oracle("port")
print("format M path | kind=strict/test/ref-vs-f64 ...")
for fmt in FORMATS:
    for M in (1, 3, 16, 40):
        rng = np.random.default_rng(FORMATS.index(fmt) * 100 + M)
        rows, cols = (256, 4096) if fmt.startswith("int4") else (128, 2048)
        d, ref, w = _layer(port, rng, fmt, rows, cols)
        row = []
        for kind in KINDS:
            xs = np.stack([_xs(rng, kind, cols) for _ in range(M)])
            y = d.spmv(torch.from_numpy(xs).cuda()).cpu().numpy().reshape(M, rows)
            scale = 1e6 if kind == "tiny" else (1e-30 if kind == "huge" else 1.0)
            try:
                e1 = max(_compare(y[m], ref(xs[m]), scale) for m in range(M))
                e2 = max(_compare(y[m], ref(xs[m]), scale, _abs_sum(w, xs[m])) for m in range(M))
                e3 = max(_ref_noise(w, xs[m], ref(xs[m])) for m in range(M)) if kind in ("big", "mixed") else 0.0
                row.append(f"{kind}={e1:.1e}/{e2:.1e}/{e3:.1e}")
            except AssertionError:
                row.append(f"{kind}=NONFINITE-POSITIONS-DIFFER")
        print(fmt, M, d.path, "|", " ".join(row), flush=True)
