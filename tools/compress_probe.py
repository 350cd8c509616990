"""GPU compression timing (egt_gpu_*): importance -> prune_nm -> quantize +
pack of the 7B layer shapes, device time per layer vs the host encoder."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_11582_b200 as egt  # noqa: E402


def dev_ms(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n


out = {}
for rows, cols in [(4096, 4096), (11008, 4096), (4096, 11008)]:
    rng = np.random.default_rng(rows + cols)
    w = torch.from_numpy(rng.uniform(-1, 1, (rows, cols)).astype(np.float32)).cuda()
    xn = torch.rand(cols, device="cuda") + 0.5
    ga = torch.rand((rows, cols), device="cuda")
    r = {}
    r["importance_ms"] = dev_ms(lambda: egt.gpu_importance(w, xn, ga))
    s = egt.gpu_importance(w, xn, ga)
    r["prune_ms"] = dev_ms(lambda: egt.gpu_prune_nm(s, 2))
    m = egt.gpu_prune_nm(s, 2)
    r["quantize_pack_ms"] = dev_ms(lambda: egt.gpu_quantize_pack(w, m, 2, 128, want_matrix=False))
    r["quantize_pack_upload_ms"] = dev_ms(lambda: egt.gpu_quantize_pack(w, m, 2, 128, want_raw=False), n=3)
    wh, mh = w.cpu().numpy(), m.cpu().numpy()
    t0 = time.perf_counter()
    q = egt.quantize_matrix(wh, 128, mh)
    egt.pack(mh, q, 2)
    r["host_encoder_ms"] = (time.perf_counter() - t0) * 1e3
    out[f"{rows}x{cols}"] = {k: round(v, 3) for k, v in r.items()}
print(json.dumps(out))
