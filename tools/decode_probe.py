"""7B decode tokens/s probe (bench.measure_decode) for quick A/B runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "int4-2:4"
r = bench.measure_decode(torch, egt, plan)
r.pop("verify_pass", None)
print(json.dumps({k: r[k] for k in ("plan", "tokens_per_s", "ms_per_token", "weight_GBps")}))
