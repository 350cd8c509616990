"""bench.measure_decode's constrained beam decode numbers (KV-cached step vs
recompute) for quick runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402

r = bench.measure_decode(torch, egt, "int4-2:4")
print(json.dumps({"constrained_beam_decode": r["constrained_beam_decode"],
                  **{k: v["ms_per_pass"] for k, v in r["verify_pass"].items()}}))
