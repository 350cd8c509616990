"""bench.measure_decode's verify-pass numbers (forward_tree over 64 / 256-node
trees after a 16-token prefix, 7B stack) for quick A/B runs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402

r = bench.measure_decode(torch, egt, sys.argv[1] if len(sys.argv) > 1 else "int4-2:4")
print(json.dumps({"tokens_per_s": r["tokens_per_s"], **{k: v["ms_per_pass"] for k, v in r["verify_pass"].items()}}))
