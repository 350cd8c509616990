"""Constrained beam decode numbers for a decode plan (default the mixed one)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_11582_b200 as egt  # noqa: E402

os.environ.setdefault("EGT_BENCH_NO_VERIFY", "")
r = bench.measure_decode(torch, egt, sys.argv[1] if len(sys.argv) > 1 else "mixed-int4dense-fp16sp24")
print(json.dumps(r["constrained_beam_decode"]))
