"""bench.py's configs[3] row-shard leg alone (per-rank GEMV us at P = 1/2/4/8)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2402_10517_b200 import plan  # noqa: E402

print(json.dumps(bench.shard70b_detail(torch, plan)))
