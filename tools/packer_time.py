"""GPU packer leg of the bench (bench.packer_detail), standalone."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

print(json.dumps(bench.packer_detail(torch)))
