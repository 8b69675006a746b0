"""Per-rank step time of bench.py's layer set at world size W (rank 0's row
shard, plain GEMV launches, no gather) on one GPU: what strong scaling leaves
per rank.  Usage: python tools/shard_step.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_10517_b200 import plan  # noqa: E402

torch.cuda.set_device(0)
out = {}
for w in (1, 2, 4, 8):
    copies = [bench.make_layer_set(torch, 1234 + c, 0, w) for c in range(bench.N_COPIES)]
    plans = bench.decode_plans(plan, copies, pdl=True)

    def step():
        for _, _, p in plans:
            p.run()

    _, ms = bench.time_graph(torch, step, 50)
    out[w] = {"ms_per_step": round(ms, 4), "speedup_vs_1": None, "launches": len(plans)}
    del copies, plans
    torch.cuda.empty_cache()
for w in out:
    out[w]["speedup_vs_1"] = round(out[1]["ms_per_step"] / out[w]["ms_per_step"], 2)
print(json.dumps(out))
