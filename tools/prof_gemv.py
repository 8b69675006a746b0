"""Profiling driver: a few GEMVs at given shape / bit-widths (used under ncu)."""
import argparse
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_10517_b200 import AnyPrecisionLayer, engine, plan

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=4096)
ap.add_argument("--cols", type=int, default=4096)
ap.add_argument("--bits", type=str, default="3,4,8")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
codes = torch.randint(0, 256, (a.rows, a.cols), dtype=torch.uint8, device="cuda", generator=g)
tables = {k: torch.sort(torch.randn(a.rows, 1 << k, device="cuda", generator=g), 1).values.half()
          for k in range(3, 9)}
layer = AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(a.rows, a.cols))
prep = engine.prepare(layer)
for k in [int(b) for b in a.bits.split(",")]:
    p = plan.GemvPlan([prep], k, m=a.m, grouped=False)
    p.x[0].normal_()
    for _ in range(a.reps):
        p.run()
torch.cuda.synchronize()
print("done")
