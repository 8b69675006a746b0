"""Debug split-item launches on a tiny layer."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine, plan
rows, cols, k, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), rows, cols, 3, 8)
layer = AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols))
prep = engine.prepare(layer)
planes = prep.planes.cpu().numpy()
x = np.random.default_rng(1).standard_normal((m, cols)).astype(np.float16)
want = ora.gemm(planes, cols, k, tables[k], ora.prep_x(x.astype(np.float64), cols, True))
p = plan.GemvPlan([prep], k, m=m, grouped=True)
p.x[0][:, :cols].copy_(torch.from_numpy(x))
for it in range(3):
    p.run(); torch.cuda.synchronize()
    y = p.y[0].cpu().numpy()
    bad = np.where(~np.isclose(y, want, rtol=1e-3, atol=1e-3))
    print("run", it, "rel_err", ora.rel_err(y, want), "bad", list(zip(*bad))[:12], "nan", int(np.isnan(y).sum()))
