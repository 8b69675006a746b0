import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine
rows, cols, m = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), rows, cols, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols)))
x = torch.randn(m, cols, device="cuda")
y = engine.gemm(prep, x, engine.GemvConfig(bit_width=4))
torch.cuda.synchronize()
W = torch.as_tensor(np.asarray(engine.dequantize(prep, 4).cpu() if hasattr(engine.dequantize(prep, 4), "cpu") else engine.dequantize(prep, 4)), dtype=torch.float64)
ref = (x.double().cpu() @ W.T)
err = ((y.double().cpu() - ref).norm() / ref.norm()).item()
print(rows, cols, m, "rel_err", err)
