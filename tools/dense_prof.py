"""One fused dense launch (gate 11008x4096, k=4, fp32 x) for ncu."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 11008, 4096, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(11008, 4096)))
x = torch.randn(m, 4096, device="cuda")
for _ in range(3):
    engine.gemm(prep, x, engine.GemvConfig(bit_width=4))
torch.cuda.synchronize()
