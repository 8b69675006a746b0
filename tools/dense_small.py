"""Small fused-dense call (debug / sanitizer)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer, engine
rows, cols, m, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), rows, cols, 2, 8)
layer = AnyPrecisionLayer(n_min=2, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols))
prep = engine.prepare(layer)
X = np.random.default_rng(1).standard_normal((m, cols)).astype(np.float32)
y = engine.gemm(prep, X, engine.GemvConfig(bit_width=k, dense_threshold=16))
W = engine.dequantize(layer, k).astype(np.float64)
print("rel_err", ora.rel_err(y, X.astype(np.float64) @ W.T))
