import sys, json, torch
sys.path.insert(0, ".")
import bench
from paper_2402_10517_b200 import engine
import numpy as np
from oracle import oracle as ora
from paper_2402_10517_b200 import AnyPrecisionLayer
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 11008, 4096, 3, 8)
layer = AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(11008, 4096))
prep = engine.prepare(layer)
print(json.dumps(bench.run_prefill(torch, [None]*4 + [prep])))
