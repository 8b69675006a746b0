import cProfile, pstats, sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_10517_b200 import engine, AnyPrecisionLayer
from oracle import oracle as ora
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 4096, 4096, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(4096, 4096)))
cfg = engine.GemvConfig(bit_width=3, activations_fp16=True)
x = np.random.default_rng(1).standard_normal(4096).astype(np.float16)
for _ in range(50): engine.gemv(prep, x, cfg)
pr = cProfile.Profile(); pr.enable()
for _ in range(2000): engine.gemv(prep, x, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
