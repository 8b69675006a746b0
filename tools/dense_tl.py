"""Per-CTA phase timeline of one fused dense launch (APBD_TL build of the library:
tools/kbench/variants.sh dtl -DAPBD_TL; run with APB_LIB_PATH pointing at it)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as ora  # noqa: E402
from paper_2402_10517_b200 import AnyPrecisionLayer, engine  # noqa: E402
from paper_2402_10517_b200._lib import load  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
rows, cols = 11008, 4096
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), rows, cols, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols)))
x = torch.randn(m, cols, device="cuda")
cfg = engine.GemvConfig(bit_width=4)
for _ in range(3):
    engine.gemm(prep, x, cfg)
torch.cuda.synchronize()
lib = load()
n = 8192 * 10
buf = (ctypes.c_ulonglong * n)()
assert lib.apbd_read_timeline(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 10).astype(np.float64)
ncta = int((a[:, 0] > 0).sum())
a = a[:ncta]
t0 = a[:, 0].min()
us = lambda v: (v - t0) / 1e3  # noqa: E731
start, alloc, first_mma, last_mma, epi, end, table = (us(a[:, i]) for i in (0, 1, 2, 3, 4, 5, 6))
wa, wx, sm = a[:, 7], a[:, 8], a[:, 9].astype(int)
print(f"M={m}: {ncta} CTAs, launch span {end.max():.1f} us")
def st(name, v):
    print(f"  {name:34s} mean {v.mean():7.2f}  p50 {np.median(v):7.2f}  p90 {np.percentile(v, 90):7.2f}  max {v.max():7.2f} us")
st("CTA duration", end - start)
st("start -> TMEM alloc done", alloc - start)
st("alloc -> table built (decoders)", table - alloc)
st("start -> first MMA issued", first_mma - start)
st("first -> last MMA issued", last_mma - first_mma)
st("last MMA issued -> accumulator ready", epi - last_mma)
st("epilogue (TMEM -> y) + teardown", end - epi)
print(f"  issuer waits: a_full {wa.mean() / 1965:.2f} us, x_full {wx.mean() / 1965:.2f} us per CTA (cycles / 1.965 GHz)")
# per SM: CTAs back to back?
gaps = []
for s in np.unique(sm):
    idx = np.where(sm == s)[0]
    o = idx[np.argsort(start[idx])]
    for i in range(1, len(o)):
        gaps.append(start[o[i]] - end[o[i - 1]])
gaps = np.array(gaps)
st("gap: CTA end -> next CTA start (same SM)", gaps)
print(f"  CTAs per SM: {np.bincount(sm).max()} max, {ncta / len(np.unique(sm)):.2f} mean")
