"""Host-side cost of one engine.gemv call (4096x4096, k=3)."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_10517_b200 import engine, AnyPrecisionLayer, _device as dev
from paper_2402_10517_b200._lib import load, APB_DTYPE_F32
from oracle import oracle as ora
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 4096, 4096, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(4096, 4096)))
cfg = engine.GemvConfig(bit_width=3, activations_fp16=True)
xh = torch.randn(4096, dtype=torch.float16).pin_memory()
xd = xh.cuda()
t = prep.tensor
y = torch.empty(1, 4096, device="cuda")
lib = load()
def bench(fn, n=300):
    for _ in range(20): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
raw = lambda: lib.apb_gemv(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, 3, dev.ptr(prep.tables16[3]),
                           dev.ptr(xd), 1, 4096, 0, dev.ptr(y), APB_DTYPE_F32, t.rows, 0, dev.stream_ptr())
print("raw C call, async (host us/call)", round(bench(raw), 1))
print("engine.gemv device x (us/call, async)", round(bench(lambda: engine.gemv(prep, xd, cfg)), 1))
print("engine.gemv pinned host x -> host y (us/call)", round(bench(lambda: engine.gemv(prep, xh, cfg)), 1))
print("engine.gemv numpy x -> numpy y (us/call)", round(bench(lambda: engine.gemv(prep, xh.numpy(), cfg)), 1))
def sync_raw():
    raw(); torch.cuda.synchronize()
print("raw C call + sync (us/call)", round(bench(sync_raw), 1))
