"""Per-call host path: 3 stream operations (H2D, launch, D2H) + sync, vs the
same three captured once as a CUDA graph (replay + sync).  4096x4096 k=3 and
11008x4096 k=8, pinned fp16 x."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2402_10517_b200 import engine, AnyPrecisionLayer, _device as dev
from oracle import oracle as ora

for rows, cols, k in ((4096, 4096, 3), (11008, 4096, 8)):
    codes, tables = ora.random_layer_arrays(np.random.default_rng(0), rows, cols, 3, 8)
    prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols)))
    cfg = engine.GemvConfig(bit_width=k, activations_fp16=True)
    x = torch.randn(cols, dtype=torch.float16).pin_memory()
    for _ in range(50):
        y = engine.gemv(prep, x, cfg)
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        y = engine.gemv(prep, x, cfg)
    a = (time.perf_counter() - t0) / n * 1e6
    plan = prep._call_plan(k, 1, 0)
    lib = plan._lib
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            st = dev.stream_ptr()
            lib.apb_memcpy_async(plan.x_ptr, plan.x_pin_ptr, plan.x_bytes, 0, st)
            plan.launch(plan.x_ptr, plan.y_ptr, st)
            lib.apb_memcpy_async(plan.y_pin_ptr, plan.y_ptr, plan.y_bytes, 1, st)
    torch.cuda.synchronize()
    xn = x.numpy()
    for _ in range(50):
        plan.x_np[0, :cols] = xn
        g.replay()
        torch.cuda.current_stream().synchronize()
    t0 = time.perf_counter()
    cur = torch.cuda.current_stream()
    for _ in range(n):
        plan.x_np[0, :cols] = xn
        g.replay()
        lib.apb_stream_sync(dev.stream_ptr())
        out = plan.y_np.copy()
    b = (time.perf_counter() - t0) / n * 1e6
    ok = np.array_equal(out[0], y.numpy() if hasattr(y, "numpy") else np.asarray(y))
    print(f"{rows}x{cols} k={k}: stream ops {a:.1f} us/call, graph {b:.1f} us/call, same={ok}")
