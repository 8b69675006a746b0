"""Time engine.gemm's dense path (fused tcgen05 vs the round-1 cuBLAS path) on
gate 11008x4096 (bench.run_prefill) and on a 4096x4096 layer at small M."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from oracle import oracle as ora  # noqa: E402
from paper_2402_10517_b200 import AnyPrecisionLayer, engine  # noqa: E402

def prep_of(r, c):
    codes, tables = ora.random_layer_arrays(np.random.default_rng(0), r, c, 3, 8)
    return engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(r, c)))

print(json.dumps(bench.run_prefill(torch, [None] * 4 + [prep_of(11008, 4096)])))
p = prep_of(4096, 4096)
out = {}
for impl in ("tcgen05", "cublas"):
    engine._DENSE_IMPL = impl
    for m in (17, 64, 128):
        x = torch.randn(m, 4096, device="cuda")
        cfg = engine.GemvConfig(bit_width=4, dense_threshold=16)
        engine.gemm(p, x, cfg)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            engine.gemm(p, x, cfg)
        b.record()
        torch.cuda.synchronize()
        out.setdefault(f"M{m}", {})[impl] = round(a.elapsed_time(b) / 20, 4)
print(json.dumps({"layer": "4096x4096 k=4 (ms)", "per_M": out}))

# kernel-only: the two C-ABI launches (activation prep + fused GEMM [+ split-K sum])
# captured in a CUDA graph and replayed (no Python in the timed region)
from paper_2402_10517_b200 import _device as dev  # noqa: E402
from paper_2402_10517_b200._lib import check, load  # noqa: E402

L = load()
kern = {}
for name, pr in (("4096x4096", p), ("11008x4096", prep_of(11008, 4096))):
    t = pr.tensor
    for m in (17, 64, 128, 512, 2048):
        x = torch.randn(m, t.cols, device="cuda")
        xp = torch.empty((2 * m, t.padded_cols), dtype=torch.float16, device="cuda")
        inv = torch.empty(m, dtype=torch.float32, device="cuda")
        y = torch.empty((m, t.rows), dtype=torch.float32, device="cuda")
        wsb = L.apb_gemm_dense_tc_workspace(t.rows, t.padded_cols, 2 * m)
        ws = torch.empty(max(wsb // 4, 1), dtype=torch.float32, device="cuda")

        def run():
            s = dev.stream_ptr()
            check(L.apb_dense_prep_x(dev.ptr(x), 0, m, t.cols, t.cols, dev.ptr(xp), t.padded_cols, dev.ptr(inv), s), "p")
            check(L.apb_gemm_dense_tc(dev.ptr(t.planes), t.n_max, t.rows, t.cols, t.padded_cols, 4,
                                      dev.ptr(pr.tables16[4]), dev.ptr(xp), 2 * m, 1, dev.ptr(inv), dev.ptr(y),
                                      t.rows, dev.ptr(ws), wsb, s), "g")
        run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                run()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        kern.setdefault(name, {})[f"M{m}"] = {"ms": round(ms, 4), "splits": wsb // max(1, 4 * 2 * m * t.rows),
                                             "TFLOPs": round(2 * m * t.rows * t.cols / (ms * 1e-3) / 1e12, 1)}
print(json.dumps({"kernel_only_k4": kern}))
