"""Per-warp cycle split (prologue / in-unit / boundary) for single and grouped launches."""
import ctypes, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2402_10517_b200 import _lib
_lib.LIB_PATH = os.path.join(HERE, "libanyprec_b200_tl.so")
lib = _lib.load()
lib.apb_debug_set_warpstat.argtypes = [ctypes.c_void_p]
import torch
import bench
from paper_2402_10517_b200 import plan
torch.cuda.set_device(0)
preps = bench.make_layer_set(torch, 1, 0, 1)
ws = torch.zeros(148 * 4 * 8 * 4, dtype=torch.int64, device="cuda")
def run(p, label):
    for x in p.x: x.normal_()
    p.run(); torch.cuda.synchronize()
    ws.zero_(); lib.apb_debug_set_warpstat(ctypes.c_void_p(ws.data_ptr()))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); p.run(); b.record(); torch.cuda.synchronize()
    lib.apb_debug_set_warpstat(ctypes.c_void_p(0))
    w = ws.view(-1, 4).cpu().numpy().astype(np.float64)
    w = w[w[:, 2] > 0]
    pro, uni, tot, n = w[:, 0], w[:, 1], w[:, 2], w[:, 3]
    bnd = tot - pro - uni
    print(f"{label:28s} {a.elapsed_time(b)*1e3:8.1f}us warps={len(w)} units/warp={n.mean():.1f} "
          f"cyc: total {tot.mean():8.0f} (max {tot.max():.0f}) prologue {pro.mean():7.0f} units {uni.mean():8.0f} "
          f"boundary {bnd.mean():7.0f}  per-unit {uni.sum()/max(n.sum(),1):6.0f}")
for k in (3, 4, 8):
    run(plan.GemvPlan(preps, k, grouped=True), f"grouped 7 layers k={k}")
    run(plan.GemvPlan([preps[4]], k, grouped=False), f"11008x4096 k={k}")
    run(plan.GemvPlan([preps[0]], k, grouped=False), f"4096x4096 k={k}")
