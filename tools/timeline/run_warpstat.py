"""Per-compute-warp cycle split: in-unit loop (incl. load waits), load waits, table waits."""
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
ws = torch.zeros(148 * 16 * 8, dtype=torch.int64, device="cuda")
def run(p, label):
    for x in p.x: x.normal_()
    p.run(); torch.cuda.synchronize()
    ws.zero_(); lib.apb_debug_set_warpstat(ctypes.c_void_p(ws.data_ptr()))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); p.run(); b.record(); torch.cuda.synchronize()
    lib.apb_debug_set_warpstat(ctypes.c_void_p(0))
    w = ws.view(-1, 8).cpu().numpy().astype(np.float64)
    w = w[w[:, 0] > 0]
    tot, uni, ldw, tbw, n = w[:, 0], w[:, 1], w[:, 2], w[:, 3], w[:, 4]
    print(f"{label:26s} {a.elapsed_time(b)*1e3:7.1f}us warps={len(w)} units/warp={n.mean():5.1f} "
          f"total {tot.mean():7.0f} (max {tot.max():.0f}) unit-loop {uni.mean():7.0f} [ldwait {ldw.mean():6.0f}] "
          f"tblwait {tbw.mean():6.0f} other {np.mean(tot-uni-tbw):6.0f} | per-unit compute {(uni-ldw).sum()/n.sum():5.0f} ldwait {ldw.sum()/n.sum():5.0f}")
for k in (3, 4, 8):
    run(plan.GemvPlan(preps, k, grouped=True), f"grouped 7 layers k={k}")
    run(plan.GemvPlan([preps[4]], k, grouped=False), f"11008x4096 k={k}")
    run(plan.GemvPlan([preps[0]], k, grouped=False), f"4096x4096 k={k}")
