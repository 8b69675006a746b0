"""Per-CTA phase timeline of the GEMV kernel (instrumented build)."""
import ctypes, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_2402_10517_b200 import _lib
_lib.LIB_PATH = os.path.join(HERE, "libanyprec_b200_tl.so")
lib = _lib.load()
lib.apb_debug_set_timeline.argtypes = [ctypes.c_void_p]
import torch
from paper_2402_10517_b200 import AnyPrecisionLayer, engine, plan

torch.cuda.set_device(0)
shapes = [(4096, 4096), (11008, 4096), (4096, 11008)]
for rows, cols in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    codes = torch.randint(0, 256, (rows, cols), dtype=torch.uint8, device="cuda", generator=g)
    tables = {k: torch.sort(torch.randn(rows, 1 << k, device="cuda", generator=g), 1).values.half() for k in range(3, 9)}
    prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(rows, cols)))
    nblk = -(-rows // 16)
    tl = torch.zeros(nblk * 8, dtype=torch.int64, device="cuda")
    for k in (3, 4, 8):
        p = plan.GemvPlan([prep], k, grouped=False)
        p.x[0].normal_()
        p.run(); torch.cuda.synchronize()
        lib.apb_debug_set_timeline(ctypes.c_void_p(tl.data_ptr()))
        tl.zero_()
        p.run(); torch.cuda.synchronize()
        lib.apb_debug_set_timeline(ctypes.c_void_p(0))
        t = tl.view(nblk, 8).cpu().numpy().astype(np.int64)[:, :6]
        t = t[t[:, 5] > 0]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0  # us
        ph = np.diff(t, axis=1) / 1000.0
        names = ["issue_planes", "lut+table", "x_stage", "items_main", "last_epilogue"]
        print(f"{rows}x{cols} k={k}: kernel span {rel[:,5].max():.2f} us; CTA start spread {rel[:,0].min():.2f}..{rel[:,0].max():.2f}; ")
        print("   phase medians(us): " + " ".join(f"{n}={np.median(ph[:,i]):.2f}/max{ph[:,i].max():.2f}" for i, n in enumerate(names)))
        # waves: histogram of start times
        hist, edges = np.histogram(rel[:, 0], bins=6)
        print("   start hist:", list(hist), [round(e, 1) for e in edges])
