import sys, torch
sys.path.insert(0, '.')
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
w16 = torch.randn(11008, 4096, device="cuda").half()
for m in (64, 512):
    x = torch.randn(m, 4096, device="cuda")
    a16 = torch.randn(2 * m, 4096, device="cuda").half()
    print(m, "mm out_dtype f32 us", round(t(lambda: torch.mm(a16, w16.T, out_dtype=torch.float32)), 1),
          "| mm f16 out us", round(t(lambda: torch.mm(a16, w16.T)), 1))
    def split():
        amax = x.abs().amax(dim=1, keepdim=True)
        expo = torch.floor(torch.log2(torch.where(amax > 0, amax, torch.ones_like(amax))))
        scale = torch.exp2(14.0 - expo)
        xs = x * scale
        hi = xs.to(torch.float16)
        lo = (xs - hi.to(torch.float32)).to(torch.float16)
        return torch.cat([hi, lo])
    print(m, "split us", round(t(split), 1))
from paper_2402_10517_b200 import engine, AnyPrecisionLayer
from paper_2402_10517_b200.engine import _dequant_device
from paper_2402_10517_b200._lib import APB_DTYPE_F16
import numpy as np
from oracle import oracle as ora
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 11008, 4096, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(11008, 4096)))
print("dequant f16 k4 us", round(t(lambda: _dequant_device(prep, 4, APB_DTYPE_F16)), 1))
