"""gemm-dense: fp16-exact dequant + hi/lo tensor-core GEMM vs fp32 dequant + fp32 GEMM."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2402_10517_b200 import engine, AnyPrecisionLayer
from paper_2402_10517_b200.engine import _dequant_device, _dense_tensor_core
from paper_2402_10517_b200._lib import APB_DTYPE_F16, APB_DTYPE_F32
from oracle import oracle as ora
codes, tables = ora.random_layer_arrays(np.random.default_rng(0), 11008, 4096, 3, 8)
prep = engine.prepare(AnyPrecisionLayer(n_min=3, n_max=8, codes=codes, centroid_tables=tables, shape=(11008, 4096)))
torch.backends.cuda.matmul.allow_tf32 = False
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
for m in (64, 512, 2048):
    X = torch.randn(m, 4096, device="cuda")
    new = t(lambda: _dense_tensor_core(torch, X, _dequant_device(prep, 4, APB_DTYPE_F16), False))
    old = t(lambda: X @ _dequant_device(prep, 4, APB_DTYPE_F32).T)
    w16 = _dequant_device(prep, 4, APB_DTYPE_F16)
    gemm_only = t(lambda: _dense_tensor_core(torch, X, w16, False))
    print(f"M={m}: tensor-core path {new:.3f} ms (GEMM part {gemm_only:.3f}) | fp32 SIMT path {old:.3f} ms")
