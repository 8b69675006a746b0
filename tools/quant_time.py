"""GPU quantizer wall time per Llama-2-7B layer shape (k = 3..8, inputs on device)."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2402_10517_b200.quantizer import build_any_precision
g = torch.Generator(device='cuda').manual_seed(0)
for rows, cols in ((4096, 4096), (11008, 4096), (4096, 11008)):
    w = torch.randn(rows, cols, device='cuda', dtype=torch.float64, generator=g) * 0.02
    s = torch.rand(rows, cols, device='cuda', dtype=torch.float64, generator=g)
    build_any_precision(w[:64], s[:64], 3, 8, as_numpy=False)
    torch.cuda.synchronize()
    for rep in range(2):  # the first full-size call also allocates the workspace
        t = time.perf_counter()
        build_any_precision(w, s, 3, 8, as_numpy=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"{rows}x{cols} (run {rep}): {dt*1e3:.1f} ms ({dt/rows*1e6:.1f} us/row)")
