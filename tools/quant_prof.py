import sys, torch
sys.path.insert(0, '.')
from paper_2402_10517_b200.quantizer import build_any_precision
g = torch.Generator(device='cuda').manual_seed(0)
rows, cols = int(sys.argv[1]), int(sys.argv[2])
w = torch.randn(rows, cols, device='cuda', dtype=torch.float64, generator=g) * 0.02
s = torch.rand(rows, cols, device='cuda', dtype=torch.float64, generator=g)
build_any_precision(w, s, 3, 8, as_numpy=False)
torch.cuda.synchronize()
