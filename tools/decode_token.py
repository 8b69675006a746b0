"""One decode token at bit-width k (for an ncu launch list): DecodeModel at the
bench's context, warm-up steps, then NVTX-free single step; pass k as argv[1]."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2402_10517_b200.decode import DecodeModel
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = DecodeModel(context=1024)
m.capture(k)
for _ in range(3):
    m.step(k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
m.step(k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
