"""apb_attention_decode alone: per-call time in a back-to-back PDL chain (graph)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2402_10517_b200 import _device as dev
from paper_2402_10517_b200._lib import check, load
lib, hd = load(), 128
for heads, pos in ((32, 1024), (32, 4095)):
    stride = (pos + 1) * hd
    q, k, v = (torch.randn(heads * hd, device="cuda").half() for _ in range(3))
    kc = torch.randn(heads * stride, device="cuda").half(); vc = torch.randn_like(kc)
    nk = torch.randn_like(kc); nv = torch.randn_like(kc)
    ang = torch.rand(hd // 2, device="cuda"); cos, sin = torch.cos(ang), torch.sin(ang)
    nb = lib.apb_attention_decode_workspace(heads, hd, pos + 1)
    ws = torch.zeros(nb, device="cuda", dtype=torch.uint8)
    out = torch.empty(heads * hd, device="cuda", dtype=torch.float16)
    P = dev.ptr
    def call(pf):
        check(lib.apb_attention_decode(P(q), P(k), P(v), P(cos), P(sin), P(kc), P(vc), heads, hd, stride, pos,
                                       hd ** -0.5, P(ws), nb, P(out), P(nk) if pf else None, P(nv) if pf else None,
                                       dev.stream_ptr()), "attn")
    for pf in (False, True):
        call(pf); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(50): call(pf)
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / 50
        kv = 2 * heads * (pos + 1) * hd * 2
        print(f"heads={heads} keys={pos+1} prefetch_next={pf}: {us:.2f} us/call  KV {kv/1e6:.1f} MB -> {kv/us/1e3:.0f} GB/s")
