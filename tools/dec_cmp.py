"""Decode-step tokens/s (bench C5 leg) -- quick A/B helper."""
import sys, torch
sys.path.insert(0, '.')
import bench
import os
if os.environ.get('NO_KV_PF'):
    from paper_2402_10517_b200 import decode
    orig = decode.DecodeModel.__init__
    def init(self, *a, **kw):
        orig(self, *a, **kw); self.kv_prefetch = False
    decode.DecodeModel.__init__ = init
out = bench.run_decode(torch, steps=20)
print({k: v['tokens_per_s'] for k, v in out['per_k'].items()})
