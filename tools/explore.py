"""Exploration: layer-set throughput under launch variants (CUDA graph timing)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2402_10517_b200 import plan

torch.cuda.set_device(0)
copies = [bench.make_layer_set(torch, 1234 + c, 0, 1) for c in range(bench.N_COPIES)]
sb = bench.step_bytes(bench.SHAPES)

def measure(make_plans, reps=50, label=""):
    plans = make_plans()
    for p in plans:
        for x in p.x: x.normal_()
    def step():
        for p in plans: p.run()
    step(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): g.replay()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{label:40s} {ms*1e3:9.1f} us/step  {sb/(ms*1e-3)/1e9:8.1f} GB/s", flush=True)
    return plans

def per_layer(pdl):
    out = []; i = 0
    for k in bench.BITS:
        for li in range(len(bench.SHAPES)):
            out.append(plan.GemvPlan([copies[i % bench.N_COPIES][li]], k, grouped=False, pdl=pdl)); i += 1
    return out

def grouped(pdl):
    return [plan.GemvPlan(copies[j % bench.N_COPIES], k, grouped=True, pdl=pdl) for j, k in enumerate(bench.BITS)]

measure(lambda: per_layer(False), label="per-layer")
measure(lambda: per_layer(True), label="per-layer + PDL")
measure(lambda: grouped(False), label="grouped")
measure(lambda: grouped(True), label="grouped + PDL")
# per-k per-shape with PDL chain of 20 identical launches (rotating copies)
for k in bench.BITS:
    row = []
    for li, (n, r, c) in enumerate(bench.SHAPES):
        ps = [plan.GemvPlan([copies[j][li]], k, grouped=False, pdl=True) for j in range(bench.N_COPIES)]
        def st():
            for _ in range(5):
                for p in ps: p.run()
        st(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g): st()
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): g.replay()
        b.record(); torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (10 * 5 * len(ps))
        row.append(f"{n}:{us:.2f}us/{bench.alg_bytes(r, c, k)/(us*1e-6)/1e9:.0f}")
    print(f"k={k}", " ".join(row), flush=True)
