"""Kernel timeline of one captured decode step (CUPTI via torch.profiler):
per-kernel-class total device time and the idle gaps between kernels."""
import json, sys, collections, torch
sys.path.insert(0, '.')
from paper_2402_10517_b200.decode import DecodeModel, LlamaConfig
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = DecodeModel(LlamaConfig())
m.capture(k)
for _ in range(5): m.step(k)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): m.step(k)
    torch.cuda.synchronize()
prof.export_chrome_trace('gpurun_out/dec_trace.json')
ev = [e for e in json.load(open('gpurun_out/dec_trace.json'))['traceEvents'] if e.get('cat') == 'kernel']
ev.sort(key=lambda e: e['ts'])
n = len(ev) // 3
ev = ev[n:2 * n]   # middle replay
tot = collections.defaultdict(float); cnt = collections.Counter(); gap = collections.defaultdict(float)
for i, e in enumerate(ev):
    name = e['name'].replace('(anonymous namespace)::', '').split('(')[0][:60]
    tot[name] += e['dur']; cnt[name] += 1
    if i:
        prev_end = ev[i - 1]['ts'] + ev[i - 1]['dur']
        gap[name] += e['ts'] - prev_end
span = ev[-1]['ts'] + ev[-1]['dur'] - ev[0]['ts']
print(f"k={k} kernels/step={len(ev)} span={span:.0f}us")
for nme in sorted(tot, key=lambda x: -tot[x]):
    print(f"{nme:60s} n={cnt[nme]:4d} dur={tot[nme]:8.1f}us gap_before={gap[nme]:8.1f}us")

print('--- one block (middle of the step): start offset / duration us')
i0 = len(ev) // 2
while 'attention' not in ev[i0]['name']:
    i0 += 1
i0 -= 1  # the q/k/v GEMV before it
t0 = ev[i0]['ts']
for e in ev[i0:i0 + 6]:
    nm = e['name'].replace('(anonymous namespace)::', '').split('(')[0][:40]
    print(f"{nm:40s} start={e['ts'] - t0:8.2f} dur={e['dur']:7.2f} end={e['ts'] + e['dur'] - t0:8.2f}")
