"""Summarise an ncu launch list + full capture into profiles/<tag>_*.md."""
import csv, collections, subprocess, sys, os, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench

tag, launches, full = sys.argv[1], sys.argv[2], sys.argv[3]
out = []
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
by = collections.defaultdict(list)
for r in rows:
    name = r[iN]
    short = "gemv_kernel" if "gemv" in name else name.split("(")[0][-70:]
    by[short].append(float(r[iV]))
tot = sum(sum(v) for v in by.values())
out.append(f"# {tag}: ncu launch list of `python bench.py --profile --steps 2 --warmup 3`\n")
out.append("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares, not absolutes).\n")
out.append("| kernel | launches | total µs | share |\n|---|---|---|---|")
for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
    out.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% |")
g = by.get("gemv_kernel", [])
# the last 2 steps x 24 launches are the timed steps; map each launch to its bytes
per_launch = []
for kbit in bench.BITS:
    for grp in bench.GROUPS:
        per_launch.append(sum(bench.alg_bytes(bench.SHAPES[j][1], bench.SHAPES[j][2], kbit) for j in grp))
last = g[-48:]
if len(last) == 48:
    out.append("\nGEMV launches of the 2 timed steps (per k: qkv | o | gate+up | down):\n")
    out.append("| k | launch | µs (ncu) | alg. MB | GB/s |\n|---|---|---|---|---|")
    names = ["qkv", "o", "gate+up", "down"]
    for i in range(24):
        us = (last[i] + last[24 + i]) / 2 / 1e3
        b = per_launch[i]
        out.append(f"| {bench.BITS[i//4]} | {names[i%4]} | {us:.2f} | {b/1e6:.2f} | {b/(us*1e-6)/1e9:.0f} |")
    step_us = sum(last[:24]) / 1e3
    out.append(f"\nSum of GEMV launch times per step (ncu, serialised): {step_us:.1f} µs -> {bench.step_bytes()/(step_us*1e-6)/1e9:.0f} GB/s; "
               f"GEMV share of all profiled GPU time: {100*sum(g)/tot:.1f}% (the rest is setup: RNG, packing).")
open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(out) + "\n")

# full capture
raw = subprocess.run(["ncu", "-i", full, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, data = rr[0], rr[1], rr[2:]
want = [("Kernel Name", ""), ("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("launch__shared_mem_per_block_dynamic", "dyn smem"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts")]
o2 = [f"# {tag}: `ncu --set full --clock-control none` of 4 GEMV launches inside the timed bench steps\n"]
want += [("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
         ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
         ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem conflicts")]
o2.append("| " + " | ".join(n or "kernel" for _, n in want) + " |")
o2.append("|" + "---|" * len(want))
for d in data:
    vals = []
    for m, n in want:
        if m in h:
            i = h.index(m); v = d[i]
            vals.append(f"{v} {u[i]}".strip() if m != "Kernel Name" else v.replace("void ", "").split("(")[0])
        else:
            vals.append("n/a")
    o2.append("| " + " | ".join(vals) + " |")
open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.md"), "w").write("\n".join(o2) + "\n")
print("\n".join(out[-8:])); print("\n".join(o2))

# per-launch DRAM traffic vs algorithmic bytes (bench.py reads this for roofline.traffic)
tr = []
for d in data:
    name = d[h.index("Kernel Name")]
    if "gemv" not in name:
        continue
    rd = float(d[h.index("dram__bytes_read.sum")]); wr = float(d[h.index("dram__bytes_write.sum")])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(u[h.index("dram__bytes_read.sum")], 1); wr *= scale.get(u[h.index("dram__bytes_write.sum")], 1)
    tr.append({"kernel": name.split("(")[0].replace("void ", ""), "dram_bytes": rd + wr})
json.dump({"source": f"profiles/{tag}_ncu_full.md (ncu --set full)", "launches": tr},
          open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_traffic.json"), "w"), indent=1)
