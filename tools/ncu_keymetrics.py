"""Key metrics of single-kernel ncu --set full captures -> markdown rows."""
import csv, subprocess, sys
KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts % of peak"),
        ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem tensor-core wavefronts % of peak"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (realtime)"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]
print("| capture | kernel | " + " | ".join(n for _, n in KEYS) + " |")
print("|---|---|" + "---|" * len(KEYS))
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u = rr[0], rr[1]
    for d in rr[2:]:
        vals = []
        for m, _ in KEYS:
            if m in h:
                i = h.index(m)
                vals.append(f"{d[i]} {u[i]}".strip())
            else:
                vals.append("n/a")
        name = d[h.index("Kernel Name")].replace("void ", "").split("(")[0]
        print(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(vals) + " |")
