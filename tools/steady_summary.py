"""profiles/<tag>_steady_state.md from full ncu captures of one steady-state
launch per k (tools/kbench 28672x8192): pipes, wavefronts, stalls, main-loop mix."""
import collections, csv, subprocess, sys

tag, reps = sys.argv[1], sys.argv[2:]
M = [("gpu__time_duration.sum", "duration (ncu, cold, us)"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
     ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
     ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU issue %"),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
     ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
     ("sm__cycles_elapsed.avg", "SM cycles"),
     ("dram__bytes_read.sum", "DRAM read")]
out = [f"# {tag}: steady-state launch (28672x8192, `tools/kbench`), `ncu --set full --clock-control none`\n",
       "Cold-cache, serialised capture (durations are not bench numbers).  smem wavefronts / (SM cycles x 148)"
       " is the shared-memory data-path utilisation (1 wavefront per cycle per SM).\n",
       "| k | " + " | ".join(n for _, n in M) + " | smem wavefronts / SM / cycle | top stalls (samples) |",
       "|" + "---|" * (len(M) + 3)]
for rep in reps:
    raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                         text=True).stdout.splitlines()))
    h, v = raw[0], raw[2]
    get = lambda m: v[h.index(m)] if m in h else "?"
    name = get("Kernel Name")
    k = name.split("<")[1].split(",")[0] if "<" in name else "?"
    vals = [get(m) for m, _ in M]
    try:
        util = float(get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")) / (float(get("sm__cycles_elapsed.avg")) * 148)
    except ValueError:
        util = float("nan")
    src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                         capture_output=True, text=True).stdout.splitlines()))
    hs = src[1]
    rows = [r for r in src[2:] if len(r) == len(hs) and r[0].startswith("0x")]
    seen, uniq = set(), []
    for r in rows:
        if r[0] in seen:
            break
        seen.add(r[0]); uniq.append(r)
    stalls = collections.Counter()
    for c in hs:
        if c.startswith("stall_") and "Not Issued" not in c:
            stalls[c[6:]] = sum(int(float(r[hs.index(c)] or 0)) for r in uniq)
    top = ", ".join(f"{n} {c}" for n, c in stalls.most_common(5))
    out.append(f"| {k} | " + " | ".join(vals) + f" | {util:.2f} | {top} |")
    # hottest basic block's opcode mix
    iE, iS = hs.index("Instructions Executed"), hs.index("Source")
    best, cur = None, []
    for r in uniq:
        e = int(r[iE] or 0)
        if cur and e != int(cur[-1][iE] or 0):
            if best is None or len(cur) * int(cur[0][iE] or 0) > len(best) * int(best[0][iE] or 0):
                best = cur
            cur = []
        cur.append(r)
    if best:
        mix = collections.Counter((r[iS].split()[1] if r[iS].startswith("@") else r[iS].split()[0]).split(".")[0]
                                  for r in best)
        out.append(f"|  | hottest block: {len(best)} instructions x {best[0][iE]} executions: "
                   + ", ".join(f"{op} {n}" for op, n in mix.most_common(8)) + " |" + " |" * (len(M) + 1))
open(f"profiles/{tag}_steady_state.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
