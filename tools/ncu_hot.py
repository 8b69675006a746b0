"""Per-instruction stall samples of a kernel in an ncu report (top N lines outside a given range)."""
import csv, subprocess, sys
rep = sys.argv[1]; lo = int(sys.argv[2]); hi = int(sys.argv[3]); topn = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:gemv",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
seen = set(); uniq = []
for r in data:
    if r[0] in seen: break
    seen.add(r[0]); uniq.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iSrc = hdr.index("Source"); iE = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lst = []
for i, r in enumerate(uniq):
    if lo <= i <= hi: continue
    try: s = int(r[iS])
    except: continue
    if s == 0: continue
    top = sorted(((int(float(r[hdr.index(c)] or 0)), c[6:]) for c in cols), reverse=True)[:2]
    lst.append((s, i, r[iSrc].strip()[:70], r[iE], top))
lst.sort(reverse=True)
for s, i, src, e, top in lst[:topn]:
    print(f"{i:5d} {s:5d} exec {e:>9} {top}  {src}")
