"""Stall-reason breakdown of a kernel in an ncu report, overall and inside loops."""
import csv, re, subprocess, sys, collections
rep, skip = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:gemv", "--launch-skip", str(skip), "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
seen = set(); uniq = []
for r in data:
    if r[0] in seen: break
    seen.add(r[0]); uniq.append(r)
data = uniq
iS = hdr.index("Warp Stall Sampling (All Samples)"); iSrc = hdr.index("Source"); iE = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def region(a, b):
    tot = collections.Counter(); n = 0; ex = 0
    for r in data[a:b]:
        try: n += int(r[iS]); ex += int(r[iE])
        except: pass
        for c in cols:
            try: tot[c] += int(float(r[hdr.index(c)]))
            except: pass
    return n, ex, tot.most_common(8)
addr = [int(r[0], 16) for r in data]
print("kernel:", rows[0][1][:60], "instructions:", len(data))
print("ALL", region(0, len(data)))
for i, r in enumerate(data):
    m = re.search(r"BRA (0x[0-9a-f]+)", r[iSrc])
    if m:
        t = int(m.group(1), 16)
        if t < addr[i] and t in addr:
            j = addr.index(t)
            n, ex, st = region(j, i + 1)
            if n > 5: print(f"loop {j}..{i}: samples {n} exec {ex} {st}")

# executed-instruction histogram by contiguous blocks of equal exec count (basic blocks)
blocks = []
cur = None
for i, r in enumerate(data):
    try: e = int(r[iE])
    except: e = 0
    s = int(r[iS]) if r[iS].isdigit() else 0
    if cur and cur[2] == e: cur[1] = i; cur[3] += e; cur[4] += s
    else:
        cur = [i, i, e, e, s]; blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
print("top basic blocks (start..end exec_per_inst total samples):")
for b in blocks[:12]:
    print(f"  {b[0]}..{b[1]} x{b[2]} total {b[3]} samples {b[4]}  first: {data[b[0]][iSrc].strip()[:60]}")
