"""ncu launch list of one decode token -> per-kernel share (profiles/<tag>_decode_launches.md)."""
import collections, csv, sys
tag, paths = sys.argv[1], sys.argv[2:]
out = [f"# {tag}: ncu launch list of ONE decode token (`tools/decode_token.py k`, "
       "`ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none`; "
       "cold-cache serialised kernel times -- shares, not the graph's overlapped time)\n"]
for p in paths:
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    by = collections.defaultdict(list)
    for r in rows:
        n = r[iN].replace("void ", "")
        short = n.split("(")[0]
        if "gemv7_kernel" in n:
            short = "gemv7_kernel (quantized linears)"
        by[short[-80:]].append(float(r[iV].replace(",", "")))
    tot = sum(sum(v) for v in by.values())
    out.append(f"\n## {p.split('/')[-1]}: {sum(len(v) for v in by.values())} launches, {tot/1e3:.1f} us serialised\n")
    out.append("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v)/1e3:.1f} | {100*sum(v)/tot:.1f} % |")
open(f"profiles/{tag}_decode_launches.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
