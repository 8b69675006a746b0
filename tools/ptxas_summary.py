"""Registers / stack / spills / smem of every kernel from the build's ptxas -v
logs (paper_2402_10517_b200/csrc/*.ptxas.log) -> profiles/<tag>_ptxas.md."""
import glob, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
rows = []
for log in sorted(glob.glob(os.path.join(ROOT, "paper_2402_10517_b200/csrc/*.ptxas.log"))):
    text = open(log).read()
    for blk in text.split("ptxas info    : Compiling entry function")[1:]:
        name = re.search(r"'(\S+)'", blk).group(1)
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(anonymous namespace\)::", "", dem).split("(")[0]
        rg = re.search(r"Used (\d+) registers", blk)
        st = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", blk)
        sm = re.search(r"(\d+) bytes smem", blk)
        rows.append((os.path.basename(log).split(".")[0], dem, rg.group(1) if rg else "?",
                     st.group(1) if st else "?", st.group(2) if st else "?", sm.group(1) if sm else "0"))
out = [f"# {tag}: ptxas -v of every kernel (sm_100a, -O3)\n",
       "| source | kernel | regs | stack B | spill stores B | static smem B |", "|---|---|---|---|---|---|"]
out += [f"| {a} | `{b}` | {c} | {d} | {e} | {f} |" for a, b, c, d, e, f in rows]
path = os.path.join(ROOT, "profiles", f"{tag}_ptxas.md")
open(path, "w").write("\n".join(out) + "\n")
print(path, len(rows), "kernels")
