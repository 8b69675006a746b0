"""ncu --cache-control none capture of the timed launch pattern -> profiles/<tag>_traffic.json.

Input: the CSV of tools/gpu_r2.sh (TRAFFIC leg: `ncu --cache-control none
--metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,
gpu__time_duration.sum` over whole steps of `bench.py --profile`, i.e. the
bench's own launch order and weight-copy rotation, caches in their natural
state between launches).  Output: per-launch DRAM bytes vs the SURVEY 8(d)
algorithmic bytes and the L2 hit rate, and the whole-step ratio bench.py
reports as roofline.traffic."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main(csv_path, out_path):
    rows = list(csv.reader(open(csv_path)))
    hdr, by, names = None, collections.defaultdict(dict), {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            by[int(d["ID"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
            names[int(d["ID"])] = d["Kernel Name"]
    alg = [sum(bench.alg_bytes(bench.SHAPES[j][1], bench.SHAPES[j][2], k) for j in g)
           for k in bench.BITS for g in bench.GROUPS]
    per = len(alg)
    launches, tot_d, tot_a = [], 0.0, 0.0
    for i in sorted(by):
        m = by[i]
        d = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        a = alg[i % per]
        tot_d += d
        tot_a += a
        k = bench.BITS[(i % per) // len(bench.GROUPS)]
        grp = "+".join(bench.SHAPES[j][0] for j in bench.GROUPS[i % len(bench.GROUPS)])
        launches.append({"launch": i, "k": k, "group": grp, "kernel": names[i].split("(")[0],
                         "dram_bytes": int(d), "alg_bytes": a, "dram_over_alg": round(d / a, 4),
                         "l2_hit_pct": m["lts__t_sector_hit_rate.pct"],
                         "ncu_us_serialised": round(m["gpu__time_duration.sum"] / 1e3, 2)})
    out = {"source": os.path.basename(csv_path) + " (ncu --cache-control none, timed launch pattern of "
                     "bench.py --profile: whole steps in the bench's own order and copy rotation)",
           "steps": len(launches) // per, "dram_over_algorithmic": round(tot_d / tot_a, 4),
           "min_launch_ratio": min(l["dram_over_alg"] for l in launches),
           "max_launch_ratio": max(l["dram_over_alg"] for l in launches),
           "launches": launches}
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    print(out_path, out["dram_over_algorithmic"], out["min_launch_ratio"], out["max_launch_ratio"])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
