import json, sys
d = json.load(open(sys.argv[1]))
pg = d.pop("per_gemv_us", {})
print({k: d.get(k) for k in ("value", "ms_per_step", "grouped_all7_GBps", "gpu_launches")}, "frac", d["roofline"]["frac"],
      d["clocks"], "e2e", d.get("e2e", {}).get("value"), "cpu", d.get("cpu_baseline", {}).get("value"))
for k, v in pg.items():
    print(k, " ".join(f"{n.split('_')[0]}:{x['us']:.1f}us/{x['GBps']:.0f}" for n, x in v.items()))
