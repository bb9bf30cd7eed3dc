import csv, json, re, sys
from collections import defaultdict
for wl in ("c3_up", "c3_down"):
    try:
        d = json.load(open(f"gpurun_out/pf_{wl}.json"))
        r = d["roofline"]
        print(f"{wl}: value {d['value']:.1f} {d['unit']}  us/step {d['ms_per_step']*1e3:.1f}  gemm {r['kernel_us']:.1f} us "
              f"{r['achieved']:.0f} TF/s frac {r['frac']:.3f}  clocks {d['clocks'].get('sm_mhz')}")
    except Exception as e:
        print(wl, "n/a", e)
rows = list(csv.reader(open("gpurun_out/pf_launches.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
agg = defaultdict(list)
for r in rows[i + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") == "gpu__time_duration.sum":
        agg[re.sub(r"\(.*", "", d["Kernel Name"])].append(float(d["Metric Value"]) / 1000)
for k, v in agg.items():
    print(f"  {k:40s} n={len(v)} avg {sum(v)/len(v):.1f} us")
