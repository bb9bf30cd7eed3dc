"""Summarise bench.py JSON lines from stdin: workload, us/step, value, unit, roofline frac."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "unavailable" in d:
        print(d)
        continue
    r = d.get("roofline") or {}
    cfg = d.get("config", {})
    print("%-8s B=%-4s n=%-3s %9.2f us/step  %9.2f %-8s frac %.3f  kernel_us %s  clocks %s" % (
        cfg.get("workload", "")[:8], cfg.get("batch"), cfg.get("n"), d["ms_per_step"] * 1e3, d["value"], d["unit"],
        r.get("frac", float("nan")), r.get("kernel_us"), (d.get("clocks") or {}).get("sm_mhz")))
