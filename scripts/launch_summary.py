"""Mean per-kernel duration from ncu --csv launch lists (gpu__time_duration.sum)."""
import csv
import sys
from collections import defaultdict

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    h = rows[0]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    d = defaultdict(list)
    for r in rows[1:]:
        d[(r[ki][:60], r[gi])].append(float(r[vi].replace(",", "")))
    print(f)
    for (k, g), v in d.items():
        print("  %-60s %-14s n=%3d mean=%8.0f ns" % (k, g, len(v), sum(v) / len(v)))
