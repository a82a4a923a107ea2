"""Print the per-launch sequence (name, duration us, grid) of an ncu --csv launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, g = None, OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        g.setdefault((int(d["ID"]), d["Kernel Name"][:40]), {})[d["Metric Name"]] = d["Metric Value"]
for (i, k), d in list(g.items())[-last:]:
    t = float(d.get("gpu__time_duration.sum", "0").replace(",", ""))
    print(f"{i:5d} {k:40s} {t / 1e3:8.2f} us  grid {d.get('launch__grid_size', '?')}")
