"""Top CUDA source lines by warp-stall samples from an ncu report (no GPU needed).
usage: python tools/ncu_src.py report.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.defaultdict(lambda: [0.0, collections.Counter(), ""])
for r in rows[hi + 1:]:
    if len(r) != len(h) or not r[0].isdigit():
        continue
    v = float(r[si] or 0)
    a = agg[int(r[0])]
    a[0] += v
    a[2] = r[1]
    for i, c in stall_cols:
        a[1][c[6:]] += float(r[i] or 0)
tot = sum(a[0] for a in agg.values())
print(f"total samples {tot:.0f}")
for ln, (v, cnt, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = " ".join(f"{k}={x:.0f}" for k, x in cnt.most_common(3) if x)
    print(f"{ln:5d} {v:6.0f} {v / tot * 100:5.1f}%  {src.strip()[:64]:64s} {top}")
