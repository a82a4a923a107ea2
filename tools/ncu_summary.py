"""Summarise ncu artefacts into text for profiles/ (run here, no GPU).
usage: python tools/ncu_summary.py launches.csv report.ncu-rep > profiles/xxx.txt"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    txt = open(path).read()
    txt = txt[txt.find('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(txt)))
    d = collections.defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            d[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print(f"== launch list ({path}): {sum(len(v) for v in d.values())} launches, "
          "gpu__time_duration.sum (cold-cache, serialised; compare shares)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {len(v):5d} x {sum(v) / len(v) / 1e3:9.2f} us  share {sum(v) / tot * 100:5.1f}%  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size"]
    print(f"== ncu --set full ({path})")
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {v[i]} {u[i]}")
    rb = float(v[h.index("dram__bytes_read.sum")].replace(",", "")) if "dram__bytes_read.sum" in h else 0
    wb = float(v[h.index("dram__bytes_write.sum")].replace(",", "")) if "dram__bytes_write.sum" in h else 0
    unit = u[h.index("dram__bytes_read.sum")]
    print(f"  traffic (dram read + write) = {rb + wb:.3f} {unit}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        if p.endswith(".csv"):
            launches(p)
        else:
            full(p)
