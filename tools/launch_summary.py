"""Summarise an `ncu --metrics gpu__time_duration.sum,dram__bytes_*.sum --csv`
launch list (development aid): per-kernel totals, then the launch sequence of
the bench's timed kernels.

Usage: python tools/launch_summary.py gpurun_out/<tag>/launches.csv > profiles/<round>/launches_summary.txt
"""
import csv
import io
import sys
from collections import OrderedDict

path = sys.argv[1]
lines = [ln for ln in open(path) if ln.startswith('"')]
rows = list(csv.reader(io.StringIO("".join(lines))))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
launch = OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))


def short(name):
    return name.split("(")[0][:56]


tot = OrderedDict()
for d in launch.values():
    k = short(d["name"])
    t = tot.setdefault(k, [0, 0.0, 0.0])
    t[0] += 1
    t[1] += d.get("gpu__time_duration.sum", 0.0) / 1e3
    t[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
print("# cold-cache, serialised per launch (ncu --clock-control none): compare shares, not absolutes")
print(f"{'kernel':58s} {'launches':>8s} {'total_us':>12s} {'dram_bytes':>12s}")
for k, (c, us, b) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:58s} {c:8d} {us:12.1f} {b:12.4e}")
print("\n# expand / count launches in order (the bench's timed kernels are the ~3.1 GB ones)")
for d in launch.values():
    if "expand_tma" in d["name"] or "::count_kernel" in d["name"]:
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        print(f"{short(d['name']):44s} {d.get('gpu__time_duration.sum', 0.0) / 1e3:9.1f} us  {b:.4e} B")
