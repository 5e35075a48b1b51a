"""Write a judged text summary of an .ncu-rep: headline metrics, DRAM bytes,
every details-page row, and the SASS instruction/stall statistics
(development aid).  usage: ncu_report.py REP > profiles/<round>/ncu_<name>.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
run = lambda *a: subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout  # noqa: E731
r = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = r[0]
ki, si, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                          "Metric Value"))
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hh = raw[0]
want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "Kernel Name")
cols = [i for i, c in enumerate(hh) if c in want]
print(f"# ncu --set full --clock-control none capture: {rep}")
for x in raw[2:]:
    print("raw:", ", ".join(f"{hh[i]}={x[i]} {raw[1][i]}".strip() for i in cols))
for x in r[1:]:
    print(f"{x[si]} | {x[mi]} = {x[vi]} {x[ui]}".rstrip())
