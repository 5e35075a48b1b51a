"""Warp-stall samples per CUDA source line of one kernel in an .ncu-rep
(development aid).  usage: ncu_lines.py REP [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
agg, ex, text, reasons = collections.Counter(), collections.Counter(), {}, collections.defaultdict(collections.Counter)
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        rs = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or not r[0].isdigit():
        continue
    try:
        v, e = int(r[si] or 0), int(r[ie] or 0)
    except ValueError:
        continue
    k = (cur, int(r[0]))
    agg[k] += v
    ex[k] += e
    text[k] = r[1].strip()[:70]
    for i, c in rs:
        reasons[k][c[6:]] += int(r[i] or 0)
tot = sum(agg.values()) or 1
print(f"stall samples {tot}, warp instructions {sum(ex.values())}")
for k, v in agg.most_common(top):
    rr = ", ".join(f"{c} {n / max(v, 1) * 100:.0f}%" for c, n in reasons[k].most_common(2) if n)
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]:<4} exec {ex[k]:>10}  {text[k]:70s} [{rr}]")
