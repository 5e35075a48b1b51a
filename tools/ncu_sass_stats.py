"""Per-instruction SASS stats of one kernel in an .ncu-rep (development aid):
total warp instructions, grouping by execution count, top stall sites and
stall-reason totals.  usage: ncu_sass_stats.py REP [unit_count]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
unit = int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, rows = r[1], r[2:]
ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[ie] or 0) for x in rows)
print("warp instructions", tot, (f"per unit {tot / unit:.1f}" if unit else ""))
c, cs = collections.Counter(), collections.Counter()
for x in rows:
    c[int(x[ie] or 0)] += int(x[ie] or 0)
    cs[int(x[ie] or 0)] += int(x[st] or 0)
for k, v in sorted(c.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  count {k}: {v} instr" + (f" ({v / unit:.1f}/unit)" if unit else "") + f", stall samples {cs[k]}")
cols = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
tots = {x: sum(int(y[h.index(x)] or 0) for y in rows) for x in cols}
print("stalls:", sorted(((k, v) for k, v in tots.items() if v), key=lambda kv: -kv[1]))
for x in sorted(rows, key=lambda x: -int(x[st] or 0))[:12]:
    print("  ", x[0][-5:], x[1][:64].ljust(64), x[ie], x[st])
