"""Stall-reason totals and top stalled SASS lines for one kernel of an .ncu-rep."""
import csv, io, subprocess, sys
rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
isrc, ie = h.index('Source'), h.index('Instructions Executed')
cols = [i for i, c in enumerate(h) if c.startswith('stall_') and 'Not Issued' not in c]
data = [r for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot = {h[i]: sum(int(r[i] or 0) for r in data) for i in cols}
print('instr', sum(int(r[ie]) for r in data))
print(sorted(((v, k) for k, v in tot.items() if v), reverse=True))
iall = h.index('Warp Stall Sampling (All Samples)')
for r in sorted(data, key=lambda r: -int(r[iall] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
    top = sorted(((int(r[i] or 0), h[i][6:]) for i in cols), reverse=True)[:2]
    print(r[iall], r[ie], r[isrc][:70], top)
