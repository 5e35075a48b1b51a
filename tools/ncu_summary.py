"""Summarise an .ncu-rep: key metrics per kernel (development aid)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, mi, ui, vi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Unit'), h.index('Metric Value')
idi = h.index('ID')
want = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Compute (SM) Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'SM Frequency', 'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block', 'L2 Hit Rate']
for x in r[1:]:
    if x[mi] in want:
        print(x[idi], x[ki][:44], '|', x[mi], x[vi], x[ui])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
cols = [i for i, c in enumerate(hh) if c in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'Kernel Name')]
for x in rr[2:]:
    print([hh[i] + '=' + x[i] for i in cols])
