"""Summarise an ncu report: key SOL metrics + top SASS instructions by warp-stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(det.splitlines()))
h = r[0]
want = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate',
        'Achieved Active Warps Per SM', 'Grid Size', 'Block Size', 'Registers Per Thread', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Issued Ipc Active', 'Dynamic Shared Memory Per Block', 'Block Limit Shared Mem',
        'Executed Instructions']
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in want:
        print(d['Metric Name'].ljust(40), d['Metric Value'], d['Metric Unit'])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
for row in rr[2:3]:
    d = dict(zip(hh, row))
    for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum', 'lts__t_bytes.sum'):
        if k in d:
            print(k.ljust(40), d[k], rr[1][hh.index(k)])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
data = rows[2:]
k = h.index('Warp Stall Sampling (All Samples)')
tot = sum(float(x[k] or 0) for x in data)
idx = sorted(range(len(data)), key=lambda i: -float(data[i][k] or 0))
stall_cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
for i in idx[:top]:
    x = data[i]
    d = dict(zip(h, x))
    t2 = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{float(x[k]) / tot * 100:5.1f}% #{i:4d} {x[1].strip()[:56]:56s} thr={d['Avg. Threads Executed']:>5} "
          f"{t2[0][1]}={int(t2[0][0])} {t2[1][1]}={int(t2[1][0])}")
