"""Dump SASS with per-instruction execution counts (normalised per CTA) and stall samples.

  python tools/ncu_sass.py report.ncu-rep [ctas] > sass.txt
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
ctas = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
hdr = None
for i, r in enumerate(csv.reader(out.splitlines())):
    if r and r[0] == "Address":
        hdr = r
        idx = 0
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    ins = float(d["Instructions Executed"] or 0) / ctas
    smp = int(float(d["Warp Stall Sampling (All Samples)"] or 0))
    thr = d["Avg. Threads Executed"]
    print(f"{idx:5d} {ins:9.3f} {smp:6d} {thr:>3} {d['Source'].strip()}")
    idx += 1
