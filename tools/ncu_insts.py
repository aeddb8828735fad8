"""Per-CUDA-source-line executed-instruction counts from an ncu report (cuda,sass view).

  python tools/ncu_insts.py report.ncu-rep [top] [file-filter]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ffilt = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    d = dict(zip(hdr, r))
    try:
        ins = float(d["Instructions Executed"] or 0)
        smp = float(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    a = agg.setdefault((fname, int(r[0])), [0.0, 0.0, r[1].strip()])
    a[0] += ins
    a[1] += smp
tot_i = sum(a[0] for a in agg.values()) or 1
tot_s = sum(a[1] for a in agg.values()) or 1
print(f"total warp instructions {tot_i:.4g}")
items = [kv for kv in agg.items() if ffilt in kv[0][0]]
for (f, ln), (i, s, src) in sorted(items, key=lambda kv: -kv[1][0])[:top]:
    print(f"{i / tot_i * 100:5.1f}% ins {s / tot_s * 100:5.1f}% smp {f}:{ln:<4} {src[:80]}")
