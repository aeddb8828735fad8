"""Per-CUDA-source-line L1 traffic from an ncu report: shared-memory wavefronts (and the excess over
ideal = bank conflicts), global L1 tag requests and L2 sectors.  python tools/ncu_mem.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, {}
cols = ["L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "L1 Tag Requests Global", "L2 Theoretical Sectors Global",
        "Instructions Executed"]
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
    key = (fname, r[0], r[1].strip()[:60])
    a = agg.setdefault(key, [0.0] * len(cols))
    for i, c in enumerate(cols):
        try:
            a[i] += float(d.get(c) or 0)
        except ValueError:
            pass
tot = [sum(a[i] for a in agg.values()) for i in range(len(cols))]
print("totals:", {c: f"{t:.3e}" for c, t in zip(cols, tot)})
score = lambda a: a[0] + a[2]
for k, a in sorted(agg.items(), key=lambda kv: -score(kv[1]))[:top]:
    print(f"smem_wf {a[0]:.2e} (excess {a[1]:.2e})  gtag {a[2]:.2e}  l2sec {a[3]:.2e}  ins {a[4]:.2e}  {k[0]}:{k[1]} {k[2]}")
