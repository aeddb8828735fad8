"""Per-CUDA-source-line warp-stall attribution from an ncu report (cuda,sass view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, agg = None, None, {}
for r in rows:
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
    k = "Warp Stall Sampling (All Samples)"
    try:
        v = float(d[k] or 0)
    except ValueError:
        continue
    stalls = {c: float(d[c] or 0) for c in hdr if c.startswith("stall_") and "Not Issued" not in c and d[c] not in ("", "-")}
    key = (fname, int(r[0]))
    a = agg.setdefault(key, [0.0, r[1].strip(), {}])
    a[0] += v
    for c, x in stalls.items():
        a[2][c] = a[2].get(c, 0) + x
tot = sum(a[0] for a in agg.values()) or 1
for (f, ln), (v, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    t2 = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{v / tot * 100:5.1f}% {f}:{ln:<4} {src[:70]:70s} " + " ".join(f"{c[6:]}={int(x)}" for c, x in t2))
