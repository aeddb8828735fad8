"""Turn a GPU-box evidence bundle (tools/profile_round.sh <tag>) into the tracked files in profiles/.

  python tools/make_profiles.py <tag>      (reads gpurun_out/<tag>_*)
"""
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
g = lambda name: os.path.join(REPO, "gpurun_out", f"{tag}_{name}")
prof = os.path.join(REPO, "profiles")


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=REPO).stdout


# 1. launch list of the bench command (cold-cache, serialised)
lines = [l for l in open(g("launches.csv")) if not l.startswith("==")]
rows = list(csv.reader(io.StringIO("".join(lines))))
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
launches = []
for r in rows[1:]:
    if len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        us = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[r[ui]]
        launches.append((us, r[ki]))
with open(os.path.join(prof, f"{tag}_launches_bench_cfg5.csv"), "w") as f:
    f.writelines(lines)
tile = [u for u, k in launches if "ttv_tile_kernel" in k]
with open(os.path.join(prof, f"{tag}_launches_bench_cfg5.txt"), "w") as f:
    f.write("ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv\n")
    f.write("  python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu   (cold-cache, serialised launches)\n")
    f.write(f"{len(launches)} launches; ttv_tile_kernel launches: {len(tile)}, mean {sum(tile) / max(1, len(tile)):.1f} us\n")
    steps = [u for u, k in launches]
    f.write("Launches in order:\n")
    for u, k in launches:
        f.write(f"  {u:12.1f} us  {k[:110]}\n")
# 2. full capture summary + traffic
rep = g("tile.ncu-rep")
summ = run([sys.executable, "tools/ncu_summary.py", rep, "20"])
lines_ = run([sys.executable, "tools/ncu_lines.py", rep, "25"])
insts = run([sys.executable, "tools/ncu_insts.py", rep, "25", "tk_"])
with open(os.path.join(prof, f"{tag}_ncu_cfg5_tile.txt"), "w") as f:
    f.write(f"ncu --set full --import-source on --clock-control none -k regex:ttv_tile -s 1 -c 1\n"
            f"  python tools/prof_ttv.py --what cfg5 --nnz 400000000 --iters 2\n\n")
    f.write(summ + "\n== top source lines by warp-stall samples ==\n" + lines_ +
            "\n== top source lines by executed warp instructions ==\n" + insts)
raw = run(["ncu", "-i", rep, "--page", "raw", "--csv"])
rr = list(csv.reader(raw.splitlines()))
d = dict(zip(rr[0], rr[2]))
units = dict(zip(rr[0], rr[1]))
def gb(k):
    v = float(d[k])
    return v * {"Gbyte": 1e9, "GB": 1e9, "Mbyte": 1e6, "MB": 1e6, "Kbyte": 1e3, "KB": 1e3, "byte": 1, "B": 1}[units[k]]
ms = float(d["gpu__time_duration.sum"]) * {"msecond": 1, "ms": 1, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}[units["gpu__time_duration.sum"]]
kname = "ttv_tile_kernel<Raw,2,768,32>"
json.dump({"kernel": kname, "nnz": 400000000, "workload": "cfg5 (4e8 nnz Zipf, mode 2)",
           "dram_bytes_read": gb("dram__bytes_read.sum"), "dram_bytes_write": gb("dram__bytes_write.sum"),
           "dram_bytes_per_launch": gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"),
           "gpu_time_ms": ms,
           "source": f"ncu --set full --clock-control none (profiles/{tag}_ncu_cfg5_tile.txt); one launch"},
          open(os.path.join(prof, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(prof, "ncu_traffic.json")).read())
