"""First-call overhead of the GPU module at the BASELINE config-1..3 sizes.

  python tools/first_call.py [out.csv]      (runs on a GPU box; 5 fresh processes per row)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01495_b200 import overhead  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "first_call.csv"
rows = [overhead.estimate_overhead(size=10**6, experiment="dot", repeats=5),
        overhead.estimate_overhead(size=4096, experiment="matvec", repeats=5),
        overhead.estimate_overhead(size=1000, experiment="ttv", density=0.001, mode=3, repeats=5)]
overhead.write_overhead_csv(rows, out)
for r in rows:
    print(f"{r.size:32s} first {r.first_call_mean_s * 1e3:9.3f} ms  steady {r.steady_mean_s * 1e3:8.3f} ms  "
          f"overhead {r.overhead_s * 1e3:9.3f} ms  ({r.repeats} processes)")
