"""Host-buffer C-ABI calls from pageable numpy arrays (the reference caller's case): dot at
config 1, matvec at config 2, ttv at config 3 -- median wall time of the drop-in kernel-module
call (GPU box)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_01495_b200 as tk  # noqa: E402
from paper_2510_01495_b200 import synth  # noqa: E402

K = tk.kernels()
res = {}
for cfg in (1, 2, 3):
    ts = []
    for trial in range(12):
        ops = synth.host_operands(cfg, schedule_index=trial)  # fresh operands, like the harness
        if cfg == 1:
            f = lambda: K.dot(ops["x"], ops["y"])
        elif cfg == 2:
            f = lambda: K.matvec(ops["a"], ops["x"])
        else:
            t = ops["tensor"]
            f = lambda: K.ttv_raw(t.subs, t.vals, t.shape, ops["x"], 2)
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    res[cfg] = float(np.median(ts[2:])) * 1e3
print({f"cfg{k}_ms": round(v, 3) for k, v in res.items()})
