"""Time the config-4 dense multi-vector TTV (kernel + fix-up, CUDA events inside the library,
256 MB L2 flush between iterations); prints the median ms.  Used for A/B runs of variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_01495_b200 import _lib
from paper_2510_01495_b200.device import DeviceCoo, uniform_vector

torch.cuda.set_device(0)
lib = _lib.load()
shape = (20000,) * 4
t = DeviceCoo.generate(shape, 100_000_000, seed=4444)
vecs = {m: uniform_vector(shape[m], 40 + m) for m in (1, 2, 3)}
out = torch.empty(shape[0], dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
ts = []
for i in range(12):
    flush.zero_()
    torch.cuda.synchronize()
    t.ttv_dense(vecs, 0, out)
    if i >= 2:
        ts.append(lib.tk_last_kernel_ms())
print(f"{sys.argv[1] if len(sys.argv) > 1 else 'cur'} {np.median(ts):.4f} ms  min {min(ts):.4f}  sum {float(out.sum()):.12e}")
