"""Config-3 TTV kernel time (L2 flushed between iterations, as bench.py's secondary) -- GPU box.
TK_TILE_LAG_RT=<tiles> overrides the count-to-fold lag."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_01495_b200 import _lib, synth
from paper_2510_01495_b200.device import DeviceCoo
lib = _lib.load()
ops = synth.host_operands(3)
t3 = ops["tensor"]
dt = DeviceCoo.from_host(t3.subs, t3.vals, t3.shape)
x3 = torch.from_numpy(ops["x"]).cuda()
o_s = torch.empty((t3.nnz, 2), dtype=torch.int64, device="cuda")
o_v = torch.empty(t3.nnz, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty((), dtype=torch.float64, device="cuda")
ts = []
for i in range(42):
    torch.cuda.synchronize()
    flush.zero_(); sink.copy_(flush.sum())
    u = dt.ttv(x3, 2, o_s, o_v)[0]
    if i >= 2:
        ts.append(lib.tk_last_kernel_ms())
print(f"lag {os.environ.get('TK_TILE_LAG_RT', 'default')}: cfg3 kernel {np.median(ts) * 1e3:.2f} us (min {min(ts) * 1e3:.2f}), u={u}")
