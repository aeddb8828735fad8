"""Config-3 (1e6 rows) and config-5 (4e8) tile-kernel time vs the count-to-fold lag
(TK_TILE_LAG_RT), kernel events under the bench's L2 flush (GPU box)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_01495_b200 import _lib, synth  # noqa: E402
from paper_2510_01495_b200.device import DeviceCoo, uniform_vector  # noqa: E402

lib = _lib.load()
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty((), dtype=torch.float64, device="cuda")


def kms(fn, n=12):
    ts = []
    for i in range(n):
        torch.cuda.synchronize()
        flush.zero_()
        sink.copy_(flush.sum())
        fn()
        if i >= 2:
            ts.append(lib.tk_last_kernel_ms())
    return float(np.median(ts))


ops = synth.host_operands(3)
t3 = ops["tensor"]
d3 = DeviceCoo.from_host(t3.subs, t3.vals, t3.shape)
x3 = torch.from_numpy(ops["x"]).cuda()
big = DeviceCoo.generate((10**6, 10**5, 10**4), 400_000_000, zipf_s=1.2, normal_vals=True, seed=12345)
x5 = uniform_vector(10**4, 777)
o5s = torch.empty((big.nnz, 2), dtype=torch.int64, device="cuda")
o5v = torch.empty(big.nnz, dtype=torch.float64, device="cuda")
for lag in (16, 32, 64, 128, 256, 512, 1024):
    os.environ["TK_TILE_LAG_RT"] = str(lag)
    a = kms(lambda: d3.ttv(x3, 2))
    b = kms(lambda: big.ttv(x5, 2, o5s, o5v), n=6)
    print(f"lag {lag:5d}: cfg3 {a * 1e3:7.2f} us   cfg5 {b:6.3f} ms", flush=True)
