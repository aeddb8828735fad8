"""Config-5 tensor, contracted mode 1 (the paper's protocol): whole-call device time of the
general path (CUDA events), default (segmented counting, tk_midmode.cu) and TK_MID_MODE=0 (the
CUB split-sort path) -- run on the GPU box: python tools/time_mode1.py [nnz]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2510_01495_b200 import _lib  # noqa: E402
from paper_2510_01495_b200.device import DeviceCoo, uniform_vector  # noqa: E402

nnz = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000_000
shape = (10**6, 10**5, 10**4)
t = DeviceCoo.generate(shape, nnz, zipf_s=1.2, normal_vals=True, seed=12345)
x = uniform_vector(shape[1], 778)
os_ = torch.empty((nnz, 2), dtype=torch.int64, device="cuda")
ov = torch.empty(nnz, dtype=torch.float64, device="cuda")
res = {}
only = os.environ.get("TK_MID_ONLY") == "1"  # skip the CUB comparison (profiling runs)
same = None
for mode in (("1",) if only else ("1", "0")):
    os.environ["TK_MID_MODE"] = mode
    ts = []
    l0 = _lib.load().tk_launch_count()
    for i in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        u = t.ttv(x, 1, os_, ov)[0]
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    res[mode] = (float(np.median(ts)), u, (_lib.load().tk_launch_count() - l0) / 6)
    if mode == "1":
        ref = (os_[:u].clone(), ov[:u].clone())
    else:
        same = torch.equal(ref[0], os_[:u]) and torch.equal(ref[1].view(torch.int64), ov[:u].view(torch.int64))
b = nnz * 32 + 8 * shape[1] + res["1"][1] * 24
print(f"counting path: {res['1'][0]:.3f} ms ({b / res['1'][0] / 1e6:.0f} GB/s alg, {res['1'][2]:.0f} launches), "
      + (f"u={res['1'][1]}" if only else f"CUB split path: {res['0'][0]:.3f} ms, u={res['1'][1]}, identical={same}"))
