"""Time sparse MTTKRP on a config-4-shaped tensor (4-way 20000^4, mode 0) for ranks given on
the command line; CUDA events inside the library, 256 MB L2 flush between iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_01495_b200 import _lib
from paper_2510_01495_b200.device import DeviceCoo

torch.cuda.set_device(0)
lib = _lib.load()
nnz = int(os.environ.get("TK_MT_NNZ", 100_000_000))
shape = (20000,) * 4
t = DeviceCoo.generate(shape, nnz, seed=4444)
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
for R in [int(a) for a in sys.argv[1:]] or [16, 32]:
    g = torch.Generator(device="cuda").manual_seed(R)
    fac = {m: torch.rand((shape[m], R), dtype=torch.float64, device="cuda", generator=g) for m in (1, 2, 3)}
    out = torch.empty((shape[0], R), dtype=torch.float64, device="cuda")
    ts = []
    for i in range(7):
        flush.zero_()
        torch.cuda.synchronize()
        t.mttkrp(fac, 0, out)
        if i >= 2:
            ts.append(lib.tk_last_kernel_ms())
    ms = float(np.median(ts))
    stream_b = nnz * 40 + 3 * 20000 * R * 8 + 20000 * R * 8
    print(f"R={R} {ms:.3f} ms  {nnz / ms / 1e6:.1f} Mnnz/ms  stream {stream_b / ms / 1e6:.0f} GB/s  "
          f"gathered {nnz * 3 * R * 8 / ms / 1e6:.0f} GB/s  checksum {float(out.sum()):.10e}")
