"""Config-1 dot and config-2 matvec, a few calls each with a 256 MB L2 flush between (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2510_01495_b200 import synth  # noqa: E402
from paper_2510_01495_b200 import device as dv  # noqa: E402

if __name__ == "__main__":
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
    ops = synth.host_operands(1)
    x, y = torch.from_numpy(ops["x"]).cuda(), torch.from_numpy(ops["y"]).cuda()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    ops2 = synth.host_operands(2)
    a, xv = torch.from_numpy(ops2["a"]).cuda(), torch.from_numpy(ops2["x"]).cuda()
    yv = torch.empty(4096, dtype=torch.float64, device="cuda")
    for _ in range(3):
        flush.zero_()
        dv.dot(x, y, out)
        flush.zero_()
        dv.matvec(a, xv, yv)
    torch.cuda.synchronize()
    print("ok", float(out))
