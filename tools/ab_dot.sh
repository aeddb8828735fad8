#!/bin/bash
# On the GPU box: config-1 dot and config-2 matvec kernel times (bench secondary protocol) per variants/*.so.
cd "$(dirname "$0")/.."
cp paper_2510_01495_b200/libtk_b200.so /tmp/tk_keep.so
for v in variants/*.so; do
  cp "$v" paper_2510_01495_b200/libtk_b200.so
  timeout 300 python - <<PY 2>/dev/null
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_01495_b200 import _lib, synth, device as dv
lib = _lib.load()
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda"); sink = torch.empty((), dtype=torch.float64, device="cuda")
ops = synth.host_operands(1)
x, y = torch.from_numpy(ops["x"]).cuda(), torch.from_numpy(ops["y"]).cuda(); out = torch.empty(1, dtype=torch.float64, device="cuda")
ts = []
for i in range(30):
    torch.cuda.synchronize(); flush.zero_(); sink.copy_(flush.sum()); dv.dot(x, y, out)
    if i >= 5: ts.append(lib.tk_last_kernel_ms())
ops2 = synth.host_operands(2)
a, xv = torch.from_numpy(ops2["a"]).cuda(), torch.from_numpy(ops2["x"]).cuda(); yv = torch.empty(4096, dtype=torch.float64, device="cuda")
tm = []
for i in range(30):
    torch.cuda.synchronize(); flush.zero_(); sink.copy_(flush.sum()); dv.matvec(a, xv, yv)
    if i >= 5: tm.append(lib.tk_last_kernel_ms())
print("$(basename $v .so)", round(float(np.median(ts)) * 1e3, 2), "us dot", round(float(np.median(tm)) * 1e3, 2), "us matvec")
PY
done
cp /tmp/tk_keep.so paper_2510_01495_b200/libtk_b200.so
