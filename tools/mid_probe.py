"""Steady-state rate of the middle-mode kernels on uniform tensors whose segments all fall in one
class (GPU box): python tools/mid_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2510_01495_b200.device import DeviceCoo, uniform_vector

def run(shape, nnz, zipf, label):
    t = DeviceCoo.generate(shape, nnz, zipf_s=zipf, normal_vals=True, seed=7)
    x = uniform_vector(shape[1], 3)
    os_ = torch.empty((nnz, 2), dtype=torch.int64, device="cuda")
    ov = torch.empty(nnz, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); u = t.ttv(x, 1, os_, ov)[0]; e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts[1:]))
    print(f"{label}: {nnz/1e6:.0f}M rows, rows/segment {nnz/shape[0]:.0f}, u={u}: {ms:.3f} ms = {ms*1e9/nnz:.1f} ps/row")

run((1000, 100000, 10000), 60_000_000, 0.0, "class M, 60K-row segments, uniform S")
run((6000, 100000, 10000), 60_000_000, 0.0, "class M, 10K-row segments, uniform S")
run((30000, 100000, 10000), 60_000_000, 0.0, "class M, 2K-row segments, uniform S")
run((100000, 100000, 10000), 60_000_000, 0.0, "class M, 600-row segments, uniform S")
run((200000, 100000, 10000), 60_000_000, 0.0, "class A, 300-row segments, uniform S")
run((1000000, 100000, 10000), 60_000_000, 0.0, "class A, 60-row segments, uniform S")
run((60, 100000, 10000), 60_000_000, 0.0, "class B, 1M-row segments, uniform S")
run((1000, 100000, 64), 60_000_000, 0.0, "class M, 60K-row segments, R = 64 (long groups)")
