"""One uniform class-M tensor (60K-row segments) through the middle-mode path, for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
shape, nnz = (1000, 100000, 10000), 60_000_000
t = DeviceCoo.generate(shape, nnz, zipf_s=0.0, normal_vals=True, seed=7)
x = uniform_vector(shape[1], 3)
os_ = torch.empty((nnz, 2), dtype=torch.int64, device="cuda")
ov = torch.empty(nnz, dtype=torch.float64, device="cuda")
for i in range(3):
    u = t.ttv(x, 1, os_, ov)[0]
torch.cuda.synchronize()
print(u)
