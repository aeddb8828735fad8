"""Config-5 tensor, contracted mode 1: segment (leading value) size classes and (i0, S) bucket sizes -- GPU box."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01495_b200.device import DeviceCoo
nnz = int(float(sys.argv[1])) if len(sys.argv) > 1 else 400_000_000
shape = (10**6, 10**5, 10**4)
t = DeviceCoo.generate(shape, nnz, zipf_s=1.2, normal_vals=True, seed=12345)
i0, i1, i2 = t.cols
_, seg = torch.unique_consecutive(i0, return_counts=True)
print(f"nnz={nnz} segments={seg.numel()} max={int(seg.max())}")
edges = [0, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 262144, 1 << 20, 1 << 22, 1 << 30]
for a, b in zip(edges[:-1], edges[1:]):
    m = (seg > a) & (seg <= b)
    print(f"  segments of {a+1:8d}..{b:10d} rows: {int(m.sum()):8d}  rows {float(seg[m].sum())/nnz*100:6.2f}%")
top = torch.sort(seg, descending=True).values[:12].tolist()
print("  largest segments:", top)
# runs of equal (i0, i1): rows per run
key01 = i0 * shape[1] + i1
_, runs = torch.unique_consecutive(key01, return_counts=True)
print(f"(i0,i1) runs: {runs.numel()} mean {nnz/runs.numel():.2f} max {int(runs.max())}")
del key01, runs
# buckets (i0, S)
key = i0 * shape[2] + i2
ks = torch.sort(key).values
del key
_, bc = torch.unique_consecutive(ks, return_counts=True)
del ks
print(f"buckets={bc.numel()} mean={nnz/bc.numel():.2f} max={int(bc.max())}")
for th in (1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 4096, 16384, 65536):
    m = bc > th
    print(f"  buckets > {th:6d} rows: {int(m.sum()):10d}  rows in them {float(bc[m].sum())/nnz*100:6.2f}%")
print("  largest buckets:", torch.sort(bc, descending=True).values[:16].tolist())
