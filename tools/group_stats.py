"""Group-size statistics of the config-5 stream (kept key = (i0, i1)) on the GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_01495_b200.device import DeviceCoo
nnz = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000_000
shape = (10**6, 10**5, 10**4)
t = DeviceCoo.generate(shape, nnz, zipf_s=1.2, normal_vals=True, seed=12345)
key = t.cols[0] * shape[1] + t.cols[1]
_, counts = torch.unique_consecutive(key, return_counts=True)
c = counts.double()
print(f"nnz={nnz} groups={counts.numel()} mean={c.mean():.2f} max={int(counts.max())}")
for th in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 768, 1024, 4096):
    m = counts > th
    print(f"  groups > {th:5d}: {int(m.sum()):10d}  rows in them: {float(c[m].sum())/nnz*100:6.2f}%")
tile = int(sys.argv[2]) if len(sys.argv) > 2 else 768
starts = torch.cumsum(counts, 0) - counts
ends = starts + counts
span = (starts // tile) != ((ends - 1) // tile)
print(f"  groups crossing a {tile}-row tile edge: {int(span.sum())} rows: {float(c[span].sum())/nnz*100:.2f}%")
# rows a tile's open group holds past its stage (tile + halo): what a second-pass chain kernel would re-read
halo = int(sys.argv[3]) if len(sys.argv) > 3 else 32
stage_end = (starts // tile + 1) * tile + halo
past = torch.clamp(ends - stage_end, min=0)
m = past > 0
print(f"  open groups past a {tile}+{halo} stage: {int(m.sum())}  rows past the stage: {float(past.sum())/nnz*100:.2f}%  "
      f"in-stage rows of those groups: {float((c[m]-past[m].double()).sum())/nnz*100:.2f}%")
for th in (64, 128, 256, 512):
    big = counts > th
    print(f"  groups > {th} rows: {int(big.sum())}, rows {float(c[big].sum())/nnz*100:.2f}%")
