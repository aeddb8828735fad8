"""Cold-read floor after a 256 MB L2 flush: torch reductions vs the library dot (GPU box)."""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2510_01495_b200 import device as dv, _lib
lib=_lib.load()
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty((), dtype=torch.float64, device="cuda")
x = torch.rand(10**6, dtype=torch.float64, device="cuda"); y = torch.rand(10**6, dtype=torch.float64, device="cuda")
big = torch.rand(16*10**6, dtype=torch.float64, device="cuda")
out = torch.empty(1, dtype=torch.float64, device="cuda")
def t(fn, n=10):
    ts=[]
    for i in range(n+2):
        torch.cuda.synchronize(); flush.zero_(); sink.copy_(flush.sum())
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        if i>=2: ts.append(e0.elapsed_time(e1))
    ts.sort(); return ts[len(ts)//2]
print("empty", t(lambda: None))
print("torch.dot 1e6", t(lambda: torch.dot(x,y)))
print("x.sum 1e6", t(lambda: x.sum()))
print("ours dot 1e6", t(lambda: dv.dot(x,y,out)))
print("big.sum 16e6 (128MB)", t(lambda: big.sum()))
print("ours dot 8e6x2 (128MB)", t(lambda: dv.dot(big[:8*10**6], big[8*10**6:], out)))
