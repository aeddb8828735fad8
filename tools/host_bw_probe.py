"""Host-side probe (GPU box): pageable vs pinned H2D, and parallel host memcpy bandwidth."""
import ctypes, os, threading, time
import numpy as np
import torch

n = 1 << 30
src = np.ones(n // 8)
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
pt = torch.from_numpy(src.view(np.uint8))
for name, h in (("pageable", pt), ("pinned", pin)):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        dev.copy_(h, non_blocking=True); torch.cuda.synchronize()
        el = time.perf_counter() - t
    print(f"H2D {name}: {n / el / 1e9:.1f} GB/s")
dst = np.empty(n // 8)
dst[:] = 0
for T in (1, 4, 8, 16):
    parts = np.array_split(np.arange(n // 8), T)
    def work(i):
        p = parts[i]
        np.copyto(dst[p[0]:p[-1] + 1], src[p[0]:p[-1] + 1])
    for _ in range(2):
        th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
        t = time.perf_counter()
        [x.start() for x in th]; [x.join() for x in th]
        el = time.perf_counter() - t
    print(f"memcpy {T:2d} threads: {n / el / 1e9:.1f} GB/s (read+write {2 * n / el / 1e9:.1f})")
fresh = time.perf_counter(); a = np.empty(n // 8); a[:] = 1.0; el = time.perf_counter() - fresh
print(f"first-touch fill 1 thread: {n / el / 1e9:.1f} GB/s")
