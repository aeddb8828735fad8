"""PCIe probe: pinned H2D on one and two streams, and H2D + D2H together (GPU box)."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); a = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    torch.cuda.synchronize(); b = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); c = time.perf_counter() - t
    print(f"1 stream H2D {n/a/1e9:.1f} GB/s; 2 streams H2D {2*n/b/1e9:.1f} GB/s; H2D+D2H {2*n/c/1e9:.1f} GB/s")
