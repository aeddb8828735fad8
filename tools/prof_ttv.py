"""Minimal driver for ncu captures of the hot kernels (no timing, no JSON).

  python tools/prof_ttv.py --what cfg5 --nnz 100000000 --iters 3
  python tools/prof_ttv.py --what cfg4 --nnz 100000000
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="cfg5", choices=["cfg5", "cfg5k1", "cfg4", "cfg3", "dot", "matvec"])
    ap.add_argument("--nnz", type=int, default=100_000_000)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    import torch
    from paper_2510_01495_b200 import device as dv
    from paper_2510_01495_b200 import synth
    from paper_2510_01495_b200.device import DeviceCoo, uniform_vector
    torch.cuda.set_device(0)
    if a.what == "cfg5k1":  # the middle mode: the general (sort) path
        shape = (10**6, 10**5, 10**4)
        t = DeviceCoo.generate(shape, a.nnz, zipf_s=1.2, normal_vals=True, seed=12345)
        x = uniform_vector(shape[1], 778)
        os_ = torch.empty((t.nnz, 2), dtype=torch.int64, device="cuda")
        ov = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
        for _ in range(a.iters):
            u, _, _ = t.ttv(x, 1, os_, ov)
        print("cfg5k1 u", u)
    elif a.what == "cfg5":
        shape = (10**6, 10**5, 10**4)
        t = DeviceCoo.generate(shape, a.nnz, zipf_s=1.2, normal_vals=True, seed=12345)
        x = uniform_vector(shape[2], 777)
        os_ = torch.empty((t.nnz, 2), dtype=torch.int64, device="cuda")
        ov = torch.empty(t.nnz, dtype=torch.float64, device="cuda")
        for _ in range(a.iters):
            u, _, _ = t.ttv(x, 2, os_, ov)
        print("cfg5 u", u)
    elif a.what == "cfg4":
        shape = (20000,) * 4
        t = DeviceCoo.generate(shape, a.nnz, seed=4444)
        vecs = {m: uniform_vector(shape[m], 40 + m) for m in (1, 2, 3)}
        out = torch.empty(shape[0], dtype=torch.float64, device="cuda")
        for _ in range(a.iters):
            t.ttv_dense(vecs, 0, out)
        print("cfg4 sum", float(out.sum()))
    elif a.what == "cfg3":
        ops = synth.host_operands(3)
        t3 = ops["tensor"]
        t = DeviceCoo.from_host(t3.subs, t3.vals, t3.shape)
        x = torch.from_numpy(ops["x"]).cuda()
        for _ in range(a.iters):
            u, _, _ = t.ttv(x, 2)
        print("cfg3 u", u)
    elif a.what == "dot":
        ops = synth.host_operands(1)
        x, y = torch.from_numpy(ops["x"]).cuda(), torch.from_numpy(ops["y"]).cuda()
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        for _ in range(a.iters):
            dv.dot(x, y, out)
        print("dot", float(out.item()))
    else:
        ops = synth.host_operands(2)
        A, x = torch.from_numpy(ops["a"]).cuda(), torch.from_numpy(ops["x"]).cuda()
        y = torch.empty(4096, dtype=torch.float64, device="cuda")
        for _ in range(a.iters):
            dv.matvec(A, x, y)
        print("matvec", float(y.sum()))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
