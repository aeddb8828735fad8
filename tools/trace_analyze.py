"""Summarise a tile-kernel phase trace (build with -DTK_TRACE, run with TK_TRACE_FILE=path).

Slots per block (clock64 of thread 0 / warp 0): 0 start (smid in bits 48+), 1 count published,
2 stage ready (mbarrier), 3 prefix known, 4 after the w barrier, 5 after the classification barrier,
6 warp 0 done with list folds, 7 spill done (0 if none).
"""
import sys
import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 8)
lag = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mask = np.uint64((1 << 48) - 1)
smid = (a[:, 0] >> np.uint64(48)).astype(np.int64)
t = (a & mask).astype(np.int64)
start = t[:, 0]
blk = np.arange(len(a))
fold = (blk >= lag + 1) & (t[:, 6] > 0)
f = t[fold]
s0 = f[:, 0]
end = np.maximum(f[:, 6], f[:, 7])
mhz = 1965.0
def us(x):
    return x / mhz
def show(name, d):
    d = us(d.astype(np.float64))
    print(f"{name:28s} mean {d.mean():7.3f} us  p50 {np.percentile(d, 50):7.3f}  p90 {np.percentile(d, 90):7.3f}  p99 {np.percentile(d, 99):7.3f}")
print(f"blocks {len(a)}, fold blocks traced {fold.sum()}, spills {(f[:, 7] > 0).sum()}")
cnt = t[(blk >= 1) & (t[:, 1] > 0)]
show("count (start->published)", cnt[:, 1] - cnt[:, 0])
show("stage ready (start->mbar)", f[:, 2] - s0)
show("prefix known (mbar->pref)", f[:, 3] - f[:, 2])
show("w barrier (mbar->w)", f[:, 4] - f[:, 2])
show("classify (w->cls barrier)", f[:, 5] - f[:, 4])
show("list folds (cls->warp0)", f[:, 6] - f[:, 5])
sp = f[f[:, 7] > 0]
show("spill (warp0->spill end)", sp[:, 7] - sp[:, 6])
show("fold-block life", end - s0)
# per-SM occupancy: summed CTA lifetimes over the SM's active span
allend = np.maximum.reduce([t[:, i] for i in range(1, 8)])
life = np.where(allend > 0, allend - start, 0)
occ = []
for sm in np.unique(smid):
    m = smid == sm
    span = allend[m].max() - start[m].min()
    occ.append(life[m].sum() / span)
print(f"resident CTAs per SM (time-averaged): mean {np.mean(occ):.2f}  min {np.min(occ):.2f}  max {np.max(occ):.2f}")
tot = us((allend.max() - start[start > 0].min()))
print(f"kernel span (SM clocks, unsynchronised across SMs): ~{tot:.0f} us")
