// tk_ttv.cu -- sparse TTV orchestration (sparse result and dense multi-vector result).
//
// Paths:
//   fast    : contracted mode is the trailing mode of a canonical tensor -> the kept
//             tuples are already sorted; one fused streaming kernel (ttv_tile_kernel<Raw>).
//   general : any other mode / unsorted input -> w and a linearised kept key per row,
//             stable device radix sort of (key, w), then the same segmented kernel
//             (<LinKey>).  Garbage kept indices or keys wider than 62 bits: LSD radix
//             passes over the kept columns (signed int64) carrying a permutation, then
//             <KeysW>.  Both sorts are stable, so every group is folded in ascending
//             original-row order, exactly like the reference (pyx:229-295).
//   dense   : multi-vector TTV to a dense vector (BASELINE config 4): one streaming
//             kernel with a deterministic block-level segmented reduction and a tiny
//             ordered fix-up for runs that cross tiles; chained single-mode TTV otherwise.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "tk_host.h"
#include "tk_tile_kernel.cuh"
#include "tk_ttv_kernels.cuh"

namespace tk {

// ============================================================================================
// helper kernels
// ============================================================================================

struct KeepCols {
  const long long* col[kMaxKeep];
  long long dims[kMaxKeep];
};

__global__ void prep_linkey_kernel2(long long n, int nk, KeepCols kc, const long long* __restrict__ subk,
                                    const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                    long long* __restrict__ key, double* __restrict__ w, Counters* ctr) {
  unsigned int flags = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long idx = subk[r];
    double wr = 0.0;
    if (idx < 0 || idx >= nx) flags |= kFlagIndex;
    else wr = __dmul_rn(vals[r], __ldg(x + idx));
    long long lin = 0;
    for (int c = 0; c < nk; ++c) {
      const long long v = kc.col[c][r];
      if (v < 0 || v >= kc.dims[c]) flags |= kFlagKeptOob;
      lin = lin * kc.dims[c] + v;
    }
    key[r] = lin;
    w[r] = wr;
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

// ---- general path, split by the leading kept mode (canonical input, contracted mode != 0) ----
// Row offsets of every leading-mode value: off[v] = first row with col0 >= v (off[n0] = n).  Flags
// kFlagUnsorted if col0 decreases and kFlagKeptOob if it leaves [0, n0): the split is then off.
__global__ void lead_offsets_kernel(long long n, const long long* __restrict__ col0, long long n0,
                                    long long* __restrict__ off, Counters* ctr) {
  constexpr int U = 4;  // rows per thread per round, every load of the round in flight at once
  unsigned int flags = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long r0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; r0 <= n; r0 += U * stride) {
    long long prev[U], cur[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long r = r0 + u * stride;
      prev[u] = (r == 0 || r > n) ? -1 : __ldg(col0 + r - 1);
      cur[u] = r < n ? __ldg(col0 + r) : n0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long r = r0 + u * stride;
      if (r > n) break;
      if (r < n && (cur[u] < 0 || cur[u] >= n0)) {
        flags |= kFlagKeptOob;
        continue;
      }
      if (cur[u] < prev[u]) {
        flags |= kFlagUnsorted;
        continue;
      }
      for (long long v = prev[u] + 1; v <= cur[u] && v <= n0; ++v) off[v] = r;
    }
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

// Split parts: leading-mode interval [lo[j], lo[j+1]) sorted on its own with 32-bit keys.
constexpr int kMaxParts = 64;
struct PartTable {
  long long lo[kMaxParts + 1];  // leading-mode value where each part starts
  int nparts;
  unsigned long long in_b;      // bit j: part j's (key, w) go to the second buffers (odd digit-pass
                                // count, so the sorted w ends in the first one: no copy in widen)
};

// w = vals * x[subk] and the 32-bit part-local key (lead - lo[part]) * R + rest, where rest is the
// row-major linearisation of the other kept modes (R = product of their dims).
__global__ void prep_key32_kernel(long long n, int nk, KeepCols kc, const long long* __restrict__ subk,
                                  const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                  PartTable pt, unsigned int* __restrict__ key, double* __restrict__ w,
                                  unsigned int* __restrict__ key_b, double* __restrict__ w_b, Counters* ctr) {
  unsigned int flags = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long idx = subk[r];
    double wr = 0.0;
    if (idx < 0 || idx >= nx) flags |= kFlagIndex;
    else wr = __dmul_rn(vals[r], __ldg(x + idx));
    const long long lead = kc.col[0][r];
    int lo = 0, hi = pt.nparts - 1;  // the part holding `lead` (lead is in range: checked by the offsets)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pt.lo[mid] <= lead) lo = mid;
      else hi = mid - 1;
    }
    long long rest = 0, R = 1;
    for (int c = 1; c < nk; ++c) {
      const long long v = kc.col[c][r];
      if (v < 0 || v >= kc.dims[c]) flags |= kFlagKeptOob;
      rest = rest * kc.dims[c] + v;
      R *= kc.dims[c];
    }
    const bool b = (pt.in_b >> lo) & 1ull;
    (b ? key_b : key)[r] = (unsigned int)((lead - pt.lo[lo]) * R + rest);
    (b ? w_b : w)[r] = wr;
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

// Back to the global linear key (lin = base + key32) and the sorted w into the tile kernel's input.
__global__ void widen_part_kernel(long long n, const unsigned int* __restrict__ k32, const double* __restrict__ ws,
                                  long long base, long long* __restrict__ key, double* __restrict__ w) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    key[r] = base + (long long)k32[r];
    if (ws != w) w[r] = ws[r];
  }
}

__global__ void iota_kernel(long long n, long long* out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    out[r] = r;
}

__global__ void gather_i64_kernel(long long n, const long long* __restrict__ src, const long long* __restrict__ idx,
                                  long long* __restrict__ dst) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    dst[r] = src[idx[r]];
}

__global__ void gather_w_kernel(long long n, const long long* __restrict__ perm, const long long* __restrict__ subk,
                                const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                double* __restrict__ w, Counters* ctr) {
  unsigned int flags = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long o = perm[r];
    const long long idx = subk[o];
    double wr = 0.0;
    if (idx < 0 || idx >= nx) flags |= kFlagIndex;
    else wr = __dmul_rn(vals[o], __ldg(x + idx));
    w[r] = wr;
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

__global__ void aos_to_soa_kernel(long long n, int d, const long long* __restrict__ aos, long long* __restrict__ soa,
                                  long long pitch) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    for (int m = 0; m < d; ++m) soa[m * pitch + r] = __ldcs(aos + r * d + m);
}

// packed host rows (tk_hostio.cu RowPack) -> SoA columns
struct UnpackPlan {
  int d;
  int shift[kMaxOrder];
  unsigned long long mask[kMaxOrder];
};

__global__ void unpack_rows_kernel(long long n, UnpackPlan p, const unsigned long long* __restrict__ packed,
                                   long long* __restrict__ soa, long long pitch) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const unsigned long long w = __ldcs(packed + r);
    for (int m = 0; m < p.d; ++m) soa[m * pitch + r] = (long long)((w >> p.shift[m]) & p.mask[m]);
  }
}

// ---- zero-group compaction (runs only when some group summed to exactly 0.0) -----------------
constexpr int kCompItems = 8;
constexpr int kCompTile = 256 * kCompItems;

__global__ void nz_count_kernel(long long n, const double* __restrict__ v, long long* __restrict__ blk) {
  using Reduce = cub::BlockReduce<int, 256>;
  __shared__ typename Reduce::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kCompTile;
  int c = 0;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + threadIdx.x * kCompItems + i;
    if (e < n && v[e] != 0.0) ++c;
  }
  const int tot = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void scan_blocks_kernel(long long nblk, long long* __restrict__ blk) {
  // single block, exclusive scan in place (sequential chunks of 256)
  using Scan = cub::BlockScan<long long, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long off = 0; off < nblk; off += 256) {
    const long long i = off + threadIdx.x;
    long long v = i < nblk ? blk[i] : 0, ex, agg;
    Scan(tmp).ExclusiveSum(v, ex, agg);
    if (i < nblk) blk[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
}

__global__ void nz_scatter_kernel(long long n, int nk, const double* __restrict__ v, const long long* __restrict__ s,
                                  const long long* __restrict__ blk, double* __restrict__ v2, long long* __restrict__ s2) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kCompTile + threadIdx.x * kCompItems;
  int c = 0;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + i;
    if (e < n && v[e] != 0.0) ++c;
  }
  int ex;
  Scan(tmp).ExclusiveSum(c, ex);
  long long o = blk[blockIdx.x] + ex;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + i;
    if (e < n && v[e] != 0.0) {
      v2[o] = v[e];
      for (int q = 0; q < nk; ++q) s2[o * nk + q] = s[e * nk + q];
      ++o;
    }
  }
}

// ============================================================================================
// dense-result multi-vector kernel
// ============================================================================================

struct DenseParams {
  long long n;
  int d, keep;
  const long long* col[kMaxOrder];
  const double* vals;
  const double* vec[kMaxOrder];
  long long dims[kMaxOrder];
  double* out;                 // == outs[0]
  double* outs[kMaxPeers];     // every output copy: this GPU's vector and peers' (NVLink-mapped)
  int nout;
  long long key_lo, key_hi;    // keep-mode indices this call owns (stores outside are dropped)
  double* c_first;
  double* c_last;
  long long* c_lastkey;
  int* c_flags;
  Counters* ctr;
  int bulk_ok;
};

struct SegPair {
  int f;
  double v;
};
// (a then b): a run head in b restarts the sum; otherwise b continues a's run.
__device__ __forceinline__ SegPair seg_combine(SegPair a, SegPair b) {
  return {a.f | b.f, b.f ? b.v : __dadd_rn(a.v, b.v)};
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;  // identical in every lane (RN addition commutes)
}

// One finished output element, stored into every output copy (this GPU and its peers: the
// merge of the sharded dense result is these direct NVLink stores, no all-reduce).  Only the
// keep-mode indices this call owns are stored; a shard split at key changes owns its keys.
__device__ __forceinline__ void dense_store(const DenseParams& p, long long key, double v) {
  if (key < p.key_lo || key >= p.key_hi) return;
  for (int i = 0; i < p.nout; ++i) p.outs[i][key] = v;
}

// Zero the owned range [lo, hi) of every output copy (keys without rows stay 0).
struct PeerOuts {
  double* p[kMaxPeers];
  int n;
};
__global__ void zero_range_kernel(PeerOuts o, long long lo, long long hi) {
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi; i += (long long)gridDim.x * blockDim.x)
    for (int c = 0; c < o.n; ++c) o.p[c][i] = 0.0;
}
// Copy [lo, hi) of src into every output copy (the chained fallback computes into src).
__global__ void bcast_range_kernel(const double* __restrict__ src, PeerOuts o, long long lo, long long hi) {
  for (long long i = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < hi; i += (long long)gridDim.x * blockDim.x) {
    const double v = src[i];
    for (int c = 0; c < o.n; ++c) o.p[c][i] = v;
  }
}

#ifndef TK_DENSE_SPAN
#define TK_DENSE_SPAN 3072  // rows per warp span (config 4: 2048 0.868 ms, 3072 0.832, 3584 0.830, 4096 0.884)
#endif
#ifndef TK_DENSE_U
#define TK_DENSE_U 1
#endif
#ifndef TK_DENSE_MINB
#define TK_DENSE_MINB 2
#endif
constexpr int kDenseSpan = TK_DENSE_SPAN;  // rows per warp span (carry unit of the fix-up)
constexpr int kDenseThreads = 256;
#ifndef TK_DENSE_SV_THREADS
#define TK_DENSE_SV_THREADS 512
#endif
#ifndef TK_DENSE_SV_MAX
#define TK_DENSE_SV_MAX (192 * 1024)  // largest staged vector (bytes); the rest of L1 caches the others
#endif
constexpr int kDenseSvThreads = TK_DENSE_SV_THREADS;
constexpr int kDenseU = TK_DENSE_U;        // 64-row sub-blocks per warp step

// Dense-result multi-vector TTV over a stream sorted by the kept mode (mode 0).
//
// One warp per span of kDenseSpan consecutive rows.  A warp step covers 64*kDenseU rows as
// 64-row sub-blocks; lane l holds rows 2l and 2l+1 of a sub-block (16-byte loads of every
// column), gathers the contracted vectors for both rows and forms
// w = ((val * x_{d-1}) * ...) * x_1, the chained-TTV association (descending modes).  Runs of
// equal keys are long (config 4: ~5000 rows), so a sub-block without a head just adds into
// per-lane accumulators; a sub-block with a head takes the slow path: the lane accumulators are
// reduced (butterfly), a segmented warp scan over the 64 rows closes every run ending in it, and
// the run left open restarts the accumulators.  A run closed inside its span is stored straight
// to out[key]; the span's leading piece (before its first head) and trailing open piece go to
// per-span carries that dense_fixup_kernel folds in span order -- every output element has
// exactly one writer, so the result is deterministic.
template <int D, int U>
struct DenseStep {
  static constexpr int DG = D > 1 ? D : 2;  // D == 0 (any order): indices re-read per row, no batching
  long long ka[U], kb[U];
  double wa[U], wb[U];
  long long ia[U][DG], ib[U][DG];
  bool oka[U], okb[U];
};

template <int D, bool V2, int U>
__device__ __forceinline__ void dense_load_step(const DenseParams& p, long long r, long long s1,
                                                DenseStep<D, U>& s) {
  const int lane = threadIdx.x & 31;
  const long long* __restrict__ kcol = p.col[0];
#pragma unroll
  for (int u = 0; u < U; ++u) {  // every column load of the step in flight at once
    const long long a = r + 64 * u + 2 * lane;
    s.oka[u] = a < s1;
    s.okb[u] = a + 1 < s1;
    if (V2 && s.okb[u]) {
      const longlong2 k2 = __ldcs(reinterpret_cast<const longlong2*>(kcol + a));
      s.ka[u] = k2.x, s.kb[u] = k2.y;
      const double2 v2 = __ldcs(reinterpret_cast<const double2*>(p.vals + a));
      s.wa[u] = v2.x, s.wb[u] = v2.y;
      if constexpr (D > 0) {
#pragma unroll
        for (int m = 1; m < D; ++m) {
          const longlong2 i2 = __ldcs(reinterpret_cast<const longlong2*>(p.col[m] + a));
          s.ia[u][m] = i2.x, s.ib[u][m] = i2.y;
        }
      }
    } else {
      s.ka[u] = s.oka[u] ? kcol[a] : 0;
      s.kb[u] = s.okb[u] ? kcol[a + 1] : 0;
      s.wa[u] = s.oka[u] ? p.vals[a] : 0.0;
      s.wb[u] = s.okb[u] ? p.vals[a + 1] : 0.0;
      if constexpr (D > 0) {
#pragma unroll
        for (int m = 1; m < D; ++m) {
          s.ia[u][m] = s.oka[u] ? p.col[m][a] : 0;
          s.ib[u][m] = s.okb[u] ? p.col[m][a + 1] : 0;
        }
      }
    }
  }
}

// Gathered contracted-vector entries of one step (rows 2l, 2l+1 of every sub-block).
template <int D, int U>
struct DenseGath {
  static constexpr int DG = D > 1 ? D : 2;
  double ga[U][DG], gb[U][DG];
};

// Issue the gathers of a loaded step (index-checked: an out-of-range contracted index raises
// and is never read).  SV: the last mode's vector is read from shared memory.
template <int D, int U, bool SV>
__device__ __forceinline__ void dense_gather_step(const DenseParams& p, const DenseStep<D, U>& s,
                                                  const double* s_vec, DenseGath<D, U>& g, unsigned int& flags) {
  if constexpr (D > 0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int m = 1; m < D; ++m) {
        const unsigned long long dm = (unsigned long long)p.dims[m];
        const bool bada = (unsigned long long)s.ia[u][m] >= dm, badb = (unsigned long long)s.ib[u][m] >= dm;
        if ((bada && s.oka[u]) || (badb && s.okb[u])) flags |= kFlagIndex;
#ifdef TK_DENSE_NOGATHER  // A/B experiment only: stream without gathers (wrong results)
        g.ga[u][m] = (double)(s.ia[u][m] & 7);
        g.gb[u][m] = (double)(s.ib[u][m] & 7);
        continue;
#endif
        if (SV && m == D - 1) {
          g.ga[u][m] = s_vec[bada ? 0 : s.ia[u][m]];
          g.gb[u][m] = s_vec[badb ? 0 : s.ib[u][m]];
        } else {
          g.ga[u][m] = __ldg(p.vec[m] + (bada ? 0 : s.ia[u][m]));
          g.gb[u][m] = __ldg(p.vec[m] + (badb ? 0 : s.ib[u][m]));
        }
      }
  }
}

// SV (staged vector): the last mode's vector is copied into shared memory once per CTA (one
// persistent CTA of kDenseSvThreads per SM), so its random gathers are LDS instead of L1/L2
// requests.
//
// Three-stage software pipeline per warp over its static sequence of spans (warp w takes spans
// w, w+W, w+2W, ...; W = warps in the grid): while step i is folded, the gathers of step i+1 and
// the column loads of step i+2 are in flight, so neither the stream nor the gathers wait on the
// fold's dependency chain.
template <int D, bool V2, bool SV>
__global__ void __launch_bounds__(SV ? kDenseSvThreads : kDenseThreads, SV ? 1 : TK_DENSE_MINB)
    dense_ttv_kernel(DenseParams p, long long nspans) {
  constexpr int U = kDenseU;
  constexpr long long STEP = 64 * U;
  extern __shared__ __align__(16) double s_vec[];
  if constexpr (SV) {
    // every load of the copy in flight at once (a serial loop of L2 round trips would cost
    // tens of microseconds per CTA)
    const long long nv = p.dims[D - 1];
    const double* __restrict__ g = p.vec[D - 1];
    constexpr int R = 8;
    for (long long i0 = 0; i0 < nv; i0 += (long long)R * blockDim.x) {
      double v[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const long long i = i0 + (long long)j * blockDim.x + threadIdx.x;
        v[j] = i < nv ? __ldg(g + i) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const long long i = i0 + (long long)j * blockDim.x + threadIdx.x;
        if (i < nv) s_vec[i] = v[j];
      }
    }
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int d = D > 0 ? D : p.d;
  const long long n = p.n;
  const unsigned long long nkeep = (unsigned long long)p.dims[0];
  const long long* __restrict__ kcol = p.col[0];
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned int flags = 0;

  auto span_end = [&](long long sp) { return min((sp + 1) * kDenseSpan, n); };
  // step cursor over the warp's span sequence
  auto advance = [&](long long& sp, long long& r) {
    r += STEP;
    if (r >= span_end(sp)) {
      sp += W;
      r = sp * kDenseSpan;
    }
  };

  long long fsp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // fold cursor
  if (fsp >= nspans) return;
  long long fr = fsp * kDenseSpan;
  long long gsp = fsp, gr = fr;  // gather cursor (one step ahead)
  advance(gsp, gr);
  long long lsp = gsp, lr = gr;  // load cursor (two steps ahead)
  advance(lsp, lr);

  DenseStep<D, U> cs, gs, ls;  // steps at the fold, gather and load cursors
  DenseGath<D, U> cg, gg;      // gathered entries of the fold / gather steps
  dense_load_step<D, V2, U>(p, fr, span_end(fsp), cs);
  if (gsp < nspans) dense_load_step<D, V2, U>(p, gr, span_end(gsp), gs);
  dense_gather_step<D, U, SV>(p, cs, s_vec, cg, flags);

  long long curkey = fsp > 0 ? __ldg(kcol + fr - 1) : 0;  // key of the row before the next one
  double acc = 0.0;
  bool seen = false;  // a head was met in this span
  while (true) {
    if (lsp < nspans) dense_load_step<D, V2, U>(p, lr, span_end(lsp), ls);
    if (gsp < nspans) dense_gather_step<D, U, SV>(p, gs, s_vec, gg, flags);

    // ---- fold the step at (fsp, fr) ----
    const long long r = fr;
    const long long s1 = span_end(fsp);
    if constexpr (D > 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int m = D - 1; m >= 1; --m) {
          cs.wa[u] = __dmul_rn(cs.wa[u], cg.ga[u][m]);
          cs.wb[u] = __dmul_rn(cs.wb[u], cg.gb[u][m]);
        }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long a = r + 64 * u + 2 * lane;
        for (int m = d - 1; m >= 1; --m) {
          const unsigned long long dm = (unsigned long long)p.dims[m];
          const long long i0 = cs.oka[u] ? p.col[m][a] : 0, i1 = cs.okb[u] ? p.col[m][a + 1] : 0;
          const bool bada = (unsigned long long)i0 >= dm, badb = (unsigned long long)i1 >= dm;
          if ((bada && cs.oka[u]) || (badb && cs.okb[u])) flags |= kFlagIndex;
          cs.wa[u] = __dmul_rn(cs.wa[u], __ldg(p.vec[m] + (bada ? 0 : i0)));
          cs.wb[u] = __dmul_rn(cs.wb[u], __ldg(p.vec[m] + (badb ? 0 : i1)));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long a = r + 64 * u + 2 * lane;
      const long long ka = cs.ka[u], kb = cs.kb[u];
      const bool oka = cs.oka[u], okb = cs.okb[u];
      const double wa = oka ? cs.wa[u] : 0.0, wb = okb ? cs.wb[u] : 0.0;
      long long pv = __shfl_up_sync(0xffffffffu, kb, 1);
      if (lane == 0) pv = curkey;
      const bool ha = oka && (ka != pv || a == 0);
      const bool hb = okb && kb != ka;
      if ((oka && a > 0 && ka < pv) || (okb && kb < ka)) flags |= kFlagUnsorted;
      if ((oka && (unsigned long long)ka >= nkeep) || (okb && (unsigned long long)kb >= nkeep)) flags |= kFlagKeptOob;
      const unsigned int hm = __ballot_sync(0xffffffffu, ha || hb);
      if (hm == 0) {
        acc = __dadd_rn(acc, wa);
        acc = __dadd_rn(acc, wb);
      } else {
        // slow path: close every run that ends in this sub-block
        const double tot = warp_sum_f64(acc);
        SegPair inc{ha || hb, hb ? wb : __dadd_rn(wa, wb)};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const SegPair up{__shfl_up_sync(0xffffffffu, inc.f, o), __shfl_up_sync(0xffffffffu, inc.v, o)};
          if (lane >= o) inc = seg_combine(up, inc);
        }
        SegPair exc{__shfl_up_sync(0xffffffffu, inc.f, 1), __shfl_up_sync(0xffffffffu, inc.v, 1)};
        if (lane == 0) exc = {0, 0.0};
        // a head at row h closes the run ending at h-1 (continuing the open run when no head
        // precedes h in the sub-block); the open run's first closing before any head of the
        // span is the span's leading carry
        auto close = [&](bool cont, long long key, double v) {
          if (cont && !seen) p.c_first[fsp] = v;
          else dense_store(p, key, v);
        };
        if (ha) close(!exc.f, pv, exc.f ? exc.v : __dadd_rn(tot, exc.v));
        if (hb) {
          const int fa = exc.f | (int)ha;
          const double va = ha ? wa : __dadd_rn(exc.v, wa);
          close(!fa, ka, fa ? va : __dadd_rn(tot, va));
        }
        const double open = __shfl_sync(0xffffffffu, inc.v, 31);
        acc = lane == 0 ? open : 0.0;
        seen = true;
      }
      // key of the last valid row of the sub-block
      const unsigned int mb = __ballot_sync(0xffffffffu, okb), ma = __ballot_sync(0xffffffffu, oka);
      if (mb == 0xffffffffu) {
        curkey = __shfl_sync(0xffffffffu, kb, 31);
      } else if (ma) {
        const int la = 31 - __clz(ma), lb = mb ? 31 - __clz(mb) : -1;
        const long long kla = __shfl_sync(0xffffffffu, ka, la);
        const long long klb = __shfl_sync(0xffffffffu, kb, lb < 0 ? 0 : lb);
        curkey = la > lb ? kla : klb;
      }
    }
    if (r + STEP >= s1) {  // span finished: its carries
      const double total = warp_sum_f64(acc);
      if (lane == 0) {
        const bool last_open = s1 < n && __ldg(kcol + s1) == curkey;
        if (!seen) {
          p.c_first[fsp] = total;
        } else if (last_open) {
          p.c_last[fsp] = total;
          p.c_lastkey[fsp] = curkey;
        } else {
          dense_store(p, curkey, total);
        }
        p.c_flags[fsp] = (seen ? 1 : 0) | (last_open ? 2 : 0);
      }
      if (gsp >= nspans) break;
      curkey = __ldg(kcol + gsp * kDenseSpan - 1);  // gsp > fsp >= 0
      acc = 0.0;
      seen = false;
    }
    // rotate the pipeline
    fsp = gsp, fr = gr;
    gsp = lsp, gr = lr;
    advance(lsp, lr);
    cs = gs;
    cg = gg;
    gs = ls;
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0 && flags) atomicOr(&p.ctr->flags, flags);
}

__global__ void dense_fixup_kernel(long long ntiles, const double* __restrict__ c_first,
                                   const double* __restrict__ c_last, const long long* __restrict__ c_lastkey,
                                   const int* __restrict__ c_flags, DenseParams p) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ntiles || (c_flags[t] & 3) != 3) return;
  double s = c_last[t];
  for (long long t2 = t + 1; t2 < ntiles; ++t2) {
    s = __dadd_rn(s, c_first[t2]);
    const int f2 = c_flags[t2];
    if ((f2 & 1) || !(f2 & 2)) break;
  }
  dense_store(p, c_lastkey[t], s);
}

// ============================================================================================
// host orchestration
// ============================================================================================

namespace {

// Opt a kernel in to >48 KB of dynamic shared memory, once per (kernel, device).
// carveout: preferred shared-memory share of the unified L1 (percent); the tile kernels take it
// all, the staged-vector dense kernel only what its vector needs (L1 caches the other vectors).
template <class K>
void set_smem_once(K kernel, size_t bytes, int carveout = 100) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{reinterpret_cast<const void*>(kernel), dev}];
  if (bytes > have) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    have = bytes;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(long long n, int per_thread = 4) {
  long long want = (n + 256LL * per_thread - 1) / (256LL * per_thread);
  long long cap = (long long)num_sms() * 16;
  return (int)std::max(1LL, std::min(want, cap));
}

template <int SRC, int NK>
int launch_stream_t(SegParams& p, cudaStream_t st, Counters* host_ctr) {
  // one CTA per tile, eight CTAs per SM (~19 KB shared memory each: L1 keeps x resident)
#ifndef TK_SPLIT_SORT
#define TK_SPLIT_SORT 1  // general path: per-interval 32-bit sorts when the leading kept mode is sorted
#endif
#ifndef TK_TILE_LAG
#define TK_TILE_LAG 1024  // tiles between a tile's count and its fold
#endif
#ifndef TK_TILE_ROWS
#define TK_TILE_ROWS 768
#endif
  constexpr int TILE = NK > 0 ? TK_TILE_ROWS : 256;
  constexpr int HALO = 32;
  const int nk = SRC == kSrcLinKey ? 1 : p.nk;
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);
  const size_t smem = tile_total_smem<SRC, TILE, HALO>(ncol, nk);
  auto kern = ttv_tile_kernel<SRC, NK, TILE, HALO>;
  // Raw source: shared memory for 7 CTAs per SM, not 8 -- the unified L1 keeps the rest (60 KB vs
  // 28 KB on sm_100), enough for the hot part of the gathered vector x: config 5 3.33 -> 3.24 ms
  // (5 CTAs: 3.80 ms).  Precomputed-w sources gather nothing and keep every CTA.
  // TK_TILE_CARVEOUT=<percent> overrides (diagnostics).
  static const int tile_carveout = [smem] {
    if (const char* e = getenv("TK_TILE_CARVEOUT")) return std::max(0, std::min(100, atoi(e)));
    if (SRC != kSrcRaw) return 100;
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    if (per_sm <= 0) return 100;
    return (int)std::min<size_t>(100, (100 * 7 * (smem + 1024) + per_sm - 1) / per_sm);
  }();
  set_smem_once(kern, smem, tile_carveout);
  if (getenv("TK_TILE_CARVEOUT")) {
    static bool once = false;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileThreads, smem);
    if (!once) fprintf(stderr, "[tk tile] carveout %d%%: %d CTAs/SM, %zu B smem each\n", tile_carveout, per_sm, smem);
    once = true;
  }
  const long long ntiles = (p.n + TILE - 1) / TILE;
  const size_t status_b = ((size_t)ntiles * 8 + 255) & ~size_t(255);
  DevBuf scratch;
  if (int rc = scratch.alloc(status_b + 256, st)) return rc;
  char* b = scratch.as<char>();
  p.status = reinterpret_cast<unsigned long long*>(b);
  p.ctr = reinterpret_cast<Counters*>(b + status_b);
  TK_CUDA(cudaMemsetAsync(b, 0, status_b + 256, st));
  DevBuf prof;
#ifdef TK_TRACE
  const char* trace_file = getenv("TK_TRACE_FILE");
  const unsigned nblk = (unsigned)(ntiles + std::min<long long>(TK_TILE_LAG, ntiles) + 1);
  if (trace_file) {
    if (int rc = prof.alloc((size_t)nblk * 64, st)) return rc;
    TK_CUDA(cudaMemsetAsync(prof.get(), 0, (size_t)nblk * 64, st));
    p.prof = prof.as<unsigned long long>();
  }
#endif
  {  // TK_TILE_LAG_RT: run-time override of the count-to-fold lag (experiments)
    const char* e = getenv("TK_TILE_LAG_RT");
    const long long lag = e ? std::max(1LL, atoll(e)) : (long long)TK_TILE_LAG;
    p.lag = std::min<long long>(lag, ntiles);
  }
  p.ntiles = ntiles;
  p.out_v2 = p.out_nk == 2 && aligned16(p.out_subs);
  const char* mp = getenv("TK_TILE_MULTIPASS");  // tests force the fallback with "1"
  bool stalled = mp && mp[0] == '1';
  if (!stalled) {
    // block 0: the prefix scanner; block b counts tile b-1 and folds tile b-1-lag
    ktimer_begin(st);
    p.mode = kTileSinglePass;
    kern<<<(unsigned)(ntiles + p.lag + 1), kTileThreads, smem, st>>>(p);
    ktimer_end(st);
    count_launch();
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(host_ctr, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    stalled = (host_ctr->flags & kFlagStall) != 0;
  }
  if (stalled) {
    // The single pass relies on in-order block dispatch; a wait gave up (or the fallback was
    // forced): redo the call as three order-independent launches.  Every tile's output lands at
    // the same place, so rows the stalled pass already wrote are simply rewritten.
    TK_CUDA(cudaMemsetAsync(b, 0, status_b + 256, st));
    ktimer_begin(st);
    p.mode = kTileCountOnly;
    kern<<<(unsigned)ntiles, kTileThreads, smem, st>>>(p);
    scan_tile_status_kernel<<<1, 1024, 0, st>>>(p.status, ntiles);
    p.mode = kTileFoldOnly;
    kern<<<(unsigned)ntiles, kTileThreads, smem, st>>>(p);
    ktimer_end(st);
    count_launch(3);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(host_ctr, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (host_ctr->flags & kFlagStall)
      return fail(TK_ECUDA, "internal error: tile pipeline wait gave up (site " +
                                std::to_string(host_ctr->grab_ticket) + ", tile " +
                                std::to_string(host_ctr->tile_ticket) + ")");
  }
#ifdef TK_TRACE
  if (trace_file) {
    std::vector<unsigned long long> h((size_t)nblk * 8);
    TK_CUDA(cudaMemcpy(h.data(), prof.get(), h.size() * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_file, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
    p.prof = nullptr;
  }
#endif
  return TK_OK;
}

template <int SRC>
int launch_stream(SegParams& p, cudaStream_t st, Counters* host_ctr) {
  const int nk = SRC == kSrcLinKey ? 1 : p.nk;
  switch (nk) {
    case 1: return launch_stream_t<SRC, 1>(p, st, host_ctr);
    case 2: return launch_stream_t<SRC, 2>(p, st, host_ctr);
    case 3: return launch_stream_t<SRC, 3>(p, st, host_ctr);
    case 4: return launch_stream_t<SRC, 4>(p, st, host_ctr);  // static key arrays up to order 7:
    case 5: return launch_stream_t<SRC, 5>(p, st, host_ctr);  // the any-order instance keeps
    case 6: return launch_stream_t<SRC, 6>(p, st, host_ctr);  // kMaxKeep-sized arrays in local memory
    default: return launch_stream_t<SRC, 0>(p, st, host_ctr);
  }
}

// Run one segmented pass over a sorted stream; returns groups/zeros/flags in host_ctr.
int run_seg(int src, SegParams& p, cudaStream_t st, Counters* host_ctr) {
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  int rc = src == kSrcRaw     ? launch_stream<kSrcRaw>(p, st, hc)
           : src == kSrcKeysW ? launch_stream<kSrcKeysW>(p, st, hc)
                              : launch_stream<kSrcLinKey>(p, st, hc);
  if (rc) return rc;
  *host_ctr = *hc;
  return TK_OK;
}

int finish(const Counters& c, int k, long long nx, int nk, long long* out_subs, double* out_vals,
           int64_t* out_nnz, cudaStream_t st, bool keep_zeros = false) {
  if (c.flags & kFlagIndex) {
    char buf[160];
    snprintf(buf, sizeof buf, "ttv: mode-%d index out of range for a vector of length %lld", k, nx);
    return fail(TK_EINDEX, buf);
  }
  if (keep_zeros) {
    *out_nnz = (int64_t)c.groups;
    return TK_OK;
  }
  if (c.zeros) {
    if (int rc = compact_zeros((long long)c.groups, nk, out_subs, out_vals, st)) return rc;
    TK_CUDA(cudaStreamSynchronize(st));
  }
  *out_nnz = (int64_t)(c.groups - c.zeros);
  return TK_OK;
}

// keys of kept modes must fit a signed 63-bit linear index
int lin_bits(const std::vector<long long>& dims) {
  unsigned __int128 prod = 1;
  for (long long dm : dims) {
    prod *= (unsigned __int128)dm;
    if (prod > ((unsigned __int128)1 << 62)) return -1;
  }
  int bits = 0;
  while (bits < 63 && ((unsigned __int128)1 << bits) < prod) ++bits;
  return std::max(bits, 1);
}

// Kept dims for decoding linear keys; the multiply-based decode when every key is < 2^52.
void set_lin_dims(SegParams& p, int nk, const std::vector<long long>& dims) {
  double prod = 1.0;
  for (int c = 0; c < nk; ++c) {
    p.dims[c] = dims[c];
    p.inv_dims[c] = 1.0 / (double)dims[c];
    prod *= (double)dims[c];
  }
  p.lin_fast = prod < 4503599627370496.0;  // 2^52
}

constexpr int kDeclined = -1;  // the split path does not apply: take the one-sort path

long long kSplitMinNnz() {  // TK_SPLIT_MIN_NNZ: smallest stream the split path takes (tests lower it)
  static const long long v = [] {
    const char* e = getenv("TK_SPLIT_MIN_NNZ");
    return e ? std::max(1LL, atoll(e)) : (1LL << 22);
  }();
  return v;
}

// General path for canonical input with a non-leading contracted mode (the paper's middle-mode
// protocol): the rows are already sorted by the leading kept mode, so they are cut into a few
// leading-mode intervals and each is sorted on its own with 32-bit keys (lead - lo) * R + rest --
// 8-bit digit passes = ceil(bits / 8), where one global sort needs ceil(log2(n0 * R) / 8) passes of
// 16-byte (key, w) pairs.  Dense leading values (the Zipf head) get narrow intervals and 2-3
// passes; the sparse tail wide ones and 4.  Stable sorts in disjoint, ordered intervals give the
// same order as the one global stable sort, so results stay bit-identical.
int ttv_general_split(long long nnz, int nk, const KeepCols& kc, const std::vector<long long>& dims,
                      const int64_t* const* cols, const double* vals, const double* x, long long nx, int k,
                      int64_t* out_subs, double* out_vals, int64_t* out_nnz, cudaStream_t st, bool keep_zeros) {
  const long long n0 = dims[0];
  long long R = 1;
  for (int c = 1; c < nk; ++c) R *= dims[c];
  if (nnz < kSplitMinNnz() || n0 > (1LL << 22) || R > (1LL << 31)) return kDeclined;
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  const int g = grid_for(nnz);
  DevBuf ctrbuf, offb;
  if (int rc = ctrbuf.alloc(sizeof(Counters), st)) return rc;
  Counters* dctr = ctrbuf.as<Counters>();
  TK_CUDA(cudaMemsetAsync(dctr, 0, sizeof(Counters), st));
  if (int rc = offb.alloc((size_t)(n0 + 1) * 8, st)) return rc;
  lead_offsets_kernel<<<g, 256, 0, st>>>(nnz, kc.col[0], n0, offb.as<long long>(), dctr);
  count_launch();
  TK_CUDA(cudaGetLastError());
  std::vector<long long> off((size_t)n0 + 1);
  TK_CUDA(cudaMemcpyAsync(off.data(), offb.get(), (size_t)(n0 + 1) * 8, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (hc->flags) return kDeclined;  // unsorted or out-of-range leading column

  // parts: at each start, the fewest digit passes whose interval holds >= kMinRows rows (or
  // reaches the end); otherwise four passes over the widest 32-bit interval
  static const long long kMinRows = [] {  // TK_SPLIT_MIN_ROWS: tests force many small intervals
    const char* e = getenv("TK_SPLIT_MIN_ROWS");
    return e ? std::max(1LL, atoll(e)) : (1LL << 23);  // config 5, k = 1: 2M 20.0, 4M 19.4, 8M 19.2, 16M 19.5 ms
  }();
  PartTable pt{};
  std::vector<int> pbits;
  long long a = 0;
  while (a < n0) {
    long long b = -1;
    for (int P = 1; P <= 4 && b < 0; ++P) {
      const long long W = (1LL << (8 * P)) / R;  // keys (b - a) * R - 1 < 2^(8P)
      if (W < 1) continue;
      const long long e = std::min(n0, a + W);
      if (P == 4 || e == n0 || off[e] - off[a] >= kMinRows) b = e;
    }
    if (b <= a || pt.nparts == kMaxParts) return kDeclined;
    pt.lo[pt.nparts++] = a;
    const unsigned long long maxkey = (unsigned long long)((b - a) * R - 1);
    int bits = 1;
    while (bits < 32 && (maxkey >> bits)) ++bits;
    pbits.push_back(bits);
    if (((bits + 7) / 8) & 1) pt.in_b |= 1ull << (pt.nparts - 1);  // CUB onesweep: 8-bit digits
    a = b;
  }
  pt.lo[pt.nparts] = n0;

  DevBuf k32a, k32b, wa, wb, keys, temp;
  if (int rc = k32a.alloc(nnz * 4, st)) return rc;
  if (int rc = k32b.alloc(nnz * 4, st)) return rc;
  if (int rc = wa.alloc(nnz * 8, st)) return rc;
  if (int rc = wb.alloc(nnz * 8, st)) return rc;
  if (int rc = keys.alloc(nnz * 8, st)) return rc;
  prep_key32_kernel<<<g, 256, 0, st>>>(nnz, nk, kc, reinterpret_cast<const long long*>(cols[k]), vals, x, nx, pt,
                                       k32a.as<unsigned int>(), wa.as<double>(), k32b.as<unsigned int>(),
                                       wb.as<double>(), dctr);
  count_launch();
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (hc->flags & kFlagIndex) return finish(*hc, k, nx, nk, nullptr, nullptr, out_nnz, st);
  if (hc->flags & kFlagKeptOob) return kDeclined;  // garbage kept indices: the LSD path

  size_t tb = 0;
  long long maxrows = 0;
  for (int j = 0; j < pt.nparts; ++j) maxrows = std::max(maxrows, off[pt.lo[j + 1]] - off[pt.lo[j]]);
  {
    cub::DoubleBuffer<unsigned int> kb(k32a.as<unsigned int>(), k32b.as<unsigned int>());
    cub::DoubleBuffer<double> vb(wa.as<double>(), wb.as<double>());
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)std::max(maxrows, 1LL), 0, 32, st));
  }
  if (int rc = temp.alloc(tb, st)) return rc;
  for (int j = 0; j < pt.nparts; ++j) {
    const long long r0 = off[pt.lo[j]], rows = off[pt.lo[j + 1]] - r0;
    if (rows == 0) continue;
    const bool in_b = (pt.in_b >> j) & 1ull;
    unsigned int *ka = k32a.as<unsigned int>() + r0, *kbb = k32b.as<unsigned int>() + r0;
    double *va = wa.as<double>() + r0, *vbb = wb.as<double>() + r0;
    cub::DoubleBuffer<unsigned int> kb(in_b ? kbb : ka, in_b ? ka : kbb);
    cub::DoubleBuffer<double> vb(in_b ? vbb : va, in_b ? va : vbb);
    size_t tbj = tb;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tbj, kb, vb, (int)rows, 0, pbits[j], st));
    widen_part_kernel<<<grid_for(rows), 256, 0, st>>>(rows, kb.Current(), vb.Current(), pt.lo[j] * R,
                                                      keys.as<long long>() + r0, wa.as<double>() + r0);
    count_launch();
    TK_CUDA(cudaGetLastError());
  }
  SegParams p{};
  p.n = nnz;
  p.nk = 1;
  p.key[0] = keys.as<long long>();
  p.a = wa.as<double>();
  p.out_nk = nk;
  set_lin_dims(p, nk, dims);
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  p.bulk_ok = aligned16(p.key[0]) && aligned16(p.a);
  Counters res{};
  if (int rc = run_seg(kSrcLinKey, p, st, &res)) return rc;
  return finish(res, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
}

int ttv_general(int d, const int64_t* shape, long long nnz, const int64_t* const* cols, const double* vals,
                const double* x, long long nx, int k, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                cudaStream_t st, bool keep_zeros) {
  const int nk = d - 1;
  std::vector<long long> dims;
  KeepCols kc{};
  for (int m = 0, c = 0; m < d; ++m)
    if (m != k) {
      kc.col[c] = reinterpret_cast<const long long*>(cols[m]);
      kc.dims[c] = shape[m];
      dims.push_back(shape[m]);
      ++c;
    }
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  const int bits = lin_bits(dims);
  const int g = grid_for(nnz);

  DevBuf keys, keys2, w, w2, ctrbuf, temp;
  if (int rc = ctrbuf.alloc(sizeof(Counters), st)) return rc;
  Counters* dctr = ctrbuf.as<Counters>();
  TK_CUDA(cudaMemsetAsync(dctr, 0, sizeof(Counters), st));
  if (int rc = keys.alloc(nnz * 8, st)) return rc;
  if (int rc = keys2.alloc(nnz * 8, st)) return rc;
  if (int rc = w.alloc(nnz * 8, st)) return rc;
  if (int rc = w2.alloc(nnz * 8, st)) return rc;

  bool linear = bits > 0;
  // TK_SPLIT_SORT=0 in the environment forces the one-sort path (parity tests compare the two)
  static const bool split_env_off = [] {
    const char* e = getenv("TK_SPLIT_SORT");
    return e && e[0] == '0';
  }();
  // TK_MID_MODE=0 in the environment disables the middle-mode counting path (parity tests)
  const char* mm = getenv("TK_MID_MODE");
  if (k == 1 && !(mm && mm[0] == '0')) {
    const int rc = ttv_middle_mode(d, shape, nnz, cols, vals, x, nx, out_subs, out_vals, out_nnz, st, keep_zeros);
    if (rc != kMidDeclined) return rc;
  }
  if (linear && k != 0 && TK_SPLIT_SORT && !split_env_off) {
    const int rc = ttv_general_split(nnz, nk, kc, dims, cols, vals, x, nx, k, out_subs, out_vals, out_nnz, st,
                                     keep_zeros);
    if (rc != kDeclined) return rc;
  }
  if (linear) {
    prep_linkey_kernel2<<<g, 256, 0, st>>>(nnz, nk, kc, reinterpret_cast<const long long*>(cols[k]), vals, x, nx,
                                           keys.as<long long>(), w.as<double>(), dctr);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (hc->flags & kFlagIndex) return finish(*hc, k, nx, nk, nullptr, nullptr, out_nnz, st);
    if (hc->flags & kFlagKeptOob) linear = false;
  }

  Counters res{};
  if (linear) {
    cub::DoubleBuffer<long long> kb(keys.as<long long>(), keys2.as<long long>());
    cub::DoubleBuffer<double> vb(w.as<double>(), w2.as<double>());
    size_t tb = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)nnz, 0, bits, st));
    if (int rc = temp.alloc(tb, st)) return rc;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kb, vb, (int)nnz, 0, bits, st));
    SegParams p{};
    p.n = nnz;
    p.nk = 1;
    p.key[0] = kb.Current();
    p.a = vb.Current();
    p.out_nk = nk;
    set_lin_dims(p, nk, dims);
    p.out_subs = reinterpret_cast<long long*>(out_subs);
    p.out_vals = out_vals;
    p.bulk_ok = aligned16(p.key[0]) && aligned16(p.a);
    if (int rc = run_seg(kSrcLinKey, p, st, &res)) return rc;
    return finish(res, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
  }

  // LSD over kept columns, last column first, signed 64-bit keys, carrying the row permutation
  DevBuf perm, perm2, sorted_cols;
  if (int rc = perm.alloc(nnz * 8, st)) return rc;
  if (int rc = perm2.alloc(nnz * 8, st)) return rc;
  iota_kernel<<<g, 256, 0, st>>>(nnz, perm.as<long long>());
  cub::DoubleBuffer<long long> pb(perm.as<long long>(), perm2.as<long long>());
  {
    size_t tb = 0;
    cub::DoubleBuffer<long long> kb(keys.as<long long>(), keys2.as<long long>());
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, pb, (int)nnz, 0, 64, st));
    if (int rc = temp.alloc(tb, st)) return rc;
    for (int c = nk - 1; c >= 0; --c) {
      cub::DoubleBuffer<long long> kc2(keys.as<long long>(), keys2.as<long long>());
      gather_i64_kernel<<<g, 256, 0, st>>>(nnz, kc.col[c], pb.Current(), kc2.Current());
      TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kc2, pb, (int)nnz, 0, 64, st));
    }
  }
  if (int rc = sorted_cols.alloc((size_t)nnz * 8 * nk, st)) return rc;
  SegParams p{};
  p.n = nnz;
  p.nk = nk;
  for (int c = 0; c < nk; ++c) {
    long long* dst = sorted_cols.as<long long>() + (size_t)c * nnz;
    gather_i64_kernel<<<g, 256, 0, st>>>(nnz, kc.col[c], pb.Current(), dst);
    p.key[c] = dst;
  }
  gather_w_kernel<<<g, 256, 0, st>>>(nnz, pb.Current(), reinterpret_cast<const long long*>(cols[k]), vals, x, nx,
                                     w.as<double>(), dctr);
  TK_CUDA(cudaGetLastError());
  p.a = w.as<double>();
  p.out_nk = nk;
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  p.bulk_ok = 0;  // per-column offsets c*nnz need not be 16-byte aligned
  if (int rc = run_seg(kSrcKeysW, p, st, &res)) return rc;
  TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  res.flags |= hc->flags;
  return finish(res, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
}

}  // namespace

int compact_zeros(long long groups, int nk, long long* out_subs, double* out_vals, cudaStream_t st) {
  const long long nblk = (groups + kCompTile - 1) / kCompTile;
  DevBuf blk, v2, s2;
  if (int rc = blk.alloc(nblk * 8, st)) return rc;
  if (int rc = v2.alloc(groups * 8, st)) return rc;
  if (int rc = s2.alloc(groups * 8 * std::max(nk, 1), st)) return rc;
  nz_count_kernel<<<(unsigned)nblk, 256, 0, st>>>(groups, out_vals, blk.as<long long>());
  scan_blocks_kernel<<<1, 256, 0, st>>>(nblk, blk.as<long long>());
  nz_scatter_kernel<<<(unsigned)nblk, 256, 0, st>>>(groups, nk, out_vals, out_subs, blk.as<long long>(),
                                                    v2.as<double>(), s2.as<long long>());
  count_launch(3);
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaMemcpyAsync(out_vals, v2.get(), groups * 8, cudaMemcpyDeviceToDevice, st));
  TK_CUDA(cudaMemcpyAsync(out_subs, s2.get(), groups * 8 * nk, cudaMemcpyDeviceToDevice, st));
  return TK_OK;
}


int ttv_prefix_try(int d, int64_t nnz, const int64_t* const* cols, const double* vals, const double* x, int64_t nx,
                   int64_t* out_subs, double* out_vals, int64_t* out_nnz, bool* unsorted, cudaStream_t st) {
  *out_nnz = 0;
  *unsorted = false;
  if (nnz == 0) return TK_OK;
  const int nk = d - 1, k = d - 1;
  SegParams p{};
  p.n = nnz;
  p.nk = nk;
  for (int c = 0; c < nk; ++c) p.key[c] = reinterpret_cast<const long long*>(cols[c]);
  p.subk = reinterpret_cast<const long long*>(cols[k]);
  p.a = vals;
  p.x = x;
  p.nx = nx;
  p.out_nk = nk;
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  bool al = aligned16(vals) && aligned16(p.subk);
  for (int c = 0; c < nk; ++c) al = al && aligned16(p.key[c]);
  p.bulk_ok = al;
  Counters c{};
  if (int rc = run_seg(kSrcRaw, p, st, &c)) return rc;
  if ((c.flags & kFlagUnsorted) && !(c.flags & kFlagIndex)) {
    *unsorted = true;
    return TK_OK;
  }
  return finish(c, k, nx, nk, p.out_subs, out_vals, out_nnz, st);
}

int ttv_sparse_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                      const double* x, int64_t nx, int k, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                      cudaStream_t st, bool keep_zeros) {
  *out_nnz = 0;
  if (nnz == 0) return TK_OK;
  const int nk = d - 1;
  if (k == d - 1) {  // kept modes form a prefix: canonical input streams in sorted order
    SegParams p{};
    p.n = nnz;
    p.nk = nk;
    for (int c = 0; c < nk; ++c) p.key[c] = reinterpret_cast<const long long*>(cols[c]);
    p.subk = reinterpret_cast<const long long*>(cols[k]);
    p.a = vals;
    p.x = x;
    p.nx = nx;
    p.out_nk = nk;
    p.out_subs = reinterpret_cast<long long*>(out_subs);
    p.out_vals = out_vals;
    bool al = aligned16(vals) && aligned16(p.subk);
    for (int c = 0; c < nk; ++c) al = al && aligned16(p.key[c]);
    p.bulk_ok = al;
    Counters c{};
    if (int rc = run_seg(kSrcRaw, p, st, &c)) return rc;
    if (!(c.flags & kFlagUnsorted) || (c.flags & kFlagIndex))
      return finish(c, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
    // not canonical after all: fall through to the sort path
  }
  return ttv_general(d, shape, nnz, cols, vals, x, nx, k, out_subs, out_vals, out_nnz, st, keep_zeros);
}

int aos_to_soa(int64_t nnz, int d, const int64_t* aos, int64_t* soa, int64_t pitch, cudaStream_t st) {
  if (nnz == 0) return TK_OK;
  aos_to_soa_kernel<<<grid_for(nnz), 256, 0, st>>>(nnz, d, reinterpret_cast<const long long*>(aos),
                                                   reinterpret_cast<long long*>(soa), pitch);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

int unpack_rows(const RowPack& rp, int64_t n, const uint64_t* packed, int64_t* soa, int64_t pitch, cudaStream_t st) {
  if (n == 0) return TK_OK;
  UnpackPlan p{};
  p.d = rp.d;
  for (int m = 0; m < rp.d; ++m) {
    const uint64_t top = rp.dim[m] - 1;
    const int bits = top == 0 ? 0 : 64 - __builtin_clzll(top);
    p.shift[m] = rp.shift[m];
    p.mask[m] = bits == 64 ? ~0ull : ((1ull << bits) - 1);
  }
  unpack_rows_kernel<<<grid_for(n), 256, 0, st>>>(n, p, reinterpret_cast<const unsigned long long*>(packed),
                                                  reinterpret_cast<long long*>(soa), pitch);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

__global__ void scatter_dense_kernel(long long n, const long long* __restrict__ idx, const double* __restrict__ v,
                                     double* __restrict__ out, long long nout) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long i = idx[r];
    if (i >= 0 && i < nout) out[i] = v[r];
  }
}

int scatter_dense(long long n, const int64_t* idx, const double* v, double* out, long long nout, cudaStream_t st) {
  scatter_dense_kernel<<<grid_for(n), 256, 0, st>>>(n, reinterpret_cast<const long long*>(idx), v, out, nout);
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

int ttv_dense_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                     int keep, const double* const* vecs, double* out, cudaStream_t st) {
  return ttv_dense_peers(d, shape, nnz, cols, vals, keep, vecs, &out, 1, 0, shape[keep], st);
}

int ttv_dense_peers(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    int keep, const double* const* vecs, double* const* outs, int nout, long long key_lo,
                    long long key_hi, cudaStream_t st) {
  const long long nkeep = shape[keep];
  double* out = outs[0];
  PeerOuts po{};
  for (int i = 0; i < nout; ++i) po.p[i] = outs[i];
  po.n = nout;
  auto zero_owned = [&]() -> int {
    if (key_hi <= key_lo) return TK_OK;
    if (nout == 1) {
      TK_CUDA(cudaMemsetAsync(out + key_lo, 0, (size_t)(key_hi - key_lo) * 8, st));
    } else {
      zero_range_kernel<<<(unsigned)std::min<long long>((key_hi - key_lo + 255) / 256, num_sms() * 4), 256, 0, st>>>(
          po, key_lo, key_hi);
      count_launch();
      TK_CUDA(cudaGetLastError());
    }
    return TK_OK;
  };
  if (int rc = zero_owned()) return rc;
  if (nnz == 0) return TK_OK;
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  if (keep == 0 && d >= 2) {
    const long long nspans = (nnz + kDenseSpan - 1) / kDenseSpan;
    DevBuf scratch;
    const size_t per = ((size_t)nspans * 8 + 255) & ~size_t(255);
    if (int rc = scratch.alloc(per * 4 + 512, st)) return rc;
    DenseParams p{};
    p.n = nnz;
    p.d = d;
    p.keep = keep;
    bool al = aligned16(vals);
    for (int m = 0; m < d; ++m) {
      p.col[m] = reinterpret_cast<const long long*>(cols[m]);
      p.vec[m] = vecs[m];
      p.dims[m] = shape[m];
      al = al && aligned16(cols[m]);
    }
    p.vals = vals;
    p.out = out;
    for (int i = 0; i < nout; ++i) p.outs[i] = outs[i];
    p.nout = nout;
    p.key_lo = key_lo;
    p.key_hi = key_hi;
    char* b = scratch.as<char>();
    p.c_first = reinterpret_cast<double*>(b);
    p.c_last = reinterpret_cast<double*>(b + per);
    p.c_lastkey = reinterpret_cast<long long*>(b + 2 * per);
    p.c_flags = reinterpret_cast<int*>(b + 3 * per);
    p.ctr = reinterpret_cast<Counters*>(b + 4 * per);
    p.bulk_ok = al;
    TK_CUDA(cudaMemsetAsync(b + 4 * per, 0, 512, st));
    using K = void (*)(DenseParams, long long);
    const size_t sv_bytes = (size_t)shape[d - 1] * 8;
    const bool sv = d >= 3 && d <= 5 && sv_bytes <= TK_DENSE_SV_MAX;
    K kern;
#define TK_DENSE_PICK(DD) \
  kern = sv ? (al ? dense_ttv_kernel<DD, true, true> : dense_ttv_kernel<DD, false, true>) \
            : (al ? dense_ttv_kernel<DD, true, false> : dense_ttv_kernel<DD, false, false>)
    switch (d) {
      case 2: kern = al ? dense_ttv_kernel<2, true, false> : dense_ttv_kernel<2, false, false>; break;
      case 3: TK_DENSE_PICK(3); break;
      case 4: TK_DENSE_PICK(4); break;
      case 5: TK_DENSE_PICK(5); break;
      default: kern = al ? dense_ttv_kernel<0, true, false> : dense_ttv_kernel<0, false, false>; break;
    }
#undef TK_DENSE_PICK
    const int threads = sv ? kDenseSvThreads : kDenseThreads;
    const size_t smem = sv ? sv_bytes : 0;
    if (sv) set_smem_once(kern, smem, (int)std::min<size_t>(100, (smem + 1024 + 2331) * 100 / (228 * 1024)));
    // resident CTAs per SM of the chosen instance (looked up once per instance and device)
    static std::mutex occ_mu;
    static std::map<std::pair<const void*, int>, int> occ_cache;
    int dev = 0, occ = 0;
    TK_CUDA(cudaGetDevice(&dev));
    {
      std::lock_guard<std::mutex> lk(occ_mu);
      int& o = occ_cache[{reinterpret_cast<const void*>(kern), dev}];
      if (!o) {
        TK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, sv ? (size_t)TK_DENSE_SV_MAX : 0));
        o = std::max(o, 1);
      }
      occ = o;
    }
    const long long wpb = threads / 32;
    const long long warps = std::min(nspans, (long long)num_sms() * occ * wpb);
    const long long blocks = (warps + wpb - 1) / wpb;
    ktimer_begin(st);
    kern<<<(unsigned)blocks, threads, smem, st>>>(p, nspans);
    dense_fixup_kernel<<<(unsigned)((nspans + 255) / 256), 256, 0, st>>>(nspans, p.c_first, p.c_last, p.c_lastkey,
                                                                         p.c_flags, p);
    ktimer_end(st);
    count_launch(2);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(hc, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (hc->flags & kFlagIndex) return fail(TK_EINDEX, "ttv: contracted-mode index out of range for its vector");
    if (hc->flags & kFlagKeptOob) return fail(TK_EDIM, "index out of bounds for shape");
    if (!(hc->flags & kFlagUnsorted)) return TK_OK;
  }
  // general case: the chain of single-mode TTVs; with one output owning every index it writes the
  // output directly, otherwise a local vector whose owned range is stored into every copy
  if (nout == 1 && key_lo == 0 && key_hi == nkeep) {
    TK_CUDA(cudaMemsetAsync(out, 0, (size_t)nkeep * 8, st));  // the fused kernel may have stored some
    return ttv_dense_chain(d, shape, nnz, cols, vals, keep, vecs, out, st);
  }
  DevBuf full;
  if (int rc = full.alloc((size_t)nkeep * 8, st)) return rc;
  TK_CUDA(cudaMemsetAsync(full.get(), 0, (size_t)nkeep * 8, st));
  if (int rc = ttv_dense_chain(d, shape, nnz, cols, vals, keep, vecs, full.as<double>(), st)) return rc;
  if (key_hi > key_lo) {
    bcast_range_kernel<<<(unsigned)std::min<long long>((key_hi - key_lo + 255) / 256, num_sms() * 4), 256, 0, st>>>(
        full.as<double>(), po, key_lo, key_hi);
    count_launch();
    TK_CUDA(cudaGetLastError());
  }
  TK_CUDA(cudaStreamSynchronize(st));  // `full` is released on return
  return TK_OK;
}

// Chained single-mode TTV on the device, descending modes (the oracle's definition), then
// densify into out (zeroed by the caller).
int ttv_dense_chain(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    int keep, const double* const* vecs, double* out, cudaStream_t st) {
  const long long nkeep = shape[keep];
  std::vector<int64_t> cur_shape(shape, shape + d);
  std::vector<const int64_t*> cur_cols(cols, cols + d);
  const double* cur_vals = vals;
  long long cur_nnz = nnz;
  int cur_d = d, cur_keep = keep;
  DevBuf bufs[2][2];  // [ping][subs|vals]
  DevBuf soa;
  int ping = 0;
  for (int m = d - 1; m >= 0; --m) {
    if (m == keep) continue;
    const int nk = cur_d - 1;
    DevBuf& bs = bufs[ping][0];
    DevBuf& bv = bufs[ping][1];
    bs.reset();
    bv.reset();
    if (int rc = bs.alloc((size_t)std::max(cur_nnz, 1LL) * 8 * nk, st)) return rc;
    if (int rc = bv.alloc((size_t)std::max(cur_nnz, 1LL) * 8, st)) return rc;
    int64_t u = 0;
    if (int rc = ttv_sparse_device(cur_d, cur_shape.data(), cur_nnz, cur_cols.data(), cur_vals, vecs[m],
                                   shape[m], m, bs.as<int64_t>(), bv.as<double>(), &u, st))
      return rc;
    // row-major (u, nk) -> SoA for the next stage
    DevBuf nsoa;
    if (int rc = nsoa.alloc((size_t)std::max<int64_t>(u, 1) * 8 * nk, st)) return rc;
    if (int rc = aos_to_soa(u, nk, bs.as<int64_t>(), nsoa.as<int64_t>(), u, st)) return rc;
    soa.reset();
    std::swap(soa, nsoa);
    cur_shape.erase(cur_shape.begin() + m);
    cur_cols.clear();
    for (int c = 0; c < nk; ++c) cur_cols.push_back(soa.as<int64_t>() + (size_t)c * u);
    cur_vals = bv.as<double>();
    cur_nnz = u;
    cur_d = nk;
    if (m < cur_keep) --cur_keep;
    ping ^= 1;
  }
  // order-1 sparse result -> dense
  return cur_nnz ? scatter_dense(cur_nnz, cur_cols[0], cur_vals, out, nkeep, st) : TK_OK;
}

}  // namespace tk
