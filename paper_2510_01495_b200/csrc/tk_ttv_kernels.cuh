// tk_ttv_kernels.cuh -- sm_100a kernels for sparse COO tensor-times-vector.
//
// Reference semantics (pkg/src/tenkern/_ckernels.pyx:313-367, _pykernels.py:71-105):
//   w[r] = vals[r] * x[subs[r,k]]          (one RN multiply, _scale_project pyx:129-150)
//   group rows by the kept-mode tuple, sum each group left to right in ascending
//   original-row order (acc = w[first]; acc += w[next] ...; _group_sum_nonzero
//   pyx:262-295), drop groups whose sum is exactly 0.0, emit groups in
//   lexicographic order of the kept tuple.
//
// GPU design: the kept-mode tuples arrive as a non-decreasing stream
// (canonical COO with a trailing contracted mode, or the output of the device radix sort on the
// general path); groups are runs of that stream.  The sparse-result kernel is ttv_tile_kernel
// (tk_tile_kernel.cuh); this header holds the stream description shared with it, the output
// helper and the declarations of the general path's helper kernels (tk_ttv.cu).
#pragma once

#include "tk_common.cuh"

namespace tk {

enum SrcKind : int {
  kSrcRaw = 0,     // SoA kept columns + contracted column + vals, x gathered here
  kSrcKeysW = 1,   // SoA kept columns (already sorted) + precomputed w
  kSrcLinKey = 2,  // one linearised kept key (sorted) + precomputed w; decode on output
};

enum TileMode : int {
  kTileSinglePass = 0,  // lagged count/fold with the scanner block (needs in-order block dispatch)
  kTileCountOnly = 1,   // fallback pass 1: block t counts tile t
  kTileFoldOnly = 2,    // fallback pass 3: block t folds tile t (prefixes already scanned)
};

struct SegParams {
  long long n;                       // rows in the stream
  int nk;                            // key columns in the stream (kSrcLinKey: 1)
  const long long* key[kMaxKeep];    // key columns (SoA, device)
  const long long* subk;             // kSrcRaw: contracted-mode column
  const double* a;                   // kSrcRaw: vals;  otherwise: w
  const double* x;                   // kSrcRaw: the vector
  long long nx;
  int out_nk;                        // output columns (= d - 1)
  long long dims[kMaxKeep];          // kSrcLinKey: kept dims for decoding
  double inv_dims[kMaxKeep];         // kSrcLinKey: 1.0 / dims (decoding by multiply + fix-up when
  int lin_fast;                      //   every key is < 2^52, so doubles hold it exactly)
  long long* out_subs;               // row-major (groups, out_nk)
  double* out_vals;
  unsigned long long* status;        // look-back words, one per tile (zeroed)
  Counters* ctr;
  int bulk_ok;                       // all stream pointers 16-byte aligned
  unsigned long long* prof;          // optional phase counters (TK_TILE_PROFILE=1), else null
  long long lag;                     // tile kernel: block b counts tile b-1 and folds tile b-1-lag
  long long ntiles;                  // tile kernel: ceil(n / TILE), computed on the host
  int mode;                          // tile kernel: TileMode
  int out_v2;                        // out_nk == 2 and out_subs 16-byte aligned: one 16-byte key store
};

// development instrumentation: clock64 deltas summed over CTAs (off unless p.prof != null)
#define TKT_NOW() (p.prof ? clock64() : 0LL)
#define TKT_ADD(slot, v)                                                   \
  do {                                                                     \
    if (p.prof) atomicAdd(p.prof + (slot), (unsigned long long)(v));       \
  } while (0)


template <int SRC, int NK>
__device__ __forceinline__ int seg_nk(const SegParams& p) {
  if constexpr (SRC == kSrcLinKey) return 1;
  if constexpr (NK > 0) return NK;
  return p.nk;
}

// lexicographic compare of stream row a (in smem) with a key vector b: -1, 0, 1
// lin / dm and lin % dm for lin < 2^52 without a 64-bit division: the double estimate of the
// quotient is off by at most one, and the remainder fixes it.
__device__ __forceinline__ long long divmod_fast(long long lin, long long dm, double inv, long long* rem) {
  long long q = (long long)((double)lin * inv);
  long long r = lin - q * dm;
  if (r < 0) {
    --q;
    r += dm;
  } else if (r >= dm) {
    ++q;
    r -= dm;
  }
  *rem = r;
  return q;
}

template <int SRC>
__device__ __forceinline__ void seg_emit(const SegParams& p, long long g, const long long* keyvals, double acc) {
  long long* o = p.out_subs + g * p.out_nk;
  if constexpr (SRC == kSrcLinKey) {
    long long lin = keyvals[0];
    for (int c = p.out_nk - 1; c >= 0; --c) {
      const long long dm = p.dims[c];
      if (p.lin_fast) {
        long long rem;
        lin = divmod_fast(lin, dm, p.inv_dims[c], &rem);
        o[c] = rem;
      } else {
        o[c] = lin % dm;
        lin /= dm;
      }
    }
  } else {
    for (int c = 0; c < p.out_nk; ++c) o[c] = keyvals[c];
  }
  p.out_vals[g] = acc;
  if (acc == 0.0) atomicAdd(&p.ctr->zeros, 1ull);
}


// ---- general path helpers --------------------------------------------------------------------

__global__ void iota_kernel(long long n, long long* out);
__global__ void gather_i64_kernel(long long n, const long long* __restrict__ src, const long long* __restrict__ idx,
                                  long long* __restrict__ dst);
__global__ void gather_w_kernel(long long n, const long long* __restrict__ perm, const long long* __restrict__ subk,
                                const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                double* __restrict__ w, Counters* ctr);

// ---- zero-group compaction (rare path) --------------------------------------------------------
__global__ void nz_count_kernel(long long n, const double* __restrict__ v, long long* __restrict__ blk);
__global__ void scan_blocks_kernel(long long nblk, long long* __restrict__ blk);
__global__ void nz_scatter_kernel(long long n, int nk, const double* __restrict__ v, const long long* __restrict__ s,
                                  const long long* __restrict__ blk, double* __restrict__ v2, long long* __restrict__ s2);

// ---- layout conversion ------------------------------------------------------------------------
__global__ void aos_to_soa_kernel(long long n, int d, const long long* __restrict__ aos, long long* __restrict__ soa,
                                  long long pitch);

}  // namespace tk
