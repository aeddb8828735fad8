// tk_ttv_kernels.cuh -- sm_100a kernels for sparse COO tensor-times-vector.
//
// Reference semantics (pkg/src/tenkern/_ckernels.pyx:313-367, _pykernels.py:71-105):
//   w[r] = vals[r] * x[subs[r,k]]          (one RN multiply, _scale_project pyx:129-150)
//   group rows by the kept-mode tuple, sum each group left to right in ascending
//   original-row order (acc = w[first]; acc += w[next] ...; _group_sum_nonzero
//   pyx:262-295), drop groups whose sum is exactly 0.0, emit groups in
//   lexicographic order of the kept tuple.
//
// GPU design:
//   * The kept-mode tuples arrive as a stream that is already non-decreasing
//     (canonical COO with a trailing contracted mode, or the output of the
//     device radix sort on the general path).  Groups are runs of that stream.
//   * One CTA = one tile of TILE rows, staged into shared memory by 1-D TMA bulk
//     copies (cp.async.bulk) completing on an mbarrier.
//   * Group ids come from head flags (key change) -> ballot bitmask -> popcount
//     prefix -> decoupled look-back across tiles.  Output slot of a group = its
//     id, known before any value is summed, so the value folds never gate the
//     scan (no convoy behind long groups).
//   * Each group is folded SERIALLY in row order with __dadd_rn by the thread that
//     owns its head row; the group that runs past the tile end is finished by the
//     whole CTA cooperatively (coalesced chunk loads, one thread folds from smem).
//     That is the reference's exact operation sequence, so values are bit-identical.
//   * Exact-zero groups are counted; a separate stable compaction runs only if
//     that count is non-zero.
#pragma once

#include "tk_common.cuh"

namespace tk {

enum SrcKind : int {
  kSrcRaw = 0,     // SoA kept columns + contracted column + vals, x gathered here
  kSrcKeysW = 1,   // SoA kept columns (already sorted) + precomputed w
  kSrcLinKey = 2,  // one linearised kept key (sorted) + precomputed w; decode on output
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
  long long* out_subs;               // row-major (groups, out_nk)
  double* out_vals;
  unsigned long long* status;        // look-back words, one per tile (zeroed)
  Counters* ctr;
  int bulk_ok;                       // all stream pointers 16-byte aligned
  unsigned long long* prof;          // optional phase counters (TK_TILE_PROFILE=1), else null
  long long lag;                     // tile kernel: block b counts tile b-1 and folds tile b-1-lag
  int out_v2;                        // out_nk == 2 and out_subs 16-byte aligned: one 16-byte key store
};

// development instrumentation: clock64 deltas summed over CTAs (off unless p.prof != null)
#define TKT_NOW() (p.prof ? clock64() : 0LL)
#define TKT_ADD(slot, v)                                                   \
  do {                                                                     \
    if (p.prof) atomicAdd(p.prof + (slot), (unsigned long long)(v));       \
  } while (0)

template <int kItems>
struct SegTile {
  static constexpr int kThreads = 256;
  static constexpr int kTile = kItems * kThreads;
  static constexpr int kWords = kTile / 32;
};

template <int SRC, int NK>
__device__ __forceinline__ int seg_nk(const SegParams& p) {
  if constexpr (SRC == kSrcLinKey) return 1;
  if constexpr (NK > 0) return NK;
  return p.nk;
}

// lexicographic compare of stream row a (in smem) with a key vector b: -1, 0, 1
template <int SRC, int NK, int TILE>
__device__ __forceinline__ int seg_cmp_row_vec(const long long* s_key, int nk, int ra, const long long* b) {
#pragma unroll
  for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
    if (NK == 0 && c >= nk) break;
    long long va = s_key[c * TILE + ra], vb = b[c];
    if (va != vb) return va < vb ? -1 : 1;
  }
  return 0;
}

template <int SRC, int NK, int TILE>
__device__ __forceinline__ int seg_cmp_rows(const long long* s_key, int nk, int ra, int rb) {
#pragma unroll
  for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
    if (NK == 0 && c >= nk) break;
    long long va = s_key[c * TILE + ra], vb = s_key[c * TILE + rb];
    if (va != vb) return va < vb ? -1 : 1;
  }
  return 0;
}

template <int SRC>
__device__ __forceinline__ void seg_emit(const SegParams& p, long long g, const long long* keyvals, double acc) {
  long long* o = p.out_subs + g * p.out_nk;
  if constexpr (SRC == kSrcLinKey) {
    long long lin = keyvals[0];
    for (int c = p.out_nk - 1; c >= 0; --c) {
      long long dm = p.dims[c];
      o[c] = lin % dm;
      lin /= dm;
    }
  } else {
    for (int c = 0; c < p.out_nk; ++c) o[c] = keyvals[c];
  }
  p.out_vals[g] = acc;
  if (acc == 0.0) atomicAdd(&p.ctr->zeros, 1ull);
}

// One CTA per tile.  Dynamic smem: s_key[nk][TILE] i64 | s_a[TILE] f64 | s_subk[TILE] i64 (raw)
template <int SRC, int NK, int kItems>
__global__ void __launch_bounds__(256) seg_ttv_kernel(SegParams p) {
  using T = SegTile<kItems>;
  constexpr int TILE = T::kTile;
  constexpr int NW = T::kWords;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int nk = seg_nk<SRC, NK>(p);
  long long* s_key = reinterpret_cast<long long*>(smem_raw);
  double* s_a = reinterpret_cast<double*>(s_key + (size_t)nk * TILE);
  long long* s_subk = reinterpret_cast<long long*>(s_a + TILE);

  __shared__ __align__(8) uint64_t s_bar;
  __shared__ unsigned int s_head[NW];
  __shared__ int s_wpref[NW];
  __shared__ long long s_tile;
  __shared__ unsigned long long s_base;
  __shared__ long long s_prev[kMaxKeep], s_next[kMaxKeep], s_gkey[kMaxKeep];
  __shared__ int s_has_prev, s_cont, s_spill, s_end;
  __shared__ long long s_spill_g;
  __shared__ double s_spill_acc;
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    s_tile = atomicAdd(&p.ctr->tile_ticket, 1u);
    s_flags = 0;
    s_spill = 0;
  }
  __syncthreads();
  const long long tile = s_tile;
  const long long start = tile * TILE;
  const int cnt = (int)min((long long)TILE, p.n - start);

  // ---- stage the tile in shared memory -------------------------------------------------------
  const bool bulk = p.bulk_ok && cnt == TILE;
  if (bulk) {
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      const uint32_t col_bytes = TILE * 8u;
      const uint32_t ncols = nk + 1 + (SRC == kSrcRaw ? 1 : 0);
      mbar_arrive_expect_tx(&s_bar, col_bytes * ncols);
      const uint64_t pol = l2_evict_first_policy();
      for (int c = 0; c < nk; ++c) bulk_g2s(s_key + (size_t)c * TILE, p.key[c] + start, col_bytes, &s_bar, pol);
      bulk_g2s(s_a, p.a + start, col_bytes, &s_bar, pol);
      if constexpr (SRC == kSrcRaw) bulk_g2s(s_subk, p.subk + start, col_bytes, &s_bar, pol);
    }
  } else {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int r = j * 256 + tid;
      if (r < cnt) {
        for (int c = 0; c < nk; ++c) s_key[c * TILE + r] = p.key[c][start + r];
        s_a[r] = p.a[start + r];
        if constexpr (SRC == kSrcRaw) s_subk[r] = p.subk[start + r];
      }
    }
  }
  if (tid == 32) {  // neighbour keys from global while the copies fly
    s_has_prev = start > 0;
    const bool has_next = start + cnt < p.n;
    for (int c = 0; c < nk; ++c) {
      if (start > 0) s_prev[c] = p.key[c][start - 1];
      if (has_next) s_next[c] = p.key[c][start + cnt];
    }
    s_cont = has_next ? 1 : 0;  // refined below once the tile is resident
  }
  __syncthreads();
  if (bulk) mbar_wait(&s_bar, 0);
  if (tid == 32 && s_cont) s_cont = seg_cmp_row_vec<SRC, NK, TILE>(s_key, nk, cnt - 1, s_next) == 0;

  // ---- w, head flags, sortedness (striped: conflict-free smem) ---------------------------------
  unsigned int flags = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int r = j * 256 + tid;
    bool head = false;
    if (r < cnt) {
      if constexpr (SRC == kSrcRaw) {
        const long long idx = s_subk[r];
        double w = 0.0;
        if (idx < 0 || idx >= p.nx) flags |= kFlagIndex;
        else w = __dmul_rn(s_a[r], __ldg(p.x + idx));
        s_a[r] = w;
      }
      int cmp;
      if (r == 0) cmp = s_has_prev ? seg_cmp_row_vec<SRC, NK, TILE>(s_key, nk, 0, s_prev) : 1;
      else cmp = seg_cmp_rows<SRC, NK, TILE>(s_key, nk, r, r - 1);
      head = cmp != 0;
      if (cmp < 0) flags |= kFlagUnsorted;
    }
    const unsigned int m = __ballot_sync(0xffffffffu, head);
    if (lane == 0) s_head[j * 8 + warp] = m;
  }
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();

  // ---- popcount prefix over head words + look-back --------------------------------------------
  if (warp == 0) {
    constexpr int WPL = NW >= 32 ? NW / 32 : 1;
    int c[WPL];
    int mine = 0;
#pragma unroll
    for (int i = 0; i < WPL; ++i) {
      const int wi = lane * WPL + i;
      c[i] = wi < NW ? __popc(s_head[wi]) : 0;
      mine += c[i];
    }
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int run = incl - mine;
#pragma unroll
    for (int i = 0; i < WPL; ++i) {
      const int wi = lane * WPL + i;
      if (wi < NW) s_wpref[wi] = run;
      run += c[i];
    }
    const unsigned long long agg = (unsigned long long)__shfl_sync(0xffffffffu, incl, 31);
    const unsigned long long excl = lookback_exclusive(p.status, tile, agg);
    if (lane == 0) {
      s_base = excl;
      if (start + cnt == p.n) p.ctr->groups = excl + agg;
      if (s_flags) atomicOr(&p.ctr->flags, s_flags);
    }
  }
  __syncthreads();

  // ---- serial folds, one per group, by the thread owning the head row (blocked rows) ----------
  const unsigned long long base = s_base;
  const int r0 = tid * kItems;
#pragma unroll 1
  for (int i = 0; i < kItems; ++i) {
    const int r = r0 + i;
    if (r >= cnt) break;
    const unsigned int word = s_head[r >> 5];
    if (!((word >> (r & 31)) & 1u)) continue;
    const long long g = (long long)(base + s_wpref[r >> 5] + __popc(word & ((1u << (r & 31)) - 1u)));
    double acc = s_a[r];
    int j = r + 1;
    while (j < cnt && !((s_head[j >> 5] >> (j & 31)) & 1u)) {
      acc = __dadd_rn(acc, s_a[j]);
      ++j;
    }
    long long kv[kMaxKeep];
    for (int c = 0; c < nk; ++c) kv[c] = s_key[c * TILE + r];
    if (j == cnt && s_cont) {
      s_spill = 1;
      s_spill_g = g;
      s_spill_acc = acc;
      for (int c = 0; c < nk; ++c) s_gkey[c] = kv[c];
    } else {
      seg_emit<SRC>(p, g, kv, acc);
    }
  }
  __syncthreads();
  if (!s_spill) return;

  // ---- the last group runs past the tile: finish it cooperatively -----------------------------
  double acc = s_spill_acc;
  long long pos = start + cnt;
#pragma unroll 1
  while (pos < p.n) {
    const int chunk = (int)min((long long)TILE, p.n - pos);
    if (tid == 0) s_end = chunk;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int r = j * 256 + tid;
      if (r < chunk) {
        bool same = true;
        for (int c = 0; c < nk; ++c) same = same && (p.key[c][pos + r] == s_gkey[c]);
        if (!same) atomicMin(&s_end, r);
        double w = p.a[pos + r];
        if constexpr (SRC == kSrcRaw) {
          const long long idx = p.subk[pos + r];
          w = (idx < 0 || idx >= p.nx) ? 0.0 : __dmul_rn(w, __ldg(p.x + idx));
        }
        s_a[r] = w;
      }
    }
    __syncthreads();
    const int end = s_end;
    if (tid == 0)
      for (int i = 0; i < end; ++i) acc = __dadd_rn(acc, s_a[i]);
    if (end < chunk) break;
    pos += chunk;
    __syncthreads();
  }
  if (tid == 0) seg_emit<SRC>(p, s_spill_g, s_gkey, acc);
}

// ---- general path helpers --------------------------------------------------------------------

// w = vals * x[subk] and the linearised kept key (row-major over kept modes == lexicographic
// order when every kept index is in bounds).  Flags contracted-mode and kept-mode range errors.
__global__ void prep_linkey_kernel(long long n, int nk, const long long* const* __restrict__ keep_cols_ptr,
                                   const long long* __restrict__ subk, const double* __restrict__ vals,
                                   const double* __restrict__ x, long long nx, const long long* __restrict__ dims,
                                   long long* __restrict__ key, double* __restrict__ w, Counters* ctr);

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
