// tk_midmode.cu -- general-mode TTV with the contracted mode second (k == 1): the paper's own
// benchmark protocol contracts the middle mode (the reference CLI's
// default --mode 2, pkg/src/tenkern/bench.py:69), so this is the sort path the workload hits.
//
// Reference semantics (_ckernels.pyx:313-367): w[r] = vals[r] * x[subs[r,1]]; rows grouped by
// the kept tuple (i0, i2, ..., i_{d-1}); each group summed left to right in ASCENDING ORIGINAL ROW
// ORDER (pyx:262-295); exact-zero sums dropped; groups emitted in lexicographic order.
//
// The input's leading column is sorted (canonical COO), so segment i0 (the rows with that
// leading value) is already in place relative to the other segments: only the rows of equal
// suffix key S = (i2, ..., i_{d-1}) (R = prod of those dims <= 2^14) WITHIN each segment have to
// meet, in row order.  That is a counting problem over small known dims -- no general sort.
// Segments come in three size classes:
//   * class A (<= kWarpMax rows, the tail: 1e6 segments at config 5): one warp per segment.  A
//     bitmap of the S present gives every row its group (the rank of its S = its output order);
//     w = vals * x[i1] is added into acc[group] in row order, 32 rows per step (the first lane of
//     a group adds the group's rows of the step in lane order).  No sort, no scratch.
//   * class M (kWarpMax < rows <= kMedMax): one CTA per segment, acc[S] for every possible S in
//     shared memory.  Chunks of 1024 rows are split stably by OWNER warp (S % 8) into contiguous
//     shared-memory lists; each warp walks its own list in dense 32-row steps, packs a step by S
//     and adds every run onto acc[S] left to right.  All rows of one S pass through one warp in
//     row order, so warps never wait on each other.
//   * class B (> kMedMax rows, the Zipf head): counting tiles of kTileRows rows.  Pass 1
//     histograms S per tile in shared memory; a two-level column scan over each segment's tiles
//     and a scan over S give every (tile, S) its exact row range; pass 2 recomputes w and scatters
//     it stably with the class-M owner lists (the cursor of S is touched by one warp only, in row
//     order), so every (i0, S) bucket holds its w in original row order; pass 3 folds every bucket
//     serially (size bins: one bucket per lane for 64..4095 rows, a whole warp with coalesced
//     loads far ahead of lane 0's chain for longer ones, longest first by ticket).
// Output rows: the groups of every segment (distinct S; counted by bitmap kernels for A and M, by
// the class-B histogram) are exclusive-scanned over i0, so each group knows its output row without
// any cross-CTA wait.  Every sum is the reference's left fold in original row order with
// __dadd_rn, started from the first w or from -0.0 (the exact additive identity): values
// bit-identical to the reference.  No library code is used.
#include <algorithm>
#include <vector>

#include "tk_host.h"
#include "tk_scan.cuh"

namespace tk {

// tk_ttv.cu
__global__ void lead_offsets_kernel(long long n, const long long* __restrict__ col0, long long n0,
                                    long long* __restrict__ off, Counters* ctr);

namespace {

constexpr int kMidThreads = 256;       // class B / class M CTAs: 8 warps, warp w owns the S with S % 8 == w
constexpr int kMidWarps = kMidThreads / 32;
#ifndef TK_MID_WARPMAX
#define TK_MID_WARPMAX 512
#endif
constexpr int kWarpMax = TK_MID_WARPMAX;  // class A: segments of at most kWarpMax rows, one warp each
constexpr long long kMidMaxR = 16384;  // suffix key S < 2^14
constexpr int kChunkTiles = 32;        // column scan: tiles per chunk
constexpr long long kMedMax = 65536;   // class M: segments of kWarpMax+1 .. kMedMax rows
constexpr long long kTileRows = 32768;  // class B counting tile: a smaller write frontier in the scatter (256K rows: +0.9 ms at config 5) against 40 KB of tables per tile

struct MidParams {
  long long nnz, n0, n1, R;
  int ns;                          // suffix modes (d - 2)
  int nk;                          // output columns (d - 1)
  const long long* c0;             // leading kept column (sorted)
  const long long* c1;             // contracted column
  const long long* sc[kMaxKeep];   // suffix kept columns
  long long sdim[kMaxKeep];
  const double* vals;
  const double* x;
  const long long* off;            // n0 + 1 segment offsets
  long long* out_subs;             // row-major (groups, nk)
  double* out_vals;
  const long long* out_base;       // n0 + 1: first output row of every segment
  long long* groups;               // n0: groups of every segment
  long long med_max;               // class M / class B boundary (rows)
  Counters* ctr;
};

template <int NS>
__device__ __forceinline__ long long suffix_key(const MidParams& p, long long r, unsigned int& flags) {
  const int ns = NS > 0 ? NS : p.ns;
  long long s = 0;
  for (int j = 0; j < ns; ++j) {
    const long long v = __ldcs(p.sc[j] + r);
    if ((unsigned long long)v >= (unsigned long long)p.sdim[j]) flags |= kFlagKeptOob;
    s = s * p.sdim[j] + v;
  }
  return s;
}

// The suffix key for pipelined loads: nothing here waits on the loaded value when there is one
// suffix column (the usual 3-way tensor) -- the consumer checks it against R later with
// suffix_check.  With several suffix columns the key is combined at once; -1 = out of range.
template <int NS>
__device__ __forceinline__ long long suffix_load(const MidParams& p, long long r) {
  if (NS == 1) return __ldcs(p.sc[0] + r);
  const int ns = NS > 0 ? NS : p.ns;
  long long s = 0;
  bool oob = false;
  for (int j = 0; j < ns; ++j) {
    const long long v = __ldcs(p.sc[j] + r);
    oob = oob || (unsigned long long)v >= (unsigned long long)p.sdim[j];
    s = s * p.sdim[j] + v;
  }
  return oob ? -1 : s;
}
// a loaded suffix key -> [0, R); out of range: flagged (the call declines), clamped for memory safety
__device__ __forceinline__ long long suffix_check(const MidParams& p, long long s, bool live, unsigned int& flags) {
  if (live && (unsigned long long)s >= (unsigned long long)p.R) flags |= kFlagKeptOob;
  return max(0LL, min(s, p.R - 1));
}

__device__ __forceinline__ double row_w(const MidParams& p, long long r, unsigned int& flags) {
  const long long i1 = __ldg(p.c1 + r);
  const bool bad = (unsigned long long)i1 >= (unsigned long long)p.n1;
  if (bad) flags |= kFlagIndex;
  return __dmul_rn(__ldg(p.vals + r), __ldg(p.x + (bad ? 0 : i1)));
}

__device__ __forceinline__ void emit_group(const MidParams& p, long long g, long long i0, long long s, double v) {
  p.out_vals[g] = v;
  if (p.ns == 1) {  // (i0, S) is the output row: one 16-byte store
    *reinterpret_cast<longlong2*>(p.out_subs + 2 * g) = make_longlong2(i0, s);
    return;
  }
  long long* o = p.out_subs + g * p.nk;
  o[0] = i0;
  for (int j = p.ns - 1; j >= 0; --j) {
    o[1 + j] = s % p.sdim[j];
    s /= p.sdim[j];
  }
}

__device__ __forceinline__ void flush_counters(const MidParams& p, unsigned int flags, unsigned int zeros) {
  flags = __reduce_or_sync(0xffffffffu, flags);
  zeros = __reduce_add_sync(0xffffffffu, zeros);
  if ((threadIdx.x & 31) == 0) {
    if (flags) atomicOr(&p.ctr->flags, flags);
    if (zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
  }
}

// Serial left fold of src[0..n) by one warp: the lanes load 32-value chunks kRingChunks chunks ahead
// and park two chunks per round in a per-warp shared ring just before they are needed; lane 0 adds
// the 64 values in order from the ring (16-byte shared loads, unrolled: the chain runs at the
// 8-cycle latency of a dependent DADD).  The accumulator starts at -0.0, the exact additive
// identity under round-to-nearest, so the result has the bits of w[0] + w[1] + ... folded left to
// right.  Lane 0's result.
constexpr int kRingChunks = 8;

__device__ __forceinline__ double fold_ring_rows(const double* c, int m, double acc) {
  int j = 0;
  for (; j + 16 <= m; j += 16) {
    double2 pr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pr[q] = *reinterpret_cast<const double2*>(c + j + 2 * q);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      acc = __dadd_rn(acc, pr[q].x);
      acc = __dadd_rn(acc, pr[q].y);
    }
  }
  for (; j < m; ++j) acc = __dadd_rn(acc, c[j]);
  return acc;
}

__device__ __forceinline__ double warp_serial_fold(const double* __restrict__ src, long long n, double* ring) {
  const int lane = threadIdx.x & 31;
  double v[kRingChunks];
#pragma unroll
  for (int a = 0; a < kRingChunks; ++a) v[a] = a * 32 + lane < n ? __ldcs(src + a * 32 + lane) : 0.0;
  double acc = -0.0;
  const long long nch = (n + 31) / 32;
  for (long long k0 = 0; k0 < nch; k0 += kRingChunks) {
#pragma unroll
    for (int a = 0; a < kRingChunks; a += 2) {  // static ring slots: chunk k lives in slot k % kRingChunks
      const long long k = k0 + a;
      if (k >= nch) break;  // warp-uniform
      ring[a * 32 + lane] = v[a];
      ring[(a + 1) * 32 + lane] = v[a + 1];
      const long long nx = (k + kRingChunks) * 32 + lane;
      v[a] = nx < n ? __ldcs(src + nx) : 0.0;  // in flight while lane 0 adds
      v[a + 1] = nx + 32 < n ? __ldcs(src + nx + 32) : 0.0;
      __syncwarp();
      if (lane == 0) acc = fold_ring_rows(ring + a * 32, (int)min(64LL, n - k * 32), acc);
      __syncwarp();
    }
  }
  return acc;
}

// Serial left fold of src[0..n) by one thread (buckets of kBigBucket..kHugeBucket rows, one per
// lane): eight values in flight ahead of the dependent adds.
__device__ __forceinline__ double lane_serial_fold(const double* __restrict__ src, unsigned int n) {
  double acc = -0.0;
  unsigned int j = 0;
  if ((reinterpret_cast<unsigned long long>(src) & 8ull) && n > 0) acc = __dadd_rn(acc, src[j++]);  // 16-byte alignment
  double2 cur[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    cur[q] = j + 2 * q + 2 <= n ? __ldcs(reinterpret_cast<const double2*>(src + j) + q) : make_double2(0.0, 0.0);
  for (; j + 8 <= n; j += 8) {
    double2 nxt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      nxt[q] = j + 8 + 2 * q + 2 <= n ? __ldcs(reinterpret_cast<const double2*>(src + j + 8) + q) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc = __dadd_rn(acc, cur[q].x);
      acc = __dadd_rn(acc, cur[q].y);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) cur[q] = nxt[q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {  // the last 0..7 values: pairs already loaded, then an odd one
    if (j + 2 <= n) {
      acc = __dadd_rn(acc, cur[q].x);
      acc = __dadd_rn(acc, cur[q].y);
      j += 2;
    }
  }
  if (j < n) acc = __dadd_rn(acc, src[j]);
  return acc;
}

// ---- planning ---------------------------------------------------------------------------------
// per segment: class-B flag, tile and chunk counts, class-M flag, class-A flag (all exclusive-scanned)
__global__ void mid_classify_kernel(long long n0, const long long* __restrict__ off, long long tile_rows,
                                    long long med_max, long long* __restrict__ isb, long long* __restrict__ ntile,
                                    long long* __restrict__ nchunk, long long* __restrict__ ism,
                                    long long* __restrict__ isa) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n0; i += (long long)gridDim.x * blockDim.x) {
    const long long L = off[i + 1] - off[i];
    const bool b = L > med_max;
    const long long nt = b ? (L + tile_rows - 1) / tile_rows : 0;
    isb[i] = b;
    ntile[i] = nt;
    nchunk[i] = (nt + kChunkTiles - 1) / kChunkTiles;
    ism[i] = L > kWarpMax && !b;
    isa[i] = L >= 1 && L <= kWarpMax;
  }
}

// class-B, class-M and class-A segment lists (ascending i0) and the segment of every class-B tile / chunk
__global__ void mid_lists_kernel(long long n0, const long long* __restrict__ bidx, const long long* __restrict__ tbase,
                                 const long long* __restrict__ cbase, const long long* __restrict__ midx,
                                 const long long* __restrict__ aidx, int* __restrict__ blist, int* __restrict__ tile_seg,
                                 int* __restrict__ chunk_seg, int* __restrict__ mlist, int* __restrict__ alist) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n0; i += (long long)gridDim.x * blockDim.x) {
    if (bidx[i + 1] != bidx[i]) {
      blist[bidx[i]] = (int)i;
      for (long long t = tbase[i]; t < tbase[i + 1]; ++t) tile_seg[t] = (int)i;
      for (long long c = cbase[i]; c < cbase[i + 1]; ++c) chunk_seg[c] = (int)i;
    }
    if (midx[i + 1] != midx[i]) mlist[midx[i]] = (int)i;
    if (aidx[i + 1] != aidx[i]) alist[aidx[i]] = (int)i;
  }
}

// ---- streaming skeleton shared by class B (stable scatter) and class M (ordered accumulate) ----
// Rows [r0, r1) go through the CTA in chunks of kChunk rows.  All threads load a chunk coalesced
// (raw columns one chunk ahead in registers, the x gathers of the next chunk in flight during the
// current one) and form (S, w = vals * x[i1]).  The chunk is then split stably by OWNER -- warp
// S % 8 owns S -- into eight contiguous lists in shared memory: every thread ranks its rows inside
// its 32-row step (one match per step), the step leaders leave the step's per-owner counts, one
// warp scans the 256 counts (owner-major, steps in row order), and every row goes to its slot.
// Each warp then walks its own list in dense 32-row steps.  All rows of one S pass through one
// warp in row order, so the warps never order themselves against each other (no token ring), and a
// step holds only S of its warp.
constexpr int kRowsPerThread = 4;
constexpr int kChunk = kRowsPerThread * kMidThreads;
constexpr int kSteps = kChunk / 32;  // 32-row steps of a chunk, in row order: step = k * kMidWarps + warp
static_assert(kSteps == 32 && kMidWarps == 8, "the count scan gives one lane eight counters of one owner");

struct StreamSmem {  // carved from dynamic shared memory by the kernels
  double* lw;           // kChunk
  unsigned short* ls;   // kChunk
  unsigned short* cnt;  // kMidWarps * kSteps, zero between chunks
  unsigned short* offs; // kMidWarps * kSteps + kMidWarps + 1: slot of (owner, step); list starts; total
};
__host__ __device__ constexpr size_t stream_smem_bytes() {
  return (size_t)kChunk * 10 + (size_t)kMidWarps * kSteps * 4 + 32;
}
__device__ __forceinline__ StreamSmem stream_carve(double* lw_aligned8, unsigned short* u16_area) {
  StreamSmem sm;
  sm.lw = lw_aligned8;
  sm.ls = u16_area;
  sm.cnt = sm.ls + kChunk;
  sm.offs = sm.cnt + kMidWarps * kSteps;
  return sm;
}

template <int NS, class Proc>
__device__ __forceinline__ void stream_owned(const MidParams& p, long long r0, long long r1, const StreamSmem& sm,
                                             unsigned int& flags, Proc&& proc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  long long sA[kRowsPerThread], iA[kRowsPerThread];
  double vA[kRowsPerThread], vB[kRowsPerThread], xB[kRowsPerThread];
  unsigned short sB[kRowsPerThread];
  auto load_raw = [&](long long cbase) {
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const long long r = cbase + k * kMidThreads + tid;
      if (r < r1) {
        sA[k] = suffix_load<NS>(p, r);
        iA[k] = __ldcs(p.c1 + r);
        vA[k] = __ldcs(p.vals + r);
      } else {
        sA[k] = 0;
        iA[k] = 0;
        vA[k] = 0.0;
      }
    }
  };
  auto advance = [&](long long cbase) {  // raw registers (chunk at cbase) -> S, value, x gather in flight
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const long long r = cbase + k * kMidThreads + tid;
      const bool bad = (unsigned long long)iA[k] >= (unsigned long long)p.n1;
      if (bad && r < r1) flags |= kFlagIndex;
      sB[k] = (unsigned short)suffix_check(p, sA[k], r < r1, flags);
      vB[k] = vA[k];
      xB[k] = __ldg(p.x + (bad || r >= r1 ? 0 : iA[k]));
    }
  };
  for (int i = tid; i < kMidWarps * kSteps; i += kMidThreads) sm.cnt[i] = 0;
  load_raw(r0);
  advance(r0);
  load_raw(r0 + kChunk);
  __syncthreads();
  for (long long cbase = r0; cbase < r1; cbase += kChunk) {
    // 1. rank of every row among the rows of its owner inside its 32-row step; per-step counts
    unsigned short sv[kRowsPerThread];
    double w[kRowsPerThread];
    int slot[kRowsPerThread];  // owner * kSteps + step, then the list slot; -1: no row
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      const bool valid = cbase + k * kMidThreads + tid < r1;
      sv[k] = sB[k];
      w[k] = __dmul_rn(vB[k], xB[k]);
      const int owner = sv[k] % kMidWarps;
      const unsigned int m = __match_any_sync(0xffffffffu, valid ? owner : kMidWarps + lane);
      const int rank = __popc(m & lt);
      const int cell = owner * kSteps + k * kMidWarps + warp;
      if (valid && rank == 0) sm.cnt[cell] = (unsigned short)__popc(m);
      slot[k] = valid ? (cell << 8) | rank : -1;
    }
    __syncthreads();
    if (cbase + kChunk < r1) {  // the next chunk's gathers and the raw loads after it
      advance(cbase + kChunk);
      load_raw(cbase + 2 * kChunk);
    }
    // 2. warp 0: exclusive scan of the counts, owner-major (lane l: owner l / 4, eight steps)
    if (warp == 0) {
      int v[8], run = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[q] = sm.cnt[lane * 8 + q];
        sm.cnt[lane * 8 + q] = 0;
        run += v[q];
      }
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      int ex = incl - run;
      if ((lane & 3) == 0) sm.offs[kMidWarps * kSteps + (lane >> 2)] = (unsigned short)ex;  // list start of the owner
      if (lane == 31) sm.offs[kMidWarps * kSteps + kMidWarps] = (unsigned short)incl;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        sm.offs[lane * 8 + q] = (unsigned short)ex;
        ex += v[q];
      }
    }
    __syncthreads();
    // 3. every row to its slot
#pragma unroll
    for (int k = 0; k < kRowsPerThread; ++k) {
      if (slot[k] >= 0) {
        const int pos = sm.offs[slot[k] >> 8] + (slot[k] & 255);
        sm.ls[pos] = sv[k];
        sm.lw[pos] = w[k];
      }
    }
    __syncthreads();
    // 4. the warp's own list, in order
    const int e0 = sm.offs[kMidWarps * kSteps + warp], e1 = sm.offs[kMidWarps * kSteps + warp + 1];
    for (int e = e0; e < e1; e += 32) {
      const int i = min(e + lane, e1 - 1);
      proc(sm.ls[i], sm.lw[i], e + lane < e1);
    }
  }
}

// ---- class B ----------------------------------------------------------------------------------
// pass 1: histogram of S per tile -> H[t][S]
template <int NS>
__global__ void __launch_bounds__(kMidThreads) mid_hist_kernel(MidParams p, long long tile_rows,
                                                             const int* __restrict__ tile_seg,
                                                             const long long* __restrict__ tbase,
                                                             unsigned int* __restrict__ H) {
  extern __shared__ unsigned int s_dyn[];
  unsigned int* s_hist = s_dyn;
  const long long t = blockIdx.x;
  const int i0 = tile_seg[t];
  const long long r0 = p.off[i0] + (t - tbase[i0]) * tile_rows;
  const long long r1 = min(r0 + tile_rows, p.off[i0 + 1]);
  for (long long s = threadIdx.x; s < p.R; s += blockDim.x) s_hist[s] = 0;
  __syncthreads();
  unsigned int flags = 0;
  for (long long r = r0 + threadIdx.x; r < r1; r += 4 * blockDim.x) {  // four loads in flight
    long long s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) s[u] = r + u * blockDim.x < r1 ? suffix_key<NS>(p, r + u * blockDim.x, flags) : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if ((unsigned long long)s[u] < (unsigned long long)p.R) atomicAdd(&s_hist[s[u]], 1u);
  }
  flush_counters(p, flags, 0);
  __syncthreads();
  unsigned int* h = H + t * p.R;
  for (long long s = threadIdx.x; s < p.R; s += blockDim.x) h[s] = s_hist[s];
}

// column scan, level 1: per chunk of kChunkTiles tiles, the sum of each S -> P[chunk][S]
__global__ void mid_chunksum_kernel(long long R, const int* __restrict__ chunk_seg, const long long* __restrict__ tbase,
                                    const long long* __restrict__ cbase, const unsigned int* __restrict__ H,
                                    unsigned int* __restrict__ P) {
  const long long c = blockIdx.x;
  const long long s = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (s >= R) return;
  const int i0 = chunk_seg[c];
  const long long t0 = tbase[i0] + (c - cbase[i0]) * kChunkTiles;
  const long long t1 = min(t0 + kChunkTiles, tbase[i0 + 1]);
  unsigned int sum = 0;
#pragma unroll
  for (int j = 0; j < kChunkTiles; ++j) sum += t0 + j < t1 ? H[(t0 + j) * R + s] : 0u;
  P[c * R + s] = sum;
}

// level 2: per class-B segment, exclusive scan of the chunk sums; TOT[b][S] = the segment's count
__global__ void mid_chunkscan_kernel(long long R, const int* __restrict__ blist, const long long* __restrict__ cbase,
                                     unsigned int* __restrict__ P, unsigned int* __restrict__ TOT) {
  const long long b = blockIdx.x;
  const long long s = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (s >= R) return;
  const int i0 = blist[b];
  unsigned int run = 0;
  for (long long c = cbase[i0]; c < cbase[i0 + 1]; ++c) {
    const unsigned int v = P[c * R + s];
    P[c * R + s] = run;
    run += v;
  }
  TOT[b * R + s] = run;
}

// level 3: H[t][S] -> exclusive prefix of S over the segment's earlier tiles
__global__ void mid_chunkapply_kernel(long long R, const int* __restrict__ chunk_seg, const long long* __restrict__ tbase,
                                      const long long* __restrict__ cbase, unsigned int* __restrict__ H,
                                      const unsigned int* __restrict__ P) {
  const long long c = blockIdx.x;
  const long long s = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  if (s >= R) return;
  const int i0 = chunk_seg[c];
  const long long t0 = tbase[i0] + (c - cbase[i0]) * kChunkTiles;
  const long long t1 = min(t0 + kChunkTiles, tbase[i0 + 1]);
  unsigned int run = P[c * R + s];
  // all loads of the chunk in flight before the first store (H is read and written: the compiler
  // must otherwise order every load after the previous store)
  unsigned int v[kChunkTiles];
#pragma unroll
  for (int j = 0; j < kChunkTiles; ++j) v[j] = t0 + j < t1 ? H[(t0 + j) * R + s] : 0u;
#pragma unroll
  for (int j = 0; j < kChunkTiles; ++j) {
    if (t0 + j < t1) H[(t0 + j) * R + s] = run;
    run += v[j];
  }
}

// per class-B segment: bucket starts (exclusive scan of TOT over S) and group ranks (scan of the
// non-empty flags); groups[i0] = the segment's non-empty buckets
__global__ void __launch_bounds__(1024) mid_segscan_kernel(long long R, const int* __restrict__ blist,
                                                           const unsigned int* __restrict__ TOT,
                                                           unsigned int* __restrict__ BB, unsigned int* __restrict__ GR,
                                                           long long* __restrict__ groups) {
  __shared__ unsigned long long ws[33];
  const long long b = blockIdx.x;
  const unsigned int* tot = TOT + b * R;
  const long long per = (R + blockDim.x - 1) / blockDim.x;
  const long long a = min(R, (long long)threadIdx.x * per), e = min(R, a + per);
  unsigned long long sum = 0;  // rows (low 32) | groups (high 32)
  for (long long s = a; s < e; ++s) sum += (unsigned long long)tot[s] | ((unsigned long long)(tot[s] != 0) << 32);
  unsigned long long total;
  unsigned long long ex = block_excl_scan(sum, ws, &total);
  for (long long s = a; s < e; ++s) {
    BB[b * R + s] = (unsigned int)ex;
    GR[b * R + s] = (unsigned int)(ex >> 32);
    ex += (unsigned long long)tot[s] | ((unsigned long long)(tot[s] != 0) << 32);
  }
  if (threadIdx.x == 0) groups[blist[b]] = (long long)(total >> 32);
}

// pass 2: stable scatter of w into every bucket's row range, in original row order.  The cursor
// of S is touched only by the warp that owns S, in row order.
template <int NS>
__global__ void __launch_bounds__(kMidThreads) mid_scatter_kernel(MidParams p, long long tile_rows,
                                                                const int* __restrict__ tile_seg,
                                                                const long long* __restrict__ tbase,
                                                                const long long* __restrict__ bidx,
                                                                const unsigned int* __restrict__ H,
                                                                const unsigned int* __restrict__ BB,
                                                                double* __restrict__ wout) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  double* lw = reinterpret_cast<double*>(s_raw);
  unsigned int* s_cur = reinterpret_cast<unsigned int*>(lw + kChunk);  // per S: next output row
  const StreamSmem sm = stream_carve(lw, reinterpret_cast<unsigned short*>(s_cur + p.R));
  const int lane = threadIdx.x & 31;
  const unsigned int lt = (1u << lane) - 1u;
  const long long t = blockIdx.x;
  const int i0 = tile_seg[t];
  const long long r0 = p.off[i0] + (t - tbase[i0]) * tile_rows;
  const long long r1 = min(r0 + tile_rows, p.off[i0 + 1]);
  const long long b = bidx[i0];
  const unsigned int seg0 = (unsigned int)p.off[i0];
  for (long long s = threadIdx.x; s < p.R; s += blockDim.x) s_cur[s] = seg0 + BB[b * p.R + s] + H[t * p.R + s];
  unsigned int flags = 0;
  auto step = [&](unsigned short sv, double w, bool valid) {
    const unsigned int m = __match_any_sync(0xffffffffu, valid ? (int)sv : -1 - lane);
    const unsigned int rank = __popc(m & lt);
    unsigned int base = 0;
    if (valid && rank == 0) {
      base = s_cur[sv];
      s_cur[sv] = base + __popc(m);
    }
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (valid) wout[base + rank] = w;
  };
  stream_owned<NS>(p, r0, r1, sm, flags, step);
  flush_counters(p, flags, 0);
}

// pass 3: fold every non-empty (i0, S) bucket.  Buckets under kBigBucket rows: one thread each,
// at once.  Longer ones are queued by size: bin j holds the buckets of [kBigBucket << j,
// kBigBucket << (j + 1)) rows (one bucket per lane, 32 chains of similar length per warp -- a
// single-lane chain costs a whole warp issue slot per add), buckets of >= kHugeBucket rows are
// folded by a whole warp (coalesced loads far ahead of lane 0's chain).
constexpr unsigned int kBigBucket = 64;
constexpr unsigned int kHugeBucket = 4096;
constexpr int kFoldBins = 6;  // log2(kHugeBucket / kBigBucket)

struct FoldQueues {
  unsigned long long* q;              // entries: class-B segment index << 32 | S
  unsigned int* cnt;                  // [0..kFoldBins) bins, [kFoldBins] huge, [kFoldBins + 1] the fold kernel's ticket
  unsigned int off[kFoldBins + 1];    // first entry of every queue
};

__global__ void mid_fold_kernel(MidParams p, const int* __restrict__ blist, const unsigned int* __restrict__ TOT,
                                const unsigned int* __restrict__ BB, const unsigned int* __restrict__ GR,
                                const double* __restrict__ w, FoldQueues fq) {
  const long long b = blockIdx.x;
  const long long s = (long long)blockIdx.y * blockDim.x + threadIdx.x;
  unsigned int zeros = 0;
  if (s < p.R) {
    const unsigned int n = TOT[b * p.R + s];
    if (n >= kBigBucket) {
      const int bin = min(kFoldBins, 31 - __clz(n / kBigBucket));
      fq.q[fq.off[bin] + atomicAdd(fq.cnt + bin, 1u)] = ((unsigned long long)b << 32) | (unsigned long long)s;
    } else if (n > 0) {
      const int i0 = blist[b];
      const long long start = p.off[i0] + BB[b * p.R + s];
      double acc = w[start];
      for (unsigned int j = 1; j < n; ++j) acc = __dadd_rn(acc, w[start + j]);
      emit_group(p, p.out_base[i0] + GR[b * p.R + s], i0, s, acc);
      zeros += acc == 0.0;
    }
  }
  flush_counters(p, 0, zeros);
}

// Persistent warps take work by ticket, longest first: the huge buckets one per warp, then the
// bins from the longest, 32 buckets per warp.  (A static round-robin over one queue resonated with
// its (segment, S) order: with 148 * 64 warps every 37th segment's S = 0 bucket -- the longest
// chains -- landed on the same warp.)
__global__ void __launch_bounds__(256) mid_fold_big_kernel(MidParams p, const int* __restrict__ blist,
                                                           const unsigned int* __restrict__ TOT,
                                                           const unsigned int* __restrict__ BB,
                                                           const unsigned int* __restrict__ GR,
                                                           const double* __restrict__ w, FoldQueues fq) {
  __shared__ __align__(16) double s_ring[8][kRingChunks * 32];
  const int lane = threadIdx.x & 31;
  const unsigned int nh = fq.cnt[kFoldBins];
  unsigned int zeros = 0;
  while (true) {
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(fq.cnt + kFoldBins + 1, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t < nh) {
      const unsigned long long e = fq.q[fq.off[kFoldBins] + t];
      const long long b = (long long)(e >> 32), s = (long long)(e & 0xffffffffu);
      const int i0 = blist[b];
      const double acc = warp_serial_fold(w + p.off[i0] + BB[b * p.R + s], TOT[b * p.R + s], s_ring[threadIdx.x >> 5]);
      if (lane == 0) {
        emit_group(p, p.out_base[i0] + GR[b * p.R + s], i0, s, acc);
        zeros += acc == 0.0;
      }
      continue;
    }
    t -= nh;
    int bin = kFoldBins - 1;
    for (; bin >= 0; --bin) {
      const unsigned int nw = (fq.cnt[bin] + 31) / 32;
      if (t < nw) break;
      t -= nw;
    }
    if (bin < 0) break;
    const unsigned int idx = t * 32 + lane;
    if (idx < fq.cnt[bin]) {
      const unsigned long long e = fq.q[fq.off[bin] + idx];
      const long long b = (long long)(e >> 32), s = (long long)(e & 0xffffffffu);
      const int i0 = blist[b];
      const double acc = lane_serial_fold(w + p.off[i0] + BB[b * p.R + s], TOT[b * p.R + s]);
      emit_group(p, p.out_base[i0] + GR[b * p.R + s], i0, s, acc);
      zeros += acc == 0.0;
    }
  }
  flush_counters(p, 0, zeros);
}

// ---- class M: one CTA per segment -----------------------------------------------------------------
// w = vals * x[i1] is added into acc[S] (one accumulator per possible S, in shared memory) in row
// order through the streaming skeleton: the warp that owns S packs each dense step's rows by S
// (groups matched inside the step, a warp scan of the group sizes gives every S a contiguous run in
// row order), and the first lane of an S loads the accumulator, adds its run left to right and
// stores it -- the reference's fold, started from -0.0 (the exact additive identity).  A bitmap of
// the S seen gives the output order (rank of S) at the end.  COUNT pass first: the bitmap alone.

// marks the S of rows [r0, r1) in the zeroed bitmap (test first: most rows repeat an S already set)
template <int NS>
__device__ __forceinline__ void mark_bitmap(const MidParams& p, long long r0, long long r1, unsigned int* bm,
                                            unsigned int& flags) {
  for (long long r = r0 + threadIdx.x; r < r1; r += 4 * kMidThreads) {
    long long s[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      s[u] = r + u * kMidThreads < r1 ? max(0LL, min(suffix_key<NS>(p, r + u * kMidThreads, flags), p.R - 1)) : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s[u] >= 0) {
        const unsigned int bit = 1u << (s[u] & 31);
        if (!(bm[s[u] >> 5] & bit)) atomicOr(&bm[s[u] >> 5], bit);
      }
  }
}

// warp 0: pre[i] = set bits in words [0, i) (skipped when pre is null); the total in every lane
__device__ __forceinline__ int bitmap_ranks(const unsigned int* bm, unsigned short* pre, int W) {
  const int lane = threadIdx.x & 31;
  const int K = (W + 31) >> 5;
  int cnt = 0;
  for (int k = 0; k < K; ++k) {
    const int i = lane * K + k;
    if (i < W) cnt += __popc(bm[i]);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (pre) {
    int run = incl - cnt;
    for (int k = 0; k < K; ++k) {
      const int i = lane * K + k;
      if (i < W) {
        pre[i] = (unsigned short)run;
        run += __popc(bm[i]);
      }
    }
  }
  return __shfl_sync(0xffffffffu, incl, 31);
}

template <int NS>
__global__ void __launch_bounds__(kMidThreads) mid_cta_count_kernel(MidParams p, const int* __restrict__ mlist) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  unsigned int* bm = reinterpret_cast<unsigned int*>(s_raw);
  const int i0 = mlist[blockIdx.x];
  const int W = (int)((p.R + 31) >> 5);
  for (int i = threadIdx.x; i < W; i += kMidThreads) bm[i] = 0;
  __syncthreads();
  unsigned int flags = 0;
  mark_bitmap<NS>(p, p.off[i0], p.off[i0 + 1], bm, flags);
  __syncthreads();
  if (threadIdx.x < 32) {
    const int G = bitmap_ranks(bm, nullptr, W);
    if (threadIdx.x == 0) p.groups[i0] = G;
  }
  flush_counters(p, flags, 0);
}

__host__ __device__ constexpr size_t cta_smem_bytes(long long R) {
  return (size_t)R * 8 + (size_t)kMidWarps * 32 * 8 + stream_smem_bytes() + (size_t)((R + 31) / 32) * 6 + 16;
}

template <int NS>
__global__ void __launch_bounds__(kMidThreads) mid_cta_kernel(MidParams p, const int* __restrict__ mlist) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int W = (int)((p.R + 31) >> 5);
  double* acc = reinterpret_cast<double*>(s_raw);
  double* runs = acc + p.R;
  double* lw = runs + kMidWarps * 32;
  unsigned int* bm = reinterpret_cast<unsigned int*>(lw + kChunk);
  unsigned short* pre = reinterpret_cast<unsigned short*>(bm + W);
  const StreamSmem sm = stream_carve(lw, pre + W + (W & 1));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  const int i0 = mlist[blockIdx.x];
  const long long r0 = p.off[i0], r1 = p.off[i0 + 1];
  for (long long s = tid; s < p.R; s += kMidThreads) acc[s] = -0.0;
  for (int i = tid; i < W; i += kMidThreads) bm[i] = 0;
  double* run = runs + warp * 32;
  unsigned int flags = 0, zeros = 0;
  auto step = [&](unsigned short sv, double w, bool valid) {
    const unsigned int m = __match_any_sync(0xffffffffu, valid ? (int)sv : -1 - lane);
    const int rank = __popc(m & lt);
    const int n = valid && rank == 0 ? __popc(m) : 0;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int off = incl - n;
    const int goff = __shfl_sync(0xffffffffu, off, __ffs(m) - 1);
    if (valid) run[goff + rank] = w;
    __syncwarp();
    if (n > 0) {
      const double* q = run + off;
      double a = __dadd_rn(acc[sv], q[0]);
      int j = 1;
      for (; j + 4 <= n; j += 4) {  // four loads ahead of four dependent adds
        const double v0 = q[j], v1 = q[j + 1], v2 = q[j + 2], v3 = q[j + 3];
        a = __dadd_rn(a, v0);
        a = __dadd_rn(a, v1);
        a = __dadd_rn(a, v2);
        a = __dadd_rn(a, v3);
      }
      for (; j < n; ++j) a = __dadd_rn(a, q[j]);
      acc[sv] = a;
      const unsigned int bit = 1u << (sv & 31);
      if (!(bm[sv >> 5] & bit)) atomicOr(&bm[sv >> 5], bit);
    }
    __syncwarp();
  };
  __syncthreads();
  stream_owned<NS>(p, r0, r1, sm, flags, step);
  __syncthreads();
  if (warp == 0) bitmap_ranks(bm, pre, W);
  __syncthreads();
  const long long obase = p.out_base[i0];
  for (int i = tid; i < W; i += kMidThreads) {
    unsigned int word = bm[i];
    int g = pre[i];
    while (word) {
      const int bit = __ffs(word) - 1;
      word &= word - 1;
      const double v = acc[i * 32 + bit];
      emit_group(p, obase + g, i0, (long long)i * 32 + bit, v);
      zeros += v == 0.0;
      ++g;
    }
  }
  flush_counters(p, flags, zeros);
}

// ---- class A: one warp per segment ------------------------------------------------------------
// A segment of L <= kWarpMax rows holds at most L distinct S.  The warp marks the S present in a
// bitmap over [0, R), turns it into ranks (prefix popcounts: the group of S is its rank among the
// S present, which is also the output order), and then adds w = vals * x[i1] into acc[group] in
// row order: per 32-row step the first lane of every distinct group loads the accumulator, adds
// its own w and then the w of the later lanes of the same group in lane order (shuffles), and
// stores it back -- the reference's left fold in original row order, started from -0.0 (the exact
// additive identity).  No sort, no scratch, no CTA barrier.  COUNT: only the group count (the
// output rows of every segment must be known before anything is written).
constexpr int kWarpsPerCta = 8;
__host__ __device__ constexpr size_t warp_smem_bytes(int W) {
  return ((size_t)kWarpMax * 8 + (size_t)W * 4 + (size_t)W * 2 + (size_t)kWarpMax * 2 + 15) & ~(size_t)15;
}

template <int NS, bool COUNT>
__global__ void __launch_bounds__(kWarpsPerCta * 32) mid_warp_kernel(MidParams p, const int* __restrict__ alist,
                                                                     long long nseg) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned int lt = (1u << lane) - 1u;
  const int W = (int)((p.R + 31) >> 5);
  unsigned char* mine = s_raw + (size_t)warp * warp_smem_bytes(W);
  double* acc = reinterpret_cast<double*>(mine);
  unsigned int* bm = reinterpret_cast<unsigned int*>(acc + kWarpMax);
  unsigned short* pre = reinterpret_cast<unsigned short*>(bm + W);
  unsigned short* skey = pre + W;
  const int K = (W + 31) >> 5;  // bitmap words per lane in the rank scan
  unsigned int flags = 0, zeros = 0;
  // A segment costs a few dependent DRAM round trips (list entry -> offsets -> rows), so the warp
  // works one segment ahead: while segment q is processed, the rows of its next segment are being
  // prefetched into L2 (lane l takes the l-th 128-byte line of each column: 512 rows) and the list
  // entry and offsets of the one after are in flight.
  const long long qstride = (long long)gridDim.x * kWarpsPerCta;
  const long long q0 = (long long)blockIdx.x * kWarpsPerCta + warp;
  auto seg_of = [&](long long q, int& i0, long long& r0, int& L) {
    i0 = q < nseg ? alist[q] : -1;
    r0 = i0 >= 0 ? p.off[i0] : 0;
    L = i0 >= 0 ? (int)(p.off[i0 + 1] - r0) : 0;
  };
  auto prefetch_rows = [&](long long r0, int L) {
    if (L <= 0) return;
    const int ns = COUNT ? 0 : 2;  // COUNT reads only the suffix columns
    for (int c = 0; c < ns + (NS > 0 ? NS : p.ns); ++c) {
      const char* col = c < ns ? (c == 0 ? (const char*)p.c1 : (const char*)p.vals) : (const char*)p.sc[c - ns];
      const char* a = col + r0 * 8, *e = a + (long long)L * 8;
      const char* line = (const char*)((unsigned long long)a & ~127ull) + 128 * lane;
      if (line < e) asm volatile("prefetch.global.L2 [%0];" ::"l"(line));
    }
  };
  int i0n, Ln, i0nn, Lnn;
  long long r0n, r0nn;
  seg_of(q0, i0n, r0n, Ln);
  seg_of(q0 + qstride, i0nn, r0nn, Lnn);
  for (long long q = q0; q < nseg; q += qstride) {
    const int i0 = i0n;
    const long long r0 = r0n;
    const int L = Ln;
    i0n = i0nn, r0n = r0nn, Ln = Lnn;
    prefetch_rows(r0n, Ln);
    seg_of(q + 2 * qstride, i0nn, r0nn, Lnn);
    if constexpr (COUNT) {
      // the count alone needs no rank scan: exactly one row per distinct S finds its bit clear when
      // it sets it; the bits are cleared again row by row (the bitmap starts and stays zero)
      if (q == q0)
        for (int i = lane; i < W; i += 32) bm[i] = 0;
      __syncwarp();
      int firsts = 0;
      for (int j = lane; j < L; j += 32) {
        const long long s = max(0LL, min(suffix_key<NS>(p, r0 + j, flags), p.R - 1));
        const unsigned int bit = 1u << (s & 31);
        firsts += !(atomicOr(&bm[s >> 5], bit) & bit);
      }
      firsts = __reduce_add_sync(0xffffffffu, firsts);
      if (lane == 0) p.groups[i0] = firsts;
      __syncwarp();
      for (int j = lane; j < L; j += 32) {  // the rows again (L1-resident): clear what they set
        unsigned int dummy = 0;
        const long long s = max(0LL, min(suffix_key<NS>(p, r0 + j, dummy), p.R - 1));
        bm[s >> 5] = 0;
      }
      __syncwarp();
      continue;
    }
    for (int i = lane; i < W; i += 32) bm[i] = 0;
    __syncwarp();
    for (int j = lane; j < L; j += 32) {
      const long long s = max(0LL, min(suffix_key<NS>(p, r0 + j, flags), p.R - 1));
      atomicOr(&bm[s >> 5], 1u << (s & 31));
    }
    __syncwarp();
    int cnt = 0;
    for (int k = 0; k < K; ++k) {
      const int i = lane * K + k;
      if (i < W) cnt += __popc(bm[i]);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int G = __shfl_sync(0xffffffffu, incl, 31);
    int run = incl - cnt;
    for (int k = 0; k < K; ++k) {
      const int i = lane * K + k;
      if (i < W) {
        pre[i] = (unsigned short)run;
        run += __popc(bm[i]);
      }
    }
    for (int g = lane; g < G; g += 32) acc[g] = -0.0;
    __syncwarp();
    // rows in order, 32 per step; the next step's raw loads are in flight during this one
    long long sn = 0, i1n = 0;
    double vn = 0.0;
    if (lane < L) {
      sn = suffix_load<NS>(p, r0 + lane);
      i1n = __ldcs(p.c1 + r0 + lane);
      vn = __ldcs(p.vals + r0 + lane);
    }
    for (int j0 = 0; j0 < L; j0 += 32) {
      const int j = j0 + lane;
      const bool valid = j < L;
      const long long s = max(0LL, min(sn, p.R - 1)), i1 = i1n;
      const double v = vn;
      if (j + 32 < L) {
        sn = suffix_load<NS>(p, r0 + j + 32);
        i1n = __ldcs(p.c1 + r0 + j + 32);
        vn = __ldcs(p.vals + r0 + j + 32);
      }
      const bool bad = (unsigned long long)i1 >= (unsigned long long)p.n1;
      if (bad && valid) flags |= kFlagIndex;
      const double w = __dmul_rn(v, __ldg(p.x + (bad || !valid ? 0 : i1)));
      const unsigned int word = bm[s >> 5];
      const int g = valid ? (int)pre[s >> 5] + __popc(word & ((1u << (s & 31)) - 1u)) : -1 - lane;
      const unsigned int m = __match_any_sync(0xffffffffu, g);
      const bool lead = valid && (m & lt) == 0;
      double a = 0.0;
      if (lead) {
        a = __dadd_rn(acc[g], w);
        skey[g] = (unsigned short)s;
      }
      unsigned int rem = lead ? m & ~(1u << lane) : 0u;  // the later rows of this group, in lane order
      while (__any_sync(0xffffffffu, rem != 0u)) {
        const int src = rem ? __ffs(rem) - 1 : lane;
        const double wv = __shfl_sync(0xffffffffu, w, src);
        if (rem) {
          a = __dadd_rn(a, wv);
          rem &= rem - 1;
        }
      }
      if (lead) acc[g] = a;
      __syncwarp();
    }
    const long long ob = p.out_base[i0];
    for (int g = lane; g < G; g += 32) {
      const double v = acc[g];
      emit_group(p, ob + g, i0, skey[g], v);
      zeros += v == 0.0;
    }
    __syncwarp();
  }
  flush_counters(p, flags, zeros);
}

int mid_grid(long long n) { return (int)std::max(1LL, std::min((n + 255) / 256, (long long)num_sms() * 16)); }

long long env_ll(const char* name, long long dflt) {
  const char* e = getenv(name);
  return e ? std::max(1LL, atoll(e)) : dflt;
}

template <int NS>
int mid_run(MidParams& p, bool keep_zeros, int64_t* out_nnz, cudaStream_t st) {
  const long long n0 = p.n0, R = p.R, nnz = p.nnz;
  // tests shrink these to put small data through every class and many tiles
  const long long tile_rows = env_ll("TK_MID_TILE", kTileRows);
  p.med_max = std::min(kMedMax, std::max<long long>(kWarpMax, env_ll("TK_MID_MEDMAX", kMedMax)));
  long long* hv = static_cast<long long*>(pinned_scratch(sizeof(Counters) + 96));
  Counters* hc = reinterpret_cast<Counters*>(hv + 8);
  DevBuf b_ctr, b_off, b_plan, b_groups;
  if (int rc = b_ctr.alloc(sizeof(Counters), st)) return rc;
  p.ctr = b_ctr.as<Counters>();
  TK_CUDA(cudaMemsetAsync(p.ctr, 0, sizeof(Counters), st));
  if (int rc = b_off.alloc((size_t)(n0 + 1) * 8, st)) return rc;
  lead_offsets_kernel<<<mid_grid(nnz), 256, 0, st>>>(nnz, p.c0, n0, b_off.as<long long>(), p.ctr);
  p.off = b_off.as<long long>();
  if (int rc = b_plan.alloc((size_t)(n0 + 1) * 8 * 5, st)) return rc;
  long long* isb = b_plan.as<long long>();  // -> bidx
  long long* tbase = isb + (n0 + 1);
  long long* cbase = tbase + (n0 + 1);
  long long* midx = cbase + (n0 + 1);
  long long* aidx = midx + (n0 + 1);
  mid_classify_kernel<<<mid_grid(n0), 256, 0, st>>>(n0, p.off, tile_rows, p.med_max, isb, tbase, cbase, midx, aidx);
  count_launch(2);
  TK_CUDA(cudaGetLastError());
  for (long long* a : {isb, tbase, cbase, midx, aidx})
    if (int rc = scan_excl_i64(a, a, n0, st)) return rc;  // [n0] = the totals
  TK_CUDA(cudaMemcpyAsync(hc, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  int j = 0;
  for (long long* a : {isb, tbase, cbase, midx, aidx}) TK_CUDA(cudaMemcpyAsync(hv + j++, a + n0, 8, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (hc->flags) return kMidDeclined;  // unsorted or out-of-range leading column
  const long long nb = hv[0], ntiles = hv[1], nchunks = hv[2], nm = hv[3], na = hv[4];

  if (int rc = b_groups.alloc((size_t)(n0 + 1) * 8, st)) return rc;
  TK_CUDA(cudaMemsetAsync(b_groups.get(), 0, (size_t)(n0 + 1) * 8, st));
  p.groups = b_groups.as<long long>();
  DevBuf b_lists, b_H, b_P, b_TOT, b_BB, b_GR, b_w, b_bigq, b_bign;
  if (int rc = b_lists.alloc((size_t)(nb + ntiles + nchunks + nm + na + 4) * 4, st)) return rc;
  int* blist = b_lists.as<int>();
  int* tseg = blist + nb;
  int* cseg = tseg + ntiles;
  int* mlist = cseg + nchunks;
  int* alist = mlist + nm;
  mid_lists_kernel<<<mid_grid(n0), 256, 0, st>>>(n0, isb, tbase, cbase, midx, aidx, blist, tseg, cseg, mlist, alist);
  count_launch();
  const dim3 blk(256);
  const unsigned int ry = (unsigned int)((R + 255) / 256);
  const size_t hsm = (size_t)R * 4;
  // ---- class B: tiles, column scans, bucket starts / group ranks / group counts
  if (nb > 0) {
    if (int rc = b_H.alloc((size_t)ntiles * R * 4, st)) return rc;
    if (int rc = b_P.alloc((size_t)nchunks * R * 4, st)) return rc;
    if (int rc = b_TOT.alloc((size_t)nb * R * 4, st)) return rc;
    if (int rc = b_BB.alloc((size_t)nb * R * 4, st)) return rc;
    if (int rc = b_GR.alloc((size_t)nb * R * 4, st)) return rc;
    TK_CUDA(cudaFuncSetAttribute(mid_hist_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
    TK_CUDA(cudaFuncSetAttribute(mid_scatter_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(hsm + stream_smem_bytes())));
    mid_hist_kernel<NS><<<(unsigned int)ntiles, kMidThreads, hsm, st>>>(p, tile_rows, tseg, tbase, b_H.as<unsigned int>());
    mid_chunksum_kernel<<<dim3((unsigned int)nchunks, ry), blk, 0, st>>>(R, cseg, tbase, cbase, b_H.as<unsigned int>(),
                                                                         b_P.as<unsigned int>());
    mid_chunkscan_kernel<<<dim3((unsigned int)nb, ry), blk, 0, st>>>(R, blist, cbase, b_P.as<unsigned int>(),
                                                                     b_TOT.as<unsigned int>());
    mid_chunkapply_kernel<<<dim3((unsigned int)nchunks, ry), blk, 0, st>>>(R, cseg, tbase, cbase, b_H.as<unsigned int>(),
                                                                           b_P.as<unsigned int>());
    mid_segscan_kernel<<<(unsigned int)nb, 1024, 0, st>>>(R, blist, b_TOT.as<unsigned int>(), b_BB.as<unsigned int>(),
                                                          b_GR.as<unsigned int>(), p.groups);
    count_launch(5);
  }
  // ---- class M: group counts
  if (nm > 0) {
    mid_cta_count_kernel<NS><<<(unsigned int)nm, kMidThreads, (size_t)((R + 31) / 32) * 4, st>>>(p, mlist);
    count_launch();
  }
  // ---- class A: group counts
  const size_t wsm = kWarpsPerCta * warp_smem_bytes((int)((R + 31) / 32));
  const unsigned int wgrid = (unsigned int)std::max(1LL, std::min((na + kWarpsPerCta - 1) / kWarpsPerCta, (long long)num_sms() * 4));
  if (na > 0) {
    TK_CUDA(cudaFuncSetAttribute(mid_warp_kernel<NS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    TK_CUDA(cudaFuncSetAttribute(mid_warp_kernel<NS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
    mid_warp_kernel<NS, true><<<wgrid, kWarpsPerCta * 32, wsm, st>>>(p, alist, na);
    count_launch();
  }
  TK_CUDA(cudaGetLastError());
  if (int rc = scan_excl_i64(p.groups, p.groups, n0, st)) return rc;  // -> out_base, [n0] = groups
  p.out_base = p.groups;
  // ---- every class: straight to the output rows
  if (nb > 0)
    if (int rc = b_w.alloc((size_t)nnz * 8, st)) return rc;
  if (nb > 0) {
    FoldQueues fq{};
    size_t qtot = 0;
    for (int j = 0; j <= kFoldBins; ++j) {  // a queue of buckets of >= kBigBucket << j rows
      fq.off[j] = (unsigned int)qtot;
      qtot += (size_t)nnz / ((size_t)kBigBucket << j) + 64;
    }
    if (int rc = b_bigq.alloc(qtot * 8, st)) return rc;
    if (int rc = b_bign.alloc(64, st)) return rc;
    TK_CUDA(cudaMemsetAsync(b_bign.get(), 0, 64, st));
    fq.q = b_bigq.as<unsigned long long>();
    fq.cnt = b_bign.as<unsigned int>();
    mid_scatter_kernel<NS><<<(unsigned int)ntiles, kMidThreads, hsm + stream_smem_bytes(), st>>>(
        p, tile_rows, tseg, tbase, isb, b_H.as<unsigned int>(), b_BB.as<unsigned int>(), b_w.as<double>());
    mid_fold_kernel<<<dim3((unsigned int)nb, ry), blk, 0, st>>>(p, blist, b_TOT.as<unsigned int>(), b_BB.as<unsigned int>(),
                                                                b_GR.as<unsigned int>(), b_w.as<double>(), fq);
    mid_fold_big_kernel<<<num_sms() * 8, 256, 0, st>>>(p, blist, b_TOT.as<unsigned int>(), b_BB.as<unsigned int>(),
                                                       b_GR.as<unsigned int>(), b_w.as<double>(), fq);
    count_launch(3);
  }
  if (nm > 0) {
    TK_CUDA(cudaFuncSetAttribute(mid_cta_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)cta_smem_bytes(R)));
    mid_cta_kernel<NS><<<(unsigned int)nm, kMidThreads, cta_smem_bytes(R), st>>>(p, mlist);
    count_launch();
  }
  if (na > 0) {
    mid_warp_kernel<NS, false><<<wgrid, kWarpsPerCta * 32, wsm, st>>>(p, alist, na);
    count_launch();
  }
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaMemcpyAsync(hc, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaMemcpyAsync(hv + 5, p.groups + n0, 8, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  const long long G = hv[5];
  if (hc->flags & kFlagIndex) {
    char buf[160];
    snprintf(buf, sizeof buf, "ttv: mode-1 index out of range for a vector of length %lld", p.n1);
    return fail(TK_EINDEX, buf);
  }
  if (hc->flags & kFlagKeptOob) return kMidDeclined;  // garbage kept indices: the LSD path
  if (keep_zeros) {
    *out_nnz = G;
    return TK_OK;
  }
  if (hc->zeros) {
    if (int rc = compact_zeros(G, p.nk, p.out_subs, p.out_vals, st)) return rc;
    TK_CUDA(cudaStreamSynchronize(st));
  }
  *out_nnz = G - (long long)hc->zeros;
  return TK_OK;
}

}  // namespace

int ttv_middle_mode(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    const double* x, int64_t nx, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                    cudaStream_t st, bool keep_zeros) {
  if (d < 3 || nnz <= 0 || nnz >= (1LL << 31) || shape[0] > (1LL << 24)) return kMidDeclined;
  long long R = 1;
  for (int m = 2; m < d; ++m) {
    R *= shape[m];
    if (R > kMidMaxR) return kMidDeclined;
  }
  MidParams p{};
  p.nnz = nnz;
  p.n0 = shape[0];
  p.n1 = nx;
  p.R = R;
  p.ns = d - 2;
  p.nk = d - 1;
  p.c0 = reinterpret_cast<const long long*>(cols[0]);
  p.c1 = reinterpret_cast<const long long*>(cols[1]);
  for (int m = 2; m < d; ++m) {
    p.sc[m - 2] = reinterpret_cast<const long long*>(cols[m]);
    p.sdim[m - 2] = shape[m];
  }
  p.vals = vals;
  p.x = x;
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  *out_nnz = 0;
  return d == 3 ? mid_run<1>(p, keep_zeros, out_nnz, st) : mid_run<0>(p, keep_zeros, out_nnz, st);
}

// ---- device-wide exclusive scan (tk_scan.cuh) --------------------------------------------------
namespace {
constexpr int kScanThreads = 1024, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(const long long* __restrict__ in, long long n,
                                                                      long long* __restrict__ sums) {
  __shared__ long long ws[33];
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  long long v = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) v += base + i < n ? in[base + i] : 0;
  long long tot;
  block_excl_scan(v, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(long long* __restrict__ sums, long long nt) {
  __shared__ long long ws[33];
  const long long per = (nt + kScanThreads - 1) / kScanThreads;
  const long long a = min(nt, (long long)threadIdx.x * per), e = min(nt, a + per);
  long long v = 0;
  for (long long i = a; i < e; ++i) v += sums[i];
  long long tot;
  long long ex = block_excl_scan(v, ws, &tot);
  for (long long i = a; i < e; ++i) {
    const long long c = sums[i];
    sums[i] = ex;
    ex += c;
  }
  if (threadIdx.x == 0) sums[nt] = tot;
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const long long* in, long long* out, long long n,
                                                                  const long long* __restrict__ sums) {
  __shared__ long long ws[33];
  const long long base = (long long)blockIdx.x * kScanTile + threadIdx.x * kScanItems;
  long long v[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? in[base + i] : 0;
    s += v[i];
  }
  long long tot;
  long long ex = block_excl_scan(s, ws, &tot) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}
}  // namespace

int scan_excl_i64(const long long* in, long long* out, long long n, cudaStream_t st) {
  const long long nt = std::max(1LL, (n + kScanTile - 1) / kScanTile);
  DevBuf sums;
  if (int rc = sums.alloc((size_t)(nt + 1) * 8, st)) return rc;
  scan_tile_sums_kernel<<<(unsigned int)nt, kScanThreads, 0, st>>>(in, n, sums.as<long long>());
  scan_sums_kernel<<<1, kScanThreads, 0, st>>>(sums.as<long long>(), nt);
  scan_apply_kernel<<<(unsigned int)nt, kScanThreads, 0, st>>>(in, out, n, sums.as<long long>());
  count_launch(3);
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

}  // namespace tk
