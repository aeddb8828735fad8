// tk_stream.cuh -- persistent, warp-specialised streaming kernel for sparse-result TTV.
//
// Cooperative launch (every CTA co-resident), 13 warps per CTA:
//   * 8 STREAMER warps: STAGES-deep TMA (cp.async.bulk) pipeline over tiles of TILE rows
//     plus HALO look-ahead rows.  Per tile: w = vals*x[subk] (RN multiply), head flags of
//     the kept-key stream; then every group headed in the tile is either folded by the
//     thread owning its head -- serially, in row order, __dadd_rn, the reference's exact
//     sequence (_ckernels.pyx:274-294) -- when it ends inside tile+halo within kShort rows,
//     or handed to the chain queue.  Folded values are staged in smem and written to the
//     output with coalesced stores once the tile's base offset is known.
//   * 1 SCAN warp: popcount prefix of the head bitmask, publishes the tile aggregate and
//     runs the decoupled look-back (group ids) WHILE the streamers fold -- its latency is
//     off the critical path.
//   * 4 CHAIN warps: drain the job queue (long or tile-spanning groups).  A chain warp
//     streams the group's rows (L2-hot: the streamers just pulled them) in coalesced
//     256-row chunks; lane 0 folds them serially from smem while the next chunk's loads
//     are in flight.  Serial chains therefore never stall the tile pipeline.
// No acquire loads or gpu-scope fences on the hot loop (each costs an L1 invalidate on
// sm_100, which would evict the x-vector working set): status words carry their payload,
// jobs carry the tile aggregate, and job slots are published with a release store and
// polled with relaxed loads.
#pragma once

#include "tk_ttv_kernels.cuh"

namespace tk {

// A chain job is ONE 64-bit word (so publishing it needs no fence):
//   [63:21] first row + 1 (never 0: 0 marks an empty slot)  [20:11] local group id  [10:0] tile head count
// The tile is first_row / TILE; the output slot is base(tile) + local id.
__host__ __device__ __forceinline__ unsigned long long job_pack(long long row, int li, int agg) {
  return ((unsigned long long)(row + 1) << 21) | ((unsigned long long)li << 11) | (unsigned long long)agg;
}
typedef unsigned long long StreamJob;

struct StreamParams {
  SegParams s;          // stream description + outputs + status/ctr
  StreamJob* jobs;      // [ntiles][kJobsPerTile] chain jobs: (row in tile << 16) | local id
  unsigned long long* jcount;  // [ntiles] (base << 8) | (njobs + 1), 0 = not yet published
  long long ntiles;
  unsigned long long* prof;  // optional per-CTA cycle counters [grid][16] (TK_STREAM_PROFILE=1)
};

// Optional phase timing (development instrumentation; off unless prof != nullptr).
#define TKP_START(var) const long long var = (sp.prof ? clock64() : 0)
#define TKP_ADD(slot, var)                                                                        \
  do {                                                                                            \
    if (sp.prof) atomicAdd(sp.prof + blockIdx.x * 16 + (slot), (unsigned long long)(clock64() - (var))); \
  } while (0)
#define TKP_COUNT(slot, v)                                                        \
  do {                                                                            \
    if (sp.prof) atomicAdd(sp.prof + blockIdx.x * 16 + (slot), (unsigned long long)(v)); \
  } while (0)
struct StreamProfDummy_ {
};

constexpr int kStreamWarps = 8;
constexpr int kScanWarp = 8;
constexpr int kChainWarps = 8;
constexpr int kStreamThreads = (kStreamWarps + 1 + kChainWarps) * 32;
constexpr int kShort = 64;   // in-thread fold limit (rows)
constexpr int kChunk = 256;  // chain-warp chunk (8 rows per lane)

// named barriers: 1 = streamers (256), 2 = streamers + scan warp (288)
__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Decoupled look-back with a D-deep window per lane (32*D predecessors per L2 round trip).
// The window must exceed the number of tiles started per round trip, otherwise the
// distance to the nearest published prefix grows without bound.
template <int D>
__device__ __forceinline__ void lookback_publish_agg(unsigned long long* status, long long tile,
                                                     unsigned long long agg) {
  if ((threadIdx.x & 31) == 0) st_relaxed(status + tile, (tile == 0 ? kStPre : kStAgg) | agg);
}

template <int D>
__device__ __forceinline__ unsigned long long lookback_wide(unsigned long long* status, long long tile,
                                                            unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  unsigned long long excl = 0;
  long long look = tile - 1;
  while (true) {
    unsigned long long s[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const long long t = look - (lane * D + i);
      s[i] = t >= 0 ? ld_relaxed(status + t) : kStPre;
    }
    // Only the entries nearer than the nearest inclusive prefix matter: wait until none of
    // those is still unpublished (entries beyond the prefix may stay invalid).
    int first_pre;
    while (true) {
      int fp = 1 << 30, fi = 1 << 30;
#pragma unroll
      for (int i = D - 1; i >= 0; --i) {
        const unsigned long long f = s[i] >> 62;
        if (f == 2) fp = lane * D + i;
        if (f == 0) fi = lane * D + i;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        fp = min(fp, __shfl_xor_sync(0xffffffffu, fp, o));
        fi = min(fi, __shfl_xor_sync(0xffffffffu, fi, o));
      }
      if (fi > fp || fi == (1 << 30)) {
        first_pre = fp;
        break;
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
        if ((s[i] >> 62) == 0 && lane * D + i < fp) s[i] = ld_relaxed(status + (look - (lane * D + i)));
    }
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < D; ++i)
      if (lane * D + i <= first_pre) v += s[i] & kStVal;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (first_pre < (1 << 30)) break;
    look -= 32 * D;
  }
  if (lane == 0) st_relaxed(status + tile, kStPre | (excl + agg));
  return excl;
}

template <int SRC, int NK>
__device__ __forceinline__ bool key_eq_global(const SegParams& p, int nk, long long r, const long long* gk) {
#pragma unroll
  for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
    if (NK == 0 && c >= nk) break;
    if (__ldcg(p.key[c] + r) != gk[c]) return false;
  }
  return true;
}

// acc, then s_a[j .. end) added in order (independent loads, dependent adds).
__device__ __forceinline__ double fold_run(const double* s_a, int j, int end, double acc) {
#ifdef TK_DIAG_NOFOLD  // diagnostics only: wrong values, measures the cost of the serial folds
  return acc + (end > j ? s_a[end - 1] : 0.0);
#endif
  // 16-byte shared loads: half the shared-memory wavefronts of a serial fold
  if ((j & 1) && j < end) acc = __dadd_rn(acc, s_a[j++]);
  for (; j + 4 <= end; j += 4) {
    const double2 v01 = *reinterpret_cast<const double2*>(s_a + j);
    const double2 v23 = *reinterpret_cast<const double2*>(s_a + j + 2);
    acc = __dadd_rn(acc, v01.x);
    acc = __dadd_rn(acc, v01.y);
    acc = __dadd_rn(acc, v23.x);
    acc = __dadd_rn(acc, v23.y);
  }
  if (j + 2 <= end) {
    const double2 v01 = *reinterpret_cast<const double2*>(s_a + j);
    acc = __dadd_rn(acc, v01.x);
    acc = __dadd_rn(acc, v01.y);
    j += 2;
  }
  if (j < end) acc = __dadd_rn(acc, s_a[j]);
  return acc;
}

template <int SRC>
__device__ __forceinline__ void write_key(const SegParams& p, long long g, int c, long long lin_or_col,
                                          const long long* keyvals) {
  (void)lin_or_col;
  long long* o = p.out_subs + g * p.out_nk;
  if constexpr (SRC == kSrcLinKey) {
    long long lin = keyvals[0];
    for (int q = p.out_nk - 1; q >= 0; --q) {
      const long long dm = p.dims[q];
      o[q] = lin % dm;
      lin /= dm;
    }
  } else {
    o[c] = keyvals[c];
  }
}

}  // namespace tk
