// tk_tile_kernel.cuh -- sparse-result TTV: one compact CTA per tile, eight CTAs per SM.
//
// Per CTA (128 threads, a 768-row tile + 32 halo rows; block b counts tile b-1 and folds tile
// b-1-lag, block 0 is the sequential prefix scanner):
//   1. thread 0 stages every column of the fold tile into shared memory with 1-D TMA bulk
//      copies (cp.async.bulk, one mbarrier); meanwhile every warp counts the group heads of the
//      count tile straight from global memory and publishes the tile aggregate;
//   2. head bitmask + order check of the staged keys, popcount prefix, each head row recorded
//      at its local id; the tile's exclusive prefix (published ~lag tiles earlier by the scanner);
//   3. w = vals * x[subk] with every gather in flight before any store;
//   4. every group closing inside the stage is folded by one thread, striped, and written at
//      base + local id; the group that runs past the stage is finished through the spill ring
//      (warps 1-3 produce 128-row chunks, warp 0 lane 0 folds).  Every fold is serial in row order
//      with __dadd_rn: the reference's exact operation sequence (_ckernels.pyx:274-294), hence
//      bit-identical values.
#pragma once

#include <climits>

#include "tk_fold.cuh"

namespace tk {

#ifndef TK_TILE_MINB
#define TK_TILE_MINB 8  // resident CTAs per SM the register budget is sized for
#endif
#ifndef TK_TILE_PF
#define TK_TILE_PF 256  // tiles ahead of the count whose columns are prefetched into L2
#endif
#ifndef TK_TILE_PFV
#define TK_TILE_PFV 64  // tiles ahead of the fold whose value columns are prefetched into L2
#endif
#ifndef TK_SCAN_D
#define TK_SCAN_D 8  // status words per scanner lane per round
#endif
#ifndef TK_TILE_THREADS
#define TK_TILE_THREADS 128
#endif
constexpr int kTileThreads = TK_TILE_THREADS;  // threads per CTA
// Development trace (-DTK_TRACE): per block, clock64 at the phase boundaries into p.prof[block*8 + slot]
// (slot 0 = smid << 48 | start clock); the host dumps it to $TK_TRACE_FILE.
#ifdef TK_TRACE
#define TKR_START()                                                                                    \
  if (threadIdx.x == 0 && p.prof) {                                                                    \
    unsigned int smid_;                                                                                \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));                                                \
    p.prof[(size_t)blockIdx.x * 8] = ((unsigned long long)smid_ << 48) | (clock64() & ((1ull << 48) - 1)); \
  }
#define TKR(slot) \
  if (p.prof) p.prof[(size_t)blockIdx.x * 8 + (slot)] = clock64() & ((1ull << 48) - 1)
#else
#define TKR_START()
#define TKR(slot)
#endif
constexpr int kTileWarps = kTileThreads / 32;
#ifndef TK_SPILL_SLOTS
#define TK_SPILL_SLOTS 6
#endif
#ifndef TK_RING_WATCHDOG
#define TK_RING_WATCHDOG 0  // spin limits on the CTA-local spill ring (costs ~3% at cfg5; debug)
#endif
#ifndef TK_SPILL_AHEAD
#define TK_SPILL_AHEAD 1  // spill chunks loaded ahead of the last one known to continue the group (2, 3: slower)
#endif
#ifndef TK_SPILL_NAP
#define TK_SPILL_NAP 32  // ns between a waiting producer's polls
#endif
#ifndef TK_SPILL_W0FIRST
#define TK_SPILL_W0FIRST 0  // with an open group, warp 0 skips the striped folds (measured slower)
#endif
constexpr int kSpillSlots = TK_SPILL_SLOTS;
// The count's key loads stream through once (the stage re-reads them by TMA, into shared memory):
// cache them in L2 only, so L1 keeps the gathered vector x.
#ifndef TK_CNT_CG
#define TK_CNT_CG 1
#endif
#if TK_CNT_CG
#define TK_CNT_LD(ptr) __ldcg(ptr)
#else
#define TK_CNT_LD(ptr) (*(ptr))
#endif  // 128-row chunks of the spill ring (in the 6.4 KB subk column)

__device__ __forceinline__ int ld_vol(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_vol(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }
// Tile status word: while counting, every warp adds (1 << 56) | its head count (so the aggregate is
// complete when the warp field reads kTileWarps); the scanner then stores kStPre | inclusive prefix.
constexpr int kStWarpShift = 56;
constexpr unsigned long long kStCntMask = (1ull << kStWarpShift) - 1;
constexpr unsigned long long kStReady = (unsigned long long)kTileWarps << kStWarpShift;
// stage columns + previous-row words + head-row ids (+ the spill's 128-row chunk buffer for the
// precomputed-w sources, which have no subk column to reuse)
template <int TILE, int HALO>
constexpr size_t tile_smem_bytes(int ncol, int nk) {
  return ((size_t)ncol * (TILE + HALO) + 2 * nk) * 8 + (size_t)(TILE + HALO) * 2;
}

template <int SRC, int TILE, int HALO>
constexpr size_t tile_total_smem(int ncol, int nk) {
  return tile_smem_bytes<TILE, HALO>(ncol, nk) + (SRC == kSrcRaw ? 0 : (size_t)128 * 8);
}

__device__ __forceinline__ void named_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// The sequential scanner (block 0 of the launch, warp 0): turns published tile aggregates into
// inclusive prefixes, in order, as fast as they appear.  Each round it takes the longest run of
// already-published aggregates in the next 32*D tiles (one L2 round trip), scans it, publishes the
// prefixes and advances.  A tile therefore waits ~one round trip after its own aggregate, and
// polls only its own status word -- no wide look-back windows hammering L2.
// A wait that gives up raises kFlagStall; the first one records where (Counters::grab_ticket =
// site, tile_ticket = tile).
__device__ __forceinline__ void tile_stall(Counters* ctr, unsigned long long site, long long tile) {
  if (atomicCAS(&ctr->grab_ticket, 0u, (unsigned int)site) == 0u) atomicExch(&ctr->tile_ticket, (unsigned int)tile);
  atomicOr(&ctr->flags, kFlagStall);
}

template <int D>
__device__ void tile_scanner(unsigned long long* status, long long ntiles, Counters* ctr) {
  const int lane = threadIdx.x & 31;
  unsigned long long carry = 0;
  long long w = 0;
  unsigned int spins = 0;
  while (w < ntiles) {
    unsigned long long v[D];
    int my_first_missing = D;  // first unpublished element of this lane
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const long long t = w + lane * D + i;
      v[i] = t < ntiles ? ld_relaxed(status + t) : kStReady;
      if ((v[i] >> kStWarpShift) != (unsigned long long)kTileWarps && my_first_missing == D) my_first_missing = i;
    }
    // global position of the first unpublished tile in the window
    int first = my_first_missing < D ? lane * D + my_first_missing : 32 * D;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (first == 0) {  // spin: the scanner's latency is every tile's latency
#ifdef TK_NO_WATCHDOG
      if (false) {
#else
      if (++spins == kSpinLimit) {
#endif
        if (lane == 0) tile_stall(ctr, 1, w);
        return;
      }
      continue;
    }
    spins = 0;
    // inclusive scan of the published run [0, first)
    unsigned long long run = 0, loc[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int e = lane * D + i;
      run += (e < first) ? (v[i] & kStCntMask) : 0ull;
      loc[i] = run;
    }
    unsigned long long incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long up = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += up;
    }
    const unsigned long long excl_lane = carry + incl - run;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int e = lane * D + i;
      const long long t = w + e;
      if (e < first && t < ntiles) st_relaxed(status + t, kStPre | (excl_lane + loc[i]));
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
    w += first;
  }
}

// A tile's exclusive prefix once the scanner has published it (tile 0: 0).
// (false: the watchdog gave up)
// `s` is an early read of the status word (issued at block start, usually already the prefix).
__device__ __forceinline__ bool tile_wait_prefix(unsigned long long* status, long long tile, unsigned long long agg,
                                                 unsigned long long s, unsigned long long* excl) {
  unsigned int spins = 0;
  while ((s >> 62) != 2) {
#ifndef TK_NO_WATCHDOG
    if (++spins == kSpinLimit) return false;
#endif
    __nanosleep(32);
    s = ld_relaxed(status + tile);
  }
  *excl = (s & kStVal) - agg;
  return true;
}

template <int SRC, int NK, int TILE, int HALO>
__global__ void __launch_bounds__(kTileThreads, TK_TILE_MINB) ttv_tile_kernel(SegParams p) {
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int ITER = (ROWS + kTileThreads - 1) / kTileThreads;
  constexpr int NKR = NK > 0 ? NK : kMaxKeep;
  static_assert(ROWS % 32 == 0 && WORDS <= 32 && TILE % 32 == 0 && ROWS <= 1024, "tile geometry");
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  long long* st = reinterpret_cast<long long*>(smem_raw);
  long long* s_key = st;
  double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
  long long* s_subk = st + (size_t)(nk + 1) * ROWS;
  long long* s_prev2 = st + (size_t)ncol * ROWS;
  // folded values by local id reuse the subk column (free once w is formed); for the
  // precomputed-w sources there is no subk column, so they get their own area
  short* s_row = reinterpret_cast<short*>(s_prev2 + 2 * nk);
  double* s_val =
      SRC == kSrcRaw ? reinterpret_cast<double*>(s_subk) : reinterpret_cast<double*>(s_row + ROWS);

  __shared__ __align__(8) uint64_t s_bar;
  __shared__ long long s_tile;
  __shared__ int s_bulk;
  __shared__ unsigned int s_head[WORDS];
  __shared__ unsigned long long s_base;
  __shared__ unsigned int s_flags;
  // spill ring (raw source): warps 1-3 produce 128-row chunks of w past the stage into
  // kSpillSlots slots of the free subk column, warp 0 folds them in order
  __shared__ int s_ready[kSpillSlots], s_end[kSpillSlots];
  __shared__ int s_known, s_last, s_consumed;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long ntiles = p.ntiles;
  if (p.mode == kTileSinglePass && blockIdx.x == 0) {  // dispatched first, stays resident: the prefix scanner
    if (warp == 0) tile_scanner<TK_SCAN_D>(p.status, ntiles, p.ctr);
    return;
  }
  // Single pass: blocks are dispatched in index order (the single-pass scan convention; if that
  // ever fails, e.g. under MPS or SM partitioning, a wait gives up and the host re-runs the call
  // as three order-independent passes: kTileCountOnly, scan_tile_status, kTileFoldOnly).  Block b
  // COUNTS the heads of tile b-1 (publishing its aggregate) and FOLDS tile b-1-lag: the prefix of
  // a tile is therefore published ~lag tiles before anyone needs it, and the fold's key columns
  // are L2-hot from the count.
  const long long count_tile = p.mode == kTileSinglePass ? (long long)blockIdx.x - 1
                               : p.mode == kTileCountOnly ? (long long)blockIdx.x : -1;
  const long long fold_tile = p.mode == kTileSinglePass ? count_tile - p.lag
                              : p.mode == kTileFoldOnly ? (long long)blockIdx.x : -1;
  TKR_START();
  // the fold tile's status word, read now: published ~lag tiles ago, so this is almost always the
  // prefix already and its L2 round trip overlaps the count instead of delaying the fold
  unsigned long long pre = 0;
  if (tid == 0 && fold_tile >= 0 && fold_tile < ntiles) pre = ld_relaxed(p.status + fold_tile);
  if (tid == 0 && fold_tile >= 0) {
    const long long tile = fold_tile;
    s_tile = tile;
    s_flags = 0;
    if constexpr (SRC == kSrcRaw) {
#pragma unroll
      for (int i = 0; i < kSpillSlots; ++i) s_ready[i] = 0;
      s_known = 0;
      s_last = INT_MAX;
      s_consumed = 0;
    }
    const long long start = tile * TILE;
    const long long avail = min((long long)ROWS, p.n - start);
    const bool bulk = p.bulk_ok && avail == ROWS;
    s_bulk = bulk;
    if (bulk) {
      mbar_init(&s_bar, 1);
      const uint32_t bytes = ROWS * 8u;
      mbar_arrive_expect_tx(&s_bar, bytes * ncol + (start > 0 ? 16u * nk : 0u));
      for (int c = 0; c < nk; ++c) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(st + (size_t)c * ROWS)),
            "l"(p.key[c] + start), "r"(bytes), "r"(smem_u32(&s_bar))
            : "memory");
        if (start > 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                  smem_u32(s_prev2 + 2 * c)),
              "l"(p.key[c] + start - 2), "r"(smem_u32(&s_bar))
              : "memory");
      }
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(s_a)),
          "l"(p.a + start), "r"(bytes), "r"(smem_u32(&s_bar))
          : "memory");
      if constexpr (SRC == kSrcRaw)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(s_subk)),
            "l"(p.subk + start), "r"(bytes), "r"(smem_u32(&s_bar))
            : "memory");
    }
  }

  // warp 0 publishes "mbarrier initialised, copies issued, shared fields set" on named barrier 3;
  // the other warps pick it up only before they touch the fold tile, so their count starts now
  if (warp == 0 && fold_tile >= 0 && fold_tile < ntiles) named_arrive(3, kTileThreads);

  // ---- L2 prefetch: the key columns of tile count_tile + TK_TILE_PF (the count's loads, and ~lag
  //      tiles later the fold's copy, then hit L2) and the value columns of tile fold_tile +
  //      TK_TILE_PFV (close to their use, so they do not crowd L2); HBM sees these async requests ----
  if (TK_TILE_PF > 0 && p.mode == kTileSinglePass && warp == 1 && lane < ncol) {
    const long long pt = lane < nk ? count_tile + TK_TILE_PF : fold_tile + TK_TILE_PFV;
    if (pt >= 0 && pt < ntiles) {
      const long long ps = pt * TILE;
      const uint32_t bytes = (uint32_t)(min((long long)TILE, p.n - ps) * 8) & ~15u;
      const void* src = lane < nk ? (const void*)(p.key[lane] + ps)
                        : lane == nk ? (const void*)(p.a + ps)
                                     : (const void*)(p.subk + ps);
      if (bytes)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  }


  // ---- count the heads of tile count_tile straight from global memory, publish the aggregate ----
  // Each warp takes 128 consecutive rows; the previous row's key comes from the neighbouring lane
  // (lane 31 carries the row before the warp's first row, then the previous iteration's last row).
  // The order check (kept keys non-decreasing) lives here too, while the keys are in registers.
  if (count_tile >= 0 && count_tile < ntiles) {
    const long long cstart = count_tile * TILE;
    const int ccnt = (int)min((long long)TILE, p.n - cstart);
    const int wrow0 = warp * (TILE / kTileWarps);
    int heads = 0;
    constexpr int WROWS = TILE / kTileWarps;
    if (NK > 0 && WROWS % 64 == 0 && ccnt == TILE && p.bulk_ok) {
      // Full tile, 16-byte aligned columns: 16-byte loads of row pairs (2*lane, 2*lane+1) per
      // 64-row block; only the pair's first row needs a neighbour (lane-1's second row).
      constexpr int NB = WROWS / 64 > 0 ? WROWS / 64 : 1;
      constexpr int NKV = NK > 0 ? NK : 1;
      longlong2 v[NB][NKV];
      long long edge[NKV];
      const long long r0 = cstart + wrow0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < NKV; ++c) v[b][c] = TK_CNT_LD(reinterpret_cast<const longlong2*>(p.key[c] + r0 + 64 * b) + lane);
#pragma unroll
      for (int c = 0; c < NKV; ++c) edge[c] = (lane == 31 && r0 > 0) ? TK_CNT_LD(p.key[c] + r0 - 1) : 0;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        bool ne0 = false, ne1 = false;
#pragma unroll
        for (int c = 0; c < NKV; ++c) {
          const long long give = lane == 31 ? (b ? v[b - 1][c].y : edge[c]) : v[b][c].y;
          const long long pv = __shfl_sync(0xffffffffu, give, (lane + 31) & 31);  // every lane
          ne0 = ne0 || v[b][c].x != pv;
          ne1 = ne1 || v[b][c].y != v[b][c].x;
        }
        heads += (ne0 || r0 + 64 * b + 2 * lane == 0) + ne1;
      }
      heads = __reduce_add_sync(0xffffffffu, heads);
    } else {
    constexpr int CJ = TILE / kTileThreads;
    long long cur[CJ][NKR], edge[NKR];
#pragma unroll
    for (int j = 0; j < CJ; ++j) {  // every key load in flight at once
      const int rl = wrow0 + j * 32 + lane;
      const bool ok = rl < ccnt;
#pragma unroll
      for (int c = 0; c < NKR; ++c) {
        if (NK == 0 && c >= nk) break;
        cur[j][c] = ok ? TK_CNT_LD(p.key[c] + cstart + rl) : 0;
      }
    }
    {
      const bool ok = lane == 31 && wrow0 < ccnt && cstart + wrow0 > 0;
#pragma unroll
      for (int c = 0; c < NKR; ++c) {
        if (NK == 0 && c >= nk) break;
        edge[c] = ok ? TK_CNT_LD(p.key[c] + cstart + wrow0 - 1) : 0;
      }
    }
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      const int rl = wrow0 + j * 32 + lane;
      bool ne = false;
#pragma unroll
      for (int c = 0; c < NKR; ++c) {
        if (NK == 0 && c >= nk) break;
        const long long give = lane == 31 ? (j ? cur[j - 1][c] : edge[c]) : cur[j][c];
        const long long pv = __shfl_sync(0xffffffffu, give, (lane + 31) & 31);  // every lane
        ne = ne || cur[j][c] != pv;
      }
      heads += __popc(__ballot_sync(0xffffffffu, rl < ccnt && (ne || cstart + rl == 0)));
    }
    }
    if (lane == 0) atomicAdd(p.status + count_tile, (1ull << kStWarpShift) | (unsigned long long)heads);
    if (tid == 0) TKR(1);
  }
  if (fold_tile < 0 || fold_tile >= ntiles) return;
  if (warp != 0) named_bar(3, kTileThreads);
  const long long tile = s_tile;
  const long long start = tile * TILE;
  const int cnt = (int)min((long long)TILE, p.n - start);
  const int avail = (int)min((long long)ROWS, p.n - start);
  if (s_bulk) {
    mbar_wait(&s_bar, 0);
    if (tid == 0) TKR(2);
  } else {
    for (int r = tid; r < avail; r += kTileThreads) {
      for (int c = 0; c < nk; ++c) s_key[(size_t)c * ROWS + r] = p.key[c][start + r];
      s_a[r] = p.a[start + r];
      if constexpr (SRC == kSrcRaw) s_subk[r] = p.subk[start + r];
    }
    if (tid < nk && start > 0) s_prev2[2 * tid + 1] = p.key[tid][start - 1];
    __syncthreads();
  }

  // ---- head bitmask of the stage (key equality with the previous row) and the order check
  //      (kept keys must be non-decreasing: lexicographic compare, same loads) ----
  unsigned int hmask[ITER];
  bool unsorted = false;
#pragma unroll
  for (int j = 0; j < ITER; ++j) {  // branch-free: rows past the stage load a clamped row
    if (j * kTileThreads + warp * 32 >= ROWS) {  // warp-uniform: this warp's rows are past the stage
      hmask[j] = 0;
      continue;
    }
    const int r = j * kTileThreads + tid;
    const int rc = min(r, ROWS - 1);
    bool hd = false, less = false;
#pragma unroll
    for (int c = 0; c < NKR; ++c) {
      if (NK == 0 && c >= nk) break;
      const long long va = s_key[c * ROWS + rc];
      const long long vb = *(rc ? s_key + c * ROWS + rc - 1 : s_prev2 + 2 * c + 1);
      less = less || (!hd && va < vb);
      hd = hd || va != vb;
    }
    const bool first = r == 0 && start == 0;
    unsorted = unsorted || (less && !first && r < cnt);
    hd = r < avail && (hd || first);
    hmask[j] = __ballot_sync(0xffffffffu, hd);
    const int wi = j * (kTileThreads / 32) + warp;
    if (lane == 0 && wi < WORDS) s_head[wi] = hmask[j];
  }
  __syncthreads();
  // ---- every warp: popcount prefix of the head words (redundant per warp: no extra barrier);
  //      each head row records itself at its local id ----
  int agg, ptot;
  {
    const unsigned int hw = lane < WORDS ? s_head[lane] : 0u;
    int incl = __popc(hw);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = incl - __popc(hw);
    ptot = __shfl_sync(0xffffffffu, incl, 31);  // heads in the stage (tile + halo)
    // heads in the tile proper == the aggregate the counting block published
    agg = __shfl_sync(0xffffffffu, excl + __popc(hw & ((1u << (cnt & 31)) - 1u)), cnt >> 5);
    const unsigned int lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < ITER; ++j) {
      const int wi = j * (kTileThreads / 32) + warp;
      const int wex = __shfl_sync(0xffffffffu, excl, wi & 31);
      if ((hmask[j] >> lane) & 1u) s_row[wex + __popc(hmask[j] & lt)] = (short)(j * kTileThreads + tid);
    }
  }
  if (warp == 0 && lane == 0) {
    // ---- this tile's exclusive prefix (the scanner block published it ~lag tiles ago) ----
    unsigned long long excl = 0;
    if (!tile_wait_prefix(p.status, tile, (unsigned long long)agg, pre, &excl)) {
      tile_stall(p.ctr, 3, tile);
      excl = ~0ull;  // no output from this tile
    }
    s_base = excl;
    if (start + cnt == p.n) p.ctr->groups = excl + (unsigned long long)agg;
    TKR(3);
  }
  unsigned int flags = unsorted ? kFlagUnsorted : 0u;  // unsorted: rare, the host takes the sort path
  // ---- w = vals * x[subk] (all gathers in flight before any store) ----
  if constexpr (SRC == kSrcRaw) {
    double xv[ITER], av[ITER];
#pragma unroll
    for (int j = 0; j < ITER; ++j) {  // branch-free: rows past the stage gather x[0]
      if (j * kTileThreads + warp * 32 >= ROWS) {  // warp-uniform: past the stage
        xv[j] = av[j] = 0.0;
        continue;
      }
      const int r = j * kTileThreads + tid;
      const int rc = min(r, ROWS - 1);
      const long long idx = s_subk[rc];
      av[j] = s_a[rc];
      const bool bad = (unsigned long long)idx >= (unsigned long long)p.nx;
      if (bad && r < avail) flags |= kFlagIndex;
      xv[j] = __ldg(p.x + (bad ? 0 : idx));
    }
#pragma unroll
    for (int j = 0; j < ITER; ++j) {
      const int r = j * kTileThreads + tid;
      if (r < avail) s_a[r] = __dmul_rn(av[j], xv[j]);
    }
  }
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();  // w, the head rows and the base are ready
  if (tid == 0) {
    if (s_flags) atomicOr(&p.ctr->flags, s_flags);
    TKR(4);
  }
  if (s_base == ~0ull) return;  // watchdog: the call fails
  const long long base = (long long)s_base;
  // one group's output row: (kept key of its head row, folded value) at base + local id
  auto emit = [&](int li, int r, double v) {
    const long long g = base + li;
    p.out_vals[g] = v;
    if constexpr (SRC == kSrcLinKey) {
      long long lin = s_key[r];
      long long* o = p.out_subs + g * p.out_nk;
      for (int q = p.out_nk - 1; q >= 0; --q) {
        const long long dm = p.dims[q];
        if (p.lin_fast) {  // multiply + fix-up instead of a 64-bit division
          long long rem;
          lin = divmod_fast(lin, dm, p.inv_dims[q], &rem);
          o[q] = rem;
        } else {
          o[q] = lin % dm;
          lin /= dm;
        }
      }
    } else {
      if constexpr (NK == 2) {
        if (p.out_v2) {  // one 16-byte store of the key pair
          *reinterpret_cast<longlong2*>(p.out_subs + 2 * g) = make_longlong2(s_key[r], s_key[ROWS + r]);
          return;
        }
      }
#pragma unroll
      for (int c = 0; c < NKR; ++c) {
        if (NK == 0 && c >= nk) break;
        p.out_subs[g * p.out_nk + c] = s_key[c * ROWS + r];
      }
    }
  };

  // ---- fold and write every group headed in the tile that closes inside the stage, one group
  //      per thread, striped (consecutive lanes write consecutive output rows); a warp with
  //      nothing left exits, so the SM can start another tile while long folds run.  The last
  //      group is open (continues past the stage) iff the halo has no head and the stream goes
  //      on -- every thread knows that without a barrier. ----
  const int open_li = (agg > 0 && agg == ptot && start + avail < p.n) ? agg - 1 : -1;
  unsigned int zeros = 0;
  // with an open group (raw source) warp 0 starts its serial chain at once: warps 1-3 take the
  // striped folds (then produce the spill chunks)
  const bool w0_chain = TK_SPILL_W0FIRST && SRC == kSrcRaw && open_li >= 0;
  const int li0 = w0_chain ? (warp == 0 ? agg : tid - 32) : tid;
  const int lstep = w0_chain ? kTileThreads - 32 : kTileThreads;
  for (int li = li0; li < agg; li += lstep) {
    if (li == open_li) continue;
    const int r = s_row[li];
    const int end = li + 1 < ptot ? s_row[li + 1] : avail;
    const double v = fold_run(s_a, r + 1, end, s_a[r]);
    emit(li, r, v);
    zeros += v == 0.0;
  }
  zeros = __reduce_add_sync(0xffffffffu, zeros);
  if (lane == 0 && zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
  if (tid == 0) TKR(6);
  if (open_li < 0) return;
#ifdef TK_DIAG_NOSPILL  // diagnostics only: the open group is never finished (wrong output)
  return;
#endif
  if constexpr (SRC == kSrcRaw) {
    // ---- the group that runs past the halo, raw source: a producer/consumer ring.  Warps 1-3
    //      (done with their folds) produce chunk c = warp-1, warp+2, ...: 128 rows past the stage
    //      (L2-hot: the next tiles' CTAs read them), key check, w = val * x[subk] with the gather,
    //      into slot c % kSpillSlots.  A chunk is loaded only once its predecessor is known to
    //      continue the group (s_known), and into a slot warp 0 has finished (s_consumed).  Warp
    //      0's lane 0 folds its in-stage rows, then the slots in chunk order: a pure serial chain,
    //      the loads and gathers of later chunks in flight meanwhile. ----
    const int r0 = s_row[open_li];
    double* ring = reinterpret_cast<double*>(s_subk);
    constexpr int RW = 4, CH = 32 * RW;
    if (warp != 0) {
      long long gk[NKR];
#pragma unroll
      for (int c = 0; c < NKR; ++c)
        if (NK > 0 || c < nk) gk[c] = s_key[c * ROWS + r0];
      for (int c = warp - 1;; c += kTileWarps - 1) {
        int go = 1;
        [[maybe_unused]] unsigned int spins = 0;
        if (lane == 0) {
          while (true) {  // predecessor known to continue, and this chunk's slot consumed
            if (c > ld_vol(&s_last)) {
              go = 0;
              break;
            }
            // up to TK_SPILL_AHEAD chunks past the last one known to continue the group are
            // loaded speculatively (wasted L2 reads when the group ends sooner)
            if (ld_vol(&s_known) >= c - TK_SPILL_AHEAD + 1 && ld_vol(&s_consumed) >= c - kSpillSlots + 1) break;
#if TK_RING_WATCHDOG
            if (++spins == kSpinLimit) {
              tile_stall(p.ctr, 5, tile);
              st_vol(&s_last, -1);  // the consumer gives up too
              go = 0;
              break;
            }
#endif
            __nanosleep(TK_SPILL_NAP);
          }
        }
        if (!__shfl_sync(0xffffffffu, go, 0)) return;
        const long long pos = start + avail + (long long)c * CH;
        long long kv[RW][NKR], sk[RW];
        double av[RW];
#pragma unroll
        for (int j = 0; j < RW; ++j) {  // every load of the chunk in flight at once
          const long long row = pos + j * 32 + lane;
          const bool ok = row < p.n;
#pragma unroll
          for (int q = 0; q < NKR; ++q)
            if (NK > 0 || q < nk) kv[j][q] = ok ? __ldcg(p.key[q] + row) : 0;
          av[j] = ok ? __ldcg(p.a + row) : 0.0;
          sk[j] = ok ? __ldcg(p.subk + row) : 0;
        }
        int end = CH;
        double xv[RW];
#pragma unroll
        for (int j = 0; j < RW; ++j) {
          bool same = pos + j * 32 + lane < p.n;
#pragma unroll
          for (int q = 0; q < NKR; ++q)
            if (NK > 0 || q < nk) same = same && kv[j][q] == gk[q];
          const unsigned int m = __ballot_sync(0xffffffffu, !same);
          if (end == CH && m) end = j * 32 + __ffs(m) - 1;
          xv[j] = (unsigned long long)sk[j] < (unsigned long long)p.nx ? __ldg(p.x + sk[j]) : 0.0;
        }
        const bool last = end < CH || pos + CH >= p.n;
        if (lane == 0) {  // later chunks may start loading (or nothing past this one is needed)
          if (last) atomicMin(&s_last, c);
          else atomicMax(&s_known, c + 1);
        }
        double* slot = ring + (c % kSpillSlots) * CH;
#pragma unroll
        for (int j = 0; j < RW; ++j) slot[j * 32 + lane] = __dmul_rn(av[j], xv[j]);
        __syncwarp();
        __threadfence_block();
        if (lane == 0) {
          st_vol(&s_end[c % kSpillSlots], end);
          __threadfence_block();
          st_vol(&s_ready[c % kSpillSlots], c + 1);
        }
        if (last) return;
      }
    }
    if (lane != 0) return;
    double acc = fold_run(s_a, r0 + 1, avail, s_a[r0]);
    for (int c = 0;; ++c) {
      const int sl = c % kSpillSlots;
      [[maybe_unused]] unsigned int spins = 0;
      while (ld_vol(&s_ready[sl]) != c + 1) {
#if TK_RING_WATCHDOG
        if (ld_vol(&s_last) < 0 || ++spins == kSpinLimit) {  // a producer gave up: the call fails
          tile_stall(p.ctr, 6, tile);
          return;
        }
#endif
        __nanosleep(16);
      }
      __threadfence_block();
      const int end = ld_vol(&s_end[sl]);
      acc = fold_run(ring + sl * CH, 0, end, acc);
      __threadfence_block();
      st_vol(&s_consumed, c + 1);
      if (end < CH || start + avail + (long long)(c + 1) * CH >= p.n) break;  // the group ended here
    }
    long long k[NKR];
#pragma unroll
    for (int c = 0; c < NKR; ++c)
      if (NK > 0 || c < nk) k[c] = s_key[c * ROWS + r0];
    seg_emit<SRC>(p, base + open_li, k, acc);
    TKR(7);
    return;
  }
  if (warp != 0) return;

  // ---- the group that runs past the halo, finished by warp 0 alone: 128-row chunks (L2-hot: the
  //      next tiles' CTAs read them), w staged in the free subk column; the next chunk's loads are
  //      in flight while lane 0 folds the current one ----
  const int r0 = s_row[open_li];
  long long gk[NKR];
#pragma unroll
  for (int c = 0; c < NKR; ++c)
    if (NK > 0 || c < nk) gk[c] = s_key[c * ROWS + r0];
  double acc = 0.0;  // meaningful in lane 0, which does every fold of this group
  if (lane == 0) acc = fold_run(s_a, r0 + 1, avail, s_a[r0]);
  double* cb = SRC == kSrcRaw ? reinterpret_cast<double*>(s_subk) : s_val;
  constexpr int RW = 4, CH = 32 * RW;
  long long kv[RW][NKR], sk[RW];
  double av[RW];
  auto load_chunk = [&](long long pos) {
#pragma unroll
    for (int j = 0; j < RW; ++j) {  // every load of the chunk in flight at once
      const long long row = pos + j * 32 + lane;
      const bool ok = row < p.n;
#pragma unroll
      for (int c = 0; c < NKR; ++c)
        if (NK > 0 || c < nk) kv[j][c] = ok ? __ldcg(p.key[c] + row) : 0;
      av[j] = ok ? __ldcg(p.a + row) : 0.0;
      sk[j] = (SRC == kSrcRaw && ok) ? __ldcg(p.subk + row) : 0;
    }
  };
  long long pos = start + avail;
  load_chunk(pos);
  while (true) {
    int end = CH;
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      const int r = j * 32 + lane;
      bool same = pos + r < p.n;
#pragma unroll
      for (int c = 0; c < NKR; ++c)
        if (NK > 0 || c < nk) same = same && kv[j][c] == gk[c];
      double w = av[j];
      if constexpr (SRC == kSrcRaw)
        w = __dmul_rn(w, (unsigned long long)sk[j] < (unsigned long long)p.nx ? __ldg(p.x + sk[j]) : 0.0);
      cb[r] = w;
      const unsigned int m = __ballot_sync(0xffffffffu, !same);
      if (end == CH && m) end = j * 32 + __ffs(m) - 1;
    }
    __syncwarp();
    const bool more = end == CH && pos + CH < p.n;
    if (more) load_chunk(pos + CH);  // in flight during the fold below
    if (lane == 0) acc = fold_run(cb, 0, end, acc);
    __syncwarp();
    if (!more) break;
    pos += CH;
  }
  if (lane == 0) {
    long long k[NKR];
#pragma unroll
    for (int c = 0; c < NKR; ++c)
      if (NK > 0 || c < nk) k[c] = gk[c];
    seg_emit<SRC>(p, base + open_li, k, acc);
    TKR(7);
  }
}

// Order-independent prefix for the three-pass fallback: status[t] holds tile t's complete
// aggregate (kTileCountOnly); one CTA turns the words into inclusive prefixes (kStPre | prefix).
__global__ void __launch_bounds__(1024) scan_tile_status_kernel(unsigned long long* status, long long ntiles) {
  __shared__ unsigned long long s_sum[1024];
  const long long per = (ntiles + 1023) / 1024;
  const long long a = min(ntiles, (long long)threadIdx.x * per), b = min(ntiles, a + per);
  unsigned long long run = 0;
  for (long long t = a; t < b; ++t) run += status[t] & kStCntMask;
  s_sum[threadIdx.x] = run;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const unsigned long long v = threadIdx.x >= (unsigned)o ? s_sum[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_sum[threadIdx.x] += v;
    __syncthreads();
  }
  run = s_sum[threadIdx.x] - run;  // exclusive prefix of this thread's range
  for (long long t = a; t < b; ++t) {
    run += status[t] & kStCntMask;
    status[t] = kStPre | run;
  }
}

}  // namespace tk
