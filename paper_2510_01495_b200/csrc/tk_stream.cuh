// tk_stream.cuh -- persistent, warp-specialised streaming kernel for sparse-result TTV.
//
// One CTA per SM slot (cooperative launch: every CTA is co-resident), 12 warps:
//   * 8 STREAMER warps run a STAGES-deep TMA pipeline over tiles of TILE rows (+HALO
//     look-ahead rows).  Per tile: w = vals*x[subk] (RN multiply), head flags of the
//     kept-key stream, popcount prefix + decoupled look-back over head counts -> every
//     group's output slot.  Groups whose head is in the tile and that end inside
//     tile+halo with at most kShort rows are folded by the thread owning the head, in row
//     order with __dadd_rn (the reference's exact sequence, _ckernels.pyx:274-294).
//   * every longer / tile-spanning group becomes a job (output slot, first row) in a
//     device work queue, drained by 4 CHAIN warps per CTA: the warp streams the group's
//     rows (L2-hot: the streamers just pulled them) in coalesced 256-row chunks, lane 0
//     folds them serially from shared memory while the next chunk's loads are in flight.
// A long group therefore never stalls a tile: the serial chains (one DADD latency per row)
// run concurrently with the stream on warps of their own.
#pragma once

#include "tk_ttv_kernels.cuh"

namespace tk {

struct StreamJob {
  long long g;
  long long start;
};

struct StreamParams {
  SegParams s;              // stream description + outputs + status/ctr
  StreamJob* jobs;          // capacity job_cap
  unsigned int* job_ready;  // zeroed
  long long job_cap;
  long long ntiles;
};

constexpr int kStreamWarps = 8;
constexpr int kChainWarps = 4;
constexpr int kStreamThreads = (kStreamWarps + kChainWarps) * 32;
constexpr int kShort = 64;       // in-thread fold limit (rows)
constexpr int kChunk = 256;      // chain-warp chunk (8 rows per lane)

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

// Serial fold of s_a[r0+1 .. end) onto acc (independent loads, dependent adds).
__device__ __forceinline__ double fold_run(const double* s_a, int j, int end, double acc) {
  for (; j + 4 <= end; j += 4) {
    const double v0 = s_a[j], v1 = s_a[j + 1], v2 = s_a[j + 2], v3 = s_a[j + 3];
    acc = __dadd_rn(acc, v0);
    acc = __dadd_rn(acc, v1);
    acc = __dadd_rn(acc, v2);
    acc = __dadd_rn(acc, v3);
  }
  for (; j < end; ++j) acc = __dadd_rn(acc, s_a[j]);
  return acc;
}

template <int SRC, int NK, int TILE, int HALO, int STAGES>
__global__ void __launch_bounds__(kStreamThreads, 1) ttv_stream_kernel(StreamParams sp) {
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int ITER = (ROWS + 255) / 256;
  constexpr int OWN = TILE / 256;  // rows owned per streamer thread (blocked)
  static_assert(ROWS % 32 == 0 && TILE % 256 == 0, "tile geometry");
  const SegParams& p = sp.s;
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // stage layout: [ncol][ROWS] 8-byte words, then [nk][2] previous-row words
  const size_t stage_words = (size_t)ncol * ROWS + 2 * nk;
  long long* stage0 = reinterpret_cast<long long*>(smem_raw);
  double* chain_buf = reinterpret_cast<double*>(stage0 + stage_words * STAGES);

  __shared__ __align__(8) uint64_t s_full[STAGES];
  __shared__ long long s_stage_tile[STAGES];
  __shared__ int s_stage_bulk[STAGES];
  __shared__ unsigned int s_head[WORDS];
  __shared__ int s_wpref[WORDS];
  __shared__ unsigned long long s_base;
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&s_full[s], 1);
    s_flags = 0;
  }
  __syncthreads();

  if (warp < kStreamWarps) {
    // =============================== streamer warps ===============================
    auto acquire_issue = [&](int s) {  // thread 0 only
      const unsigned int t = atomicAdd(&p.ctr->tile_ticket, 1u);
      if ((long long)t >= sp.ntiles) {
        s_stage_tile[s] = -1;
        return;
      }
      s_stage_tile[s] = t;
      const long long start = (long long)t * TILE;
      const long long avail = min((long long)ROWS, p.n - start);
      long long* st = stage0 + stage_words * s;
      const bool bulk = p.bulk_ok && avail == ROWS;
      s_stage_bulk[s] = bulk;
      if (!bulk) return;  // filled cooperatively by the streamers
      const uint32_t bytes = ROWS * 8u;
      const uint32_t total = bytes * ncol + (start > 0 ? 16u * nk : 0u);
      mbar_arrive_expect_tx(&s_full[s], total);
      const uint64_t pol = 0;  // default (evict-normal): chain warps re-read spans from L2
      (void)pol;
      for (int c = 0; c < nk; ++c) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(st + (size_t)c * ROWS)),
            "l"(p.key[c] + start), "r"(bytes), "r"(smem_u32(&s_full[s]))
            : "memory");
        if (start > 0)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                  smem_u32(st + (size_t)ncol * ROWS + 2 * c)),
              "l"(p.key[c] + start - 2), "r"(smem_u32(&s_full[s]))
              : "memory");
      }
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(st + (size_t)nk * ROWS)),
          "l"(p.a + start), "r"(bytes), "r"(smem_u32(&s_full[s]))
          : "memory");
      if constexpr (SRC == kSrcRaw)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(st + (size_t)(nk + 1) * ROWS)),
            "l"(p.subk + start), "r"(bytes), "r"(smem_u32(&s_full[s]))
            : "memory");
    };

    if (tid == 0)
      for (int s = 0; s < STAGES; ++s) acquire_issue(s);
    unsigned int phase = 0;  // bit s = parity of stage s
    int s = 0;
    while (true) {
      named_bar(1, kStreamWarps * 32);
      const long long tile = s_stage_tile[s];
      if (tile < 0) break;
      long long* st = stage0 + stage_words * s;
      long long* s_key = st;
      double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
      const long long* s_subk = st + (size_t)(nk + 1) * ROWS;
      const long long* s_prev2 = st + (size_t)ncol * ROWS;  // [c][2]: rows start-2, start-1
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      const int avail = (int)min((long long)ROWS, p.n - start);
      if (s_stage_bulk[s]) {
        mbar_wait(&s_full[s], (phase >> s) & 1u);
        phase ^= 1u << s;
      } else {
        for (int r = tid; r < avail; r += kStreamWarps * 32) {
          for (int c = 0; c < nk; ++c) s_key[c * ROWS + r] = p.key[c][start + r];
          s_a[r] = p.a[start + r];
          if constexpr (SRC == kSrcRaw) st[(size_t)(nk + 1) * ROWS + r] = p.subk[start + r];
        }
        if (tid < nk && start > 0) st[(size_t)ncol * ROWS + 2 * tid + 1] = p.key[tid][start - 1];
        named_bar(1, kStreamWarps * 32);
      }

      // ---- w and head flags (striped rows: conflict-free shared memory) ----
      unsigned int flags = 0;
#pragma unroll
      for (int j = 0; j < ITER; ++j) {
        const int r = j * 256 + tid;
        bool head = false;
        if (r < avail) {
          if constexpr (SRC == kSrcRaw) {
            const long long idx = s_subk[r];
            double w = 0.0;
            if (idx < 0 || idx >= p.nx) flags |= kFlagIndex;
            else w = __dmul_rn(s_a[r], __ldg(p.x + idx));
            s_a[r] = w;
          }
          int cmp = 0;
          if (r == 0) {
            if (start == 0) cmp = 1;
            else {
#pragma unroll
              for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
                if (NK == 0 && c >= nk) break;
                const long long va = s_key[c * ROWS], vb = s_prev2[2 * c + 1];
                if (va != vb) { cmp = va < vb ? -1 : 1; break; }
              }
            }
          } else {
#pragma unroll
            for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
              if (NK == 0 && c >= nk) break;
              const long long va = s_key[c * ROWS + r], vb = s_key[c * ROWS + r - 1];
              if (va != vb) { cmp = va < vb ? -1 : 1; break; }
            }
          }
          head = cmp != 0;
          if (cmp < 0 && r < cnt) flags |= kFlagUnsorted;
        }
        const unsigned int m = __ballot_sync(0xffffffffu, head);
        const int wi = j * 8 + warp;
        if (lane == 0 && wi < WORDS) s_head[wi] = m;
      }
      if (flags) atomicOr(&s_flags, flags);
      named_bar(1, kStreamWarps * 32);

      // ---- group ids: popcount prefix over the tile's words + decoupled look-back ----
      if (warp == 0) {
        int mine = 0;
        int cw[(WORDS + 31) / 32];
#pragma unroll
        for (int i = 0; i < (WORDS + 31) / 32; ++i) {
          const int wi = lane * ((WORDS + 31) / 32) + i;
          unsigned int word = 0;
          if (wi < WORDS && wi * 32 < cnt) {
            word = s_head[wi];
            if (wi * 32 + 32 > cnt) word &= (1u << (cnt - wi * 32)) - 1u;
          }
          cw[i] = __popc(word);
          mine += cw[i];
        }
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        int run = incl - mine;
#pragma unroll
        for (int i = 0; i < (WORDS + 31) / 32; ++i) {
          const int wi = lane * ((WORDS + 31) / 32) + i;
          if (wi < WORDS) s_wpref[wi] = run;
          run += cw[i];
        }
        const unsigned long long agg = (unsigned long long)__shfl_sync(0xffffffffu, incl, 31);
        const unsigned long long excl = lookback_exclusive(p.status, tile, agg);
        if (lane == 0) {
          s_base = excl;
          if (start + cnt == p.n) p.ctr->groups = excl + agg;
        }
      }
      named_bar(1, kStreamWarps * 32);

      // ---- folds of short groups; long / spanning groups become chain jobs ----
      const unsigned long long base = s_base;
      const int r0 = tid * OWN;
#pragma unroll 1
      for (int i = 0; i < OWN; ++i) {
        const int r = r0 + i;
        if (r >= cnt) break;
        const unsigned int word = s_head[r >> 5];
        if (!((word >> (r & 31)) & 1u)) continue;
        const long long g = (long long)(base + s_wpref[r >> 5] + __popc(word & ((1u << (r & 31)) - 1u)));
        // end = next head after r within the stage (or `avail`)
        int end = avail;
        {
          int q = r + 1;
          int wi = q >> 5;
          unsigned int wb = (q < avail && wi < WORDS) ? (s_head[wi] & (0xffffffffu << (q & 31))) : 0u;
          while (wb == 0 && (wi + 1) * 32 < avail) wb = s_head[++wi];
          if (wb) end = min(avail, wi * 32 + __ffs(wb) - 1);
        }
        const bool open = end == avail && start + avail < p.n;
        if (!open && end - r <= kShort) {
          const double acc = fold_run(s_a, r + 1, end, s_a[r]);
          long long kv[kMaxKeep];
          for (int c = 0; c < nk; ++c) kv[c] = s_key[c * ROWS + r];
          seg_emit<SRC>(p, g, kv, acc);
        } else {
          const unsigned long long slot = atomicAdd(&p.ctr->q_tail, 1ull);
          sp.jobs[slot] = StreamJob{g, start + r};
          __threadfence();
          st_release_u32(sp.job_ready + slot, 1u);
        }
      }
      named_bar(1, kStreamWarps * 32);  // stage s consumed
      if (tid == 0) acquire_issue(s);
      s = (s + 1) % STAGES;
    }
    if (tid == 0) {
      if (s_flags) atomicOr(&p.ctr->flags, s_flags);
      __threadfence();
      atomicAdd(&p.ctr->streamers_done, 1u);
    }
    return;
  }

  // ================================ chain warps ==================================
  double* cbuf = chain_buf + (size_t)(warp - kStreamWarps) * kChunk;
  while (true) {
    long long slot = -1;
    if (lane == 0) {
      const unsigned long long t = atomicAdd(&p.ctr->q_head, 1ull);
      while (true) {
        if (t < ld_acquire_u64(&p.ctr->q_tail)) {
          while (!ld_acquire_u32(sp.job_ready + t)) __nanosleep(32);
          slot = (long long)t;
          break;
        }
        if (ld_acquire_u32(&p.ctr->streamers_done) == gridDim.x) {
          if (t < ld_acquire_u64(&p.ctr->q_tail)) continue;
          break;
        }
        __nanosleep(256);
      }
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (slot < 0) break;
    long long g = 0, start = 0;
    if (lane == 0) {
      g = __ldcg(&sp.jobs[slot].g);
      start = __ldcg(&sp.jobs[slot].start);
    }
    g = __shfl_sync(0xffffffffu, g, 0);
    start = __shfl_sync(0xffffffffu, start, 0);
    long long gk[kMaxKeep];
    for (int c = 0; c < nk; ++c) gk[c] = __ldcg(p.key[c] + start);

    double acc = 0.0;
    bool first = true;
    long long pos = start;
    // chunk registers: 8 rows per lane (row = pos + i*32 + lane)
    double av[8];
    long long sk[8];
    bool same[8];
    auto load_chunk = [&](long long base) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const long long r = base + i * 32 + lane;
        same[i] = r < p.n && key_eq_global<SRC, NK>(p, nk, r, gk);
        av[i] = r < p.n ? __ldcg(p.a + r) : 0.0;
        if constexpr (SRC == kSrcRaw) sk[i] = r < p.n ? __ldcg(p.subk + r) : 0;
      }
    };
    load_chunk(pos);
    while (true) {
      int end = kChunk;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double w = av[i];
        if constexpr (SRC == kSrcRaw) w = (sk[i] < 0 || sk[i] >= p.nx) ? 0.0 : __dmul_rn(w, __ldg(p.x + sk[i]));
        cbuf[i * 32 + lane] = w;
        const unsigned int mm = __ballot_sync(0xffffffffu, !same[i]);
        if (mm && end == kChunk) end = i * 32 + __ffs(mm) - 1;
      }
      __syncwarp();
      const bool more = end == kChunk;
      if (more) load_chunk(pos + kChunk);  // in flight while lane 0 folds
      if (lane == 0) {
        int j = 0;
        if (first && end > 0) {
          acc = cbuf[0];
          j = 1;
        }
        acc = fold_run(cbuf, j, end, acc);
      }
      first = false;
      __syncwarp();
      if (!more) break;
      pos += kChunk;
    }
    if (lane == 0) seg_emit<SRC>(p, g, gk, acc);
  }
}

}  // namespace tk
