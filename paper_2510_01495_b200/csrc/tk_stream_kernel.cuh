// tk_stream_kernel.cuh -- the persistent streaming TTV kernel.
//
// Roles per CTA (cooperative launch, 1 CTA / SM, static round-robin tiles: CTA c handles
// tiles c, c+G, c+2G, ... so every role can compute its own tile sequence):
//   PRODUCER warp   : stage ring of STAGES slots; waits EMPTY[s], issues the TMA bulk copies of
//                     tile k into slot k % STAGES (or fills a partial tail tile itself), and
//                     publishes the previous occupant's chain-job count with a release store.
//   LOOKAHEAD warps : NLA warps, tile k handled by warp k % NLA as soon as FULL[s] fires:
//                     count the tile's group heads, publish the aggregate, decoupled look-back,
//                     base -> BASE[s].  They run ahead of the streamers by up to STAGES-1 tiles,
//                     so a base is normally ready before the streamers need it.
//   STREAMER warps  : w = vals * x[subk] (all gathers issued before any store), head bitmask,
//                     then groups striped over threads: a group that ends inside tile+halo
//                     within kShort rows is folded serially by one thread (__dadd_rn, row
//                     order: the reference's exact sequence, _ckernels.pyx:274-294) and written
//                     at base + local id once BASE[s] fires; longer / tile-crossing groups become
//                     per-tile chain jobs (no global atomics on this path).  Then EMPTY[s].
//   CHAIN warps     : take tiles by ticket, wait for the tile's published job list, fold each
//                     job's rows (L2-hot) in 256-row chunks: lane 0 folds from smem while the
//                     next chunk is in flight.
// Shared memory stays ~120 KB so L1 keeps the gathered vector x resident.
#pragma once

#include "tk_stream.cuh"

namespace tk {

constexpr int kLookWarps = 3;  // 20 warps total: 5 per SMSP x 96 registers = one SMSP register file
constexpr int kJobsPerTile = 16;  // 1 open group + TILE/(kShort+1) long closed groups (TILE <= 1024)
constexpr int kWarpsTotal = 1 + kLookWarps + kStreamWarps + kChainWarps;
constexpr int kThreadsV6 = kWarpsTotal * 32;

template <int TILE, int HALO, int STAGES>
constexpr size_t stream_smem_bytes(int ncol, int nk) {
  return ((size_t)ncol * (TILE + HALO) + 2 * nk) * 8 * STAGES + (size_t)kChainWarps * kChunk * 8;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_release_u64g(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int SRC, int NK, int TILE, int HALO, int STAGES, int LBD>
__global__ void __maxnreg__(96) ttv_stream_kernel(StreamParams sp) {  // 21 warps x 96 regs fit an SM
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int TWORDS = TILE / 32;
  constexpr int ITER = (ROWS + 255) / 256;
  constexpr int NSB = kStreamWarps * 32;
  constexpr int GPT = TILE / NSB;  // max groups per streamer thread (nheads <= TILE)
  constexpr int NKR = NK > 0 ? NK : kMaxKeep;
  static_assert(ROWS % 32 == 0 && TILE % 256 == 0 && TILE <= 1024 && TWORDS <= 32, "tile geometry");
  static_assert(1 + TILE / (kShort + 1) <= kJobsPerTile, "job slots per tile");
  const SegParams& p = sp.s;
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const size_t stage_words = (size_t)ncol * ROWS + 2 * nk;  // + [nk][2] previous-row words
  long long* stage0 = reinterpret_cast<long long*>(smem_raw);
  double* chain_buf = reinterpret_cast<double*>(stage0 + stage_words * STAGES);

  __shared__ __align__(8) uint64_t s_full[STAGES], s_empty[STAGES], s_based[STAGES];
  __shared__ unsigned long long s_base[STAGES];
  __shared__ unsigned long long s_jc[STAGES];  // (base << 8) | (njobs + 1) of the slot's tile
  __shared__ unsigned int s_head[WORDS];
  __shared__ int s_wpref[TWORDS + 1];
  __shared__ int s_njobs;
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 1);
      mbar_init(&s_based[s], 1);
    }
    s_flags = 0;
    s_njobs = 0;
  }
  __syncthreads();
  auto tile_of = [&](long long k) { return (long long)blockIdx.x + k * G; };

  // =========================================== producer ===========================================
  if (warp == 0) {
    for (long long k = 0;; ++k) {
      const long long tile = tile_of(k);
      const int s = (int)(k % STAGES);
      if (k >= STAGES) {
        mbar_wait(&s_empty[s], (unsigned)(((k / STAGES) - 1) & 1));
        // publish the chain-job list of the tile that just left slot s
        if (lane == 0) st_release_u64g(sp.jcount + tile_of(k - STAGES), s_jc[s]);
      }
      if (tile >= sp.ntiles) break;
      const long long start = tile * TILE;
      const long long avail = min((long long)ROWS, p.n - start);
      long long* st = stage0 + stage_words * s;
      if (p.bulk_ok && avail == ROWS) {
        if (lane == 0) {
          const uint32_t bytes = ROWS * 8u;
          mbar_arrive_expect_tx(&s_full[s], bytes * ncol + (start > 0 ? 16u * nk : 0u));
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
        }
      } else {  // partial / unaligned tile: plain loads by this warp
        for (int r = lane; r < avail; r += 32) {
          for (int c = 0; c < nk; ++c) st[(size_t)c * ROWS + r] = p.key[c][start + r];
          st[(size_t)nk * ROWS + r] = reinterpret_cast<const long long*>(p.a)[start + r];
          if constexpr (SRC == kSrcRaw) st[(size_t)(nk + 1) * ROWS + r] = p.subk[start + r];
        }
        if (lane < nk && start > 0) st[(size_t)ncol * ROWS + 2 * lane + 1] = p.key[lane][start - 1];
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_full[s]);
      }
    }
    return;
  }

  // ========================================= look-ahead scan =========================================
  if (warp <= kLookWarps) {
    const int me = warp - 1;
    for (long long k = me;; k += kLookWarps) {
      const long long tile = tile_of(k);
      if (tile >= sp.ntiles) break;
      const int s = (int)(k % STAGES);
      mbar_wait(&s_full[s], (unsigned)((k / STAGES) & 1));
      const long long* st = stage0 + stage_words * s;
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      // heads among rows [0, cnt): row r is a head if its key differs from row r-1's
      int agg = 0;
      for (int r = lane; r < cnt; r += 32) {
        bool head = (r == 0 && start == 0);
        if (!head) {
#pragma unroll
          for (int c = 0; c < NKR; ++c) {
            if (NK == 0 && c >= nk) break;
            const long long va = st[(size_t)c * ROWS + r];
            const long long vb = r ? st[(size_t)c * ROWS + r - 1] : st[(size_t)ncol * ROWS + 2 * c + 1];
            head = head || va != vb;
          }
        }
        agg += __popc(__ballot_sync(__activemask(), head)) * (lane == 0);
      }
      agg = __shfl_sync(0xffffffffu, agg, 0);
      lookback_publish_agg<LBD>(p.status, tile, (unsigned long long)agg);
      const unsigned long long excl = lookback_wide<LBD>(p.status, tile, (unsigned long long)agg);
      if (lane == 0) {
        s_base[s] = excl;
        if (start + cnt == p.n) p.ctr->groups = excl + (unsigned long long)agg;
        mbar_arrive(&s_based[s]);
      }
    }
    return;
  }

  // ============================================ streamers ============================================
  if (warp <= kLookWarps + kStreamWarps) {
    const int t = tid - (1 + kLookWarps) * 32;  // 0..NSB-1
    const int swarp = t >> 5;
    unsigned int flags = 0;
    for (long long k = 0;; ++k) {
      const long long tile = tile_of(k);
      if (tile >= sp.ntiles) break;
      const int s = (int)(k % STAGES);
      const unsigned int par = (unsigned)((k / STAGES) & 1);
      long long* st = stage0 + stage_words * s;
      long long* s_key = st;
      double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
      const long long* s_subk = st + (size_t)(nk + 1) * ROWS;
      const long long* s_prev2 = st + (size_t)ncol * ROWS;
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      const int avail = (int)min((long long)ROWS, p.n - start);
      TKP_START(t_m);
      mbar_wait(&s_full[s], par);
      if (t == 0) TKP_ADD(0, t_m);

      // ---- w = vals * x[subk]: every gather in flight before any store ----
      if constexpr (SRC == kSrcRaw) {
        double xv[ITER], av[ITER];
#pragma unroll
        for (int j = 0; j < ITER; ++j) {
          const int r = j * NSB + t;
          xv[j] = 0.0;
          av[j] = 0.0;
          if (r < avail) {
            const long long idx = s_subk[r];
            av[j] = s_a[r];
            if (idx < 0 || idx >= p.nx) flags |= kFlagIndex;
            else xv[j] = __ldg(p.x + idx);
          }
        }
#pragma unroll
        for (int j = 0; j < ITER; ++j) {
          const int r = j * NSB + t;
          if (r < avail) s_a[r] = __dmul_rn(av[j], xv[j]);
        }
      }
      // ---- head bitmask over tile + halo (striped rows) ----
#pragma unroll
      for (int j = 0; j < ITER; ++j) {
        const int r = j * NSB + t;
        bool head = false;
        if (r < avail) {
          int cmp = 0;
#pragma unroll
          for (int c = 0; c < NKR; ++c) {
            if (NK == 0 && c >= nk) break;
            const long long va = s_key[c * ROWS + r];
            const long long vb = r ? s_key[c * ROWS + r - 1] : s_prev2[2 * c + 1];
            if (va != vb) {
              cmp = va < vb ? -1 : 1;
              break;
            }
          }
          if (r == 0 && start == 0) cmp = 1;
          head = cmp != 0;
          if (cmp < 0 && r < cnt) flags |= kFlagUnsorted;
        }
        const unsigned int m = __ballot_sync(0xffffffffu, head);
        const int wi = j * kStreamWarps + swarp;
        if ((t & 31) == 0 && wi < WORDS) s_head[wi] = m;
      }
      named_bar(1, NSB);  // heads visible
      if (swarp == 0) {   // exclusive popcount prefix of the tile's words
        unsigned int w = 0;
        if (lane < TWORDS && lane * 32 < cnt) {
          w = s_head[lane];
          if (lane * 32 + 32 > cnt) w &= (1u << (cnt - lane * 32)) - 1u;
        }
        int incl = __popc(w);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (lane < TWORDS) s_wpref[lane] = incl - __popc(w);
        if (lane == 31) s_wpref[TWORDS] = incl;  // head count of the tile
      }
      named_bar(1, NSB);
      if (t == 0) TKP_ADD(1, t_m);
      TKP_START(t_f);

      // ---- groups striped over threads: fold short ones, queue the rest ----
      const int nheads = s_wpref[TWORDS];
      double gval[GPT];
      short grow[GPT];
#pragma unroll
      for (int m = 0; m < GPT; ++m) {
        const int li = t + m * NSB;
        grow[m] = -1;
        gval[m] = 0.0;
        if (li >= nheads) continue;
        // select: word holding the li-th head, then the bit inside it
        int lo = 0, hi = TWORDS - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_wpref[mid] <= li) lo = mid;
          else hi = mid - 1;
        }
        const unsigned int wd = s_head[lo];
        const int r = lo * 32 + (int)__fns(wd, 0, li - s_wpref[lo] + 1);
        int end = avail;
        {
          const int q1 = r + 1;
          int wi = q1 >> 5;
          unsigned int wb = (q1 < avail) ? (s_head[wi] & (0xffffffffu << (q1 & 31))) : 0u;
          while (wb == 0 && (wi + 1) * 32 < avail) wb = s_head[++wi];
          if (wb) end = min(avail, wi * 32 + __ffs(wb) - 1);
        }
        const bool open = end == avail && start + avail < p.n;
        if (!open && end - r <= kShort) {
          gval[m] = fold_run(s_a, r + 1, end, s_a[r]);
          grow[m] = (short)r;
        } else {
          const int j = atomicAdd(&s_njobs, 1);
          sp.jobs[tile * kJobsPerTile + j] = ((unsigned long long)r << 16) | (unsigned long long)li;
        }
      }
      if (t == 0) TKP_ADD(3, t_f);
      TKP_START(t_d);
      mbar_wait(&s_based[s], par);
      if (t == 0) TKP_ADD(4, t_d);
      TKP_START(t_o);
      const long long base = (long long)s_base[s];
      unsigned int zeros = 0;
#pragma unroll
      for (int m = 0; m < GPT; ++m) {
        const int r = grow[m];
        if (r < 0) continue;
        const long long g = base + t + m * NSB;
        p.out_vals[g] = gval[m];
        zeros += gval[m] == 0.0;
        if constexpr (SRC == kSrcLinKey) {
          long long lin = s_key[r];
          long long* o = p.out_subs + g * p.out_nk;
          for (int q = p.out_nk - 1; q >= 0; --q) {
            const long long dm = p.dims[q];
            o[q] = lin % dm;
            lin /= dm;
          }
        } else {
#pragma unroll
          for (int c = 0; c < NKR; ++c) {
            if (NK == 0 && c >= nk) break;
            p.out_subs[g * p.out_nk + c] = s_key[c * ROWS + r];
          }
        }
      }
      if (zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
      named_bar(1, NSB);  // slot s consumed, job list complete
      if (t == 0) {
        s_jc[s] = ((unsigned long long)base << 8) | (unsigned long long)(s_njobs + 1);
        s_njobs = 0;
        mbar_arrive(&s_empty[s]);
        TKP_ADD(5, t_o);
        TKP_COUNT(7, 1);
      }
    }
    if (flags) atomicOr(&s_flags, flags);
    named_bar(1, NSB);
    if (t == 0) {
      if (s_flags) atomicOr(&p.ctr->flags, s_flags);
      // the producer publishes each tile's job list when its slot is recycled; the last
      // STAGES tiles of this CTA are never recycled, so publish them here
      const long long kdone = (sp.ntiles - blockIdx.x + G - 1) / G;  // tiles of this CTA
      for (long long k = max(0LL, kdone - STAGES); k < kdone; ++k)
        st_release_u64g(sp.jcount + tile_of(k), s_jc[(int)(k % STAGES)]);
    }
    return;
  }

  // ============================================= chain warps =============================================
  double* cbuf = chain_buf + (size_t)(warp - (1 + kLookWarps + kStreamWarps)) * kChunk;
  while (true) {
    long long tile = 0;
    unsigned long long jc = 0;
    TKP_START(t_idle);
    if (lane == 0) {
      tile = (long long)atomicAdd(&p.ctr->tile_ticket, 1u);
      if (tile < sp.ntiles)
        while ((jc = ld_relaxed_u64(sp.jcount + tile)) == 0) __nanosleep(256);
    }
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (lane == 0) TKP_ADD(10, t_idle);
    if (tile >= sp.ntiles) break;
    jc = __shfl_sync(0xffffffffu, jc, 0);
    const int njobs = (int)(jc & 0xff) - 1;
    const long long base = (long long)(jc >> 8);
    for (int jb = 0; jb < njobs; ++jb) {
      TKP_START(t_busy);
      const unsigned long long job = ld_relaxed_u64(sp.jobs + tile * kJobsPerTile + jb);
      const long long start = tile * TILE + (long long)(job >> 16);
      const long long g = base + (long long)(job & 0xffff);

      long long gk[NKR];
      double acc = 0.0;
      bool first = true;
      long long pos = start;
      long long kv[8][NKR];
      double av[8];
      long long sk[8];
      auto load_chunk = [&](long long b0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const long long r = b0 + q * 32 + lane;
          const bool ok = r < p.n;
#pragma unroll
          for (int c = 0; c < NKR; ++c)
            if (NK > 0 || c < nk) kv[q][c] = ok ? __ldcg(p.key[c] + r) : 0;
          av[q] = ok ? __ldcg(p.a + r) : 0.0;
          if constexpr (SRC == kSrcRaw) sk[q] = ok ? __ldcg(p.subk + r) : 0;
        }
      };
      load_chunk(pos);
#pragma unroll
      for (int c = 0; c < NKR; ++c) gk[c] = __shfl_sync(0xffffffffu, kv[0][c], 0);  // the group's key
      while (true) {
        double xv[8];
        if constexpr (SRC == kSrcRaw) {
#pragma unroll
          for (int q = 0; q < 8; ++q) xv[q] = (sk[q] < 0 || sk[q] >= p.nx) ? 0.0 : __ldg(p.x + sk[q]);
        }
        int end = kChunk;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          bool same = pos + q * 32 + lane < p.n;
#pragma unroll
          for (int c = 0; c < NKR; ++c)
            if (NK > 0 || c < nk) same = same && kv[q][c] == gk[c];
          cbuf[q * 32 + lane] = (SRC == kSrcRaw) ? __dmul_rn(av[q], xv[q]) : av[q];
          const unsigned int mm = __ballot_sync(0xffffffffu, !same);
          if (mm && end == kChunk) end = q * 32 + __ffs(mm) - 1;
        }
        __syncwarp();
        const bool more = end == kChunk;
        if (more) load_chunk(pos + kChunk);  // in flight while lane 0 folds
        if (lane == 0) {
          int j = 0;
          if (first) {
            acc = cbuf[0];
            j = 1;
          }
          acc = fold_run(cbuf, j, end, acc);
        }
        first = false;
        __syncwarp();
        if (!more) {
          if (lane == 0) TKP_COUNT(13, pos - start + end);
          break;
        }
        pos += kChunk;
      }
      if (lane == 0) {
        seg_emit<SRC>(p, g, gk, acc);
        TKP_ADD(11, t_busy);
        TKP_COUNT(12, 1);
      }
    }
  }
}

}  // namespace tk
