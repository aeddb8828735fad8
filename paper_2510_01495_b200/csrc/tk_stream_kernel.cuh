// tk_stream_kernel.cuh -- the persistent streaming TTV kernel.
//
// Cooperative launch, 1 CTA per SM, static round-robin tiles (CTA c: tiles c, c+G, c+2G, ...;
// the CTA-local index k names them), 20 warps in five roles:
//   PRODUCER  (1 warp)  : STAGES-slot TMA ring (cp.async.bulk of every column of tile k into slot
//                         k % STAGES; partial tail tiles by plain loads); recycles a slot once its
//                         pipe is done and publishes that tile's chain-job list (release store).
//   LOOKAHEAD (kLookWarps) : tile k -> warp k % kLookWarps, up to RING tiles ahead of the pipes:
//                         reads the tile's KEY columns straight from global memory (this also pulls
//                         them into L2 for the TMA), counts group heads, publishes the tile aggregate
//                         and runs the decoupled look-back -> base ring.  Bases are ready long before
//                         the pipes need them, so the look-back latency never stalls the stream.
//   PIPES     (2 x 4 warps) : pipe k % 2 processes tile k: w = vals * x[subk] (gathers issued before
//                         any store), head bitmask, then each group headed in the tile is
//                           short  (<= kShortFold rows, ends in tile+halo): folded at once by a thread;
//                           medium (<= kShort rows, ends in tile+halo): queued in smem and then folded
//                                   one group per lane, packed into as few warps as possible;
//                           long / open (crosses the halo): a chain job (per-tile slot, no atomics).
//                         Every fold is serial in row order with __dadd_rn -- the reference's exact
//                         operation sequence (_ckernels.pyx:274-294) -- and outputs go to base + id.
//   CHAIN     (kChainWarps) : take tiles by ticket, wait for the published job list, stream each
//                         job's rows (L2-hot) in 256-row chunks, lane 0 folds while the next chunk is
//                         in flight.
// Shared memory ~150 KB, leaving L1 room for the gathered vector x.
#pragma once

#include "tk_stream.cuh"

namespace tk {

constexpr int kLookWarps = 5;
constexpr int kPipes = 2;
constexpr int kPipeWarps = 4;
constexpr int kChainW = 5;
constexpr int kWarpsTotal = 2 + kLookWarps + kPipes * kPipeWarps + kChainW;  // 20
constexpr int kThreadsV6 = kWarpsTotal * 32;
constexpr int kRing = 12;        // look-ahead lead (tiles) / base ring slots
constexpr int kShortFold = 8;    // in-place fold limit (rows) -- bounded SIMT divergence
constexpr int kMaxMedium = 128;  // medium groups per tile (> TILE / (kShortFold + 1))
constexpr int kJobsPerTile = 16; // 1 open group + TILE/(kShort+1) long closed groups (TILE <= 1024)
static_assert(kWarpsTotal == 20, "5 warps per SMSP x 96 registers");

template <int TILE, int HALO, int STAGES>
constexpr size_t stream_smem_bytes(int ncol, int nk) {
  return ((size_t)ncol * (TILE + HALO) + 2 * nk) * 8 * STAGES + (size_t)kChainW * kChunk * 8 +
         (size_t)kPipes * kMaxMedium * 8;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void st_release_u64g(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int SRC, int NK, int TILE, int HALO, int STAGES, int LBD>
__global__ void __maxnreg__(96) ttv_stream_kernel(StreamParams sp) {  // 20 warps x 96 regs = one SM
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int TWORDS = TILE / 32;
  constexpr int NPT = kPipeWarps * 32;       // threads per pipe
  constexpr int ITER = (ROWS + NPT - 1) / NPT;
  constexpr int GPT = TILE / NPT;            // group rounds per pipe thread (nheads <= TILE)
  constexpr int NKR = NK > 0 ? NK : kMaxKeep;
  constexpr int LPR = TILE / 32;             // look-ahead rows per lane
  static_assert(ROWS % 32 == 0 && TILE % NPT == 0 && TILE <= 1024 && TWORDS <= 32, "tile geometry");
  static_assert(1 + TILE / (kShort + 1) <= kJobsPerTile && TILE / (kShortFold + 1) < kMaxMedium, "slots");
  static_assert(STAGES >= kPipes + 1, "a slot per pipe plus one in flight");
  const SegParams& p = sp.s;
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const size_t stage_words = (size_t)ncol * ROWS + 2 * nk;  // + [nk][2] previous-row words
  long long* stage0 = reinterpret_cast<long long*>(smem_raw);
  double* chain_buf = reinterpret_cast<double*>(stage0 + stage_words * STAGES);
  unsigned long long* s_med_all = reinterpret_cast<unsigned long long*>(chain_buf + kChainW * kChunk);

  __shared__ __align__(8) uint64_t s_full[STAGES], s_empty[STAGES], s_based[kRing], s_tq[kRing];
  __shared__ unsigned long long s_base[kRing];
  __shared__ long long s_tileq[kRing];             // tile id of CTA-local index k (-1: no more)
  __shared__ volatile long long s_ack[kRing];      // CTA-local tile whose base slot was consumed
  __shared__ unsigned long long s_jc[STAGES];       // (base << 8) | (njobs + 1) of the slot's tile
  __shared__ unsigned int s_head[kPipes][WORDS];
  __shared__ int s_wpref[kPipes][TWORDS + 1];
  __shared__ int s_njobs[kPipes], s_nmed[kPipes];
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 1);
    }
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&s_based[s], 1);
      mbar_init(&s_tq[s], 1);
      s_ack[s] = -1;
    }
    for (int q = 0; q < kPipes; ++q) s_njobs[q] = s_nmed[q] = 0;
    s_flags = 0;
  }
  __syncthreads();
  (void)G;
  // tile id of CTA-local index k, once the ticketer has published it
  auto tile_at = [&](long long k) {
    mbar_wait(&s_tq[k % kRing], (unsigned)((k / kRing) & 1));
    return s_tileq[k % kRing];
  };

  // ============================================ ticketer ============================================
  // Hands tiles to this CTA in global processing order (dynamic: a slow CTA simply takes fewer),
  // at most kRing ahead of the pipes.  After the first exhausted ticket it publishes enough -1
  // sentinels for every role to stop.
  if (warp == 0) {
    if (lane == 0) {
      long long kend = -1;
      for (long long k = 0;; ++k) {
        const int slot = (int)(k % kRing);
        if (kend >= 0 && k > kend + kLookWarps) break;
        if (k >= kRing)
          while (s_ack[slot] != k - kRing) __nanosleep(64);  // the pipes are done with k - kRing
        long long tile = -1;
        if (kend < 0) {
          tile = (long long)atomicAdd(&p.ctr->grab_ticket, 1u);
          if (tile >= sp.ntiles) {
            tile = -1;
            kend = k;
          }
        }
        s_tileq[slot] = tile;
        mbar_arrive(&s_tq[slot]);
      }
    }
    return;
  }

  // =========================================== producer ===========================================
  if (warp == 1) {
    // iteration k loads tile k and publishes the job list of tile k - STAGES (whose slot it reuses);
    // after the last tile, STAGES more iterations only drain
    long long kend = 1LL << 62;
    long long prev_tiles[STAGES];
#pragma unroll
    for (int q = 0; q < STAGES; ++q) prev_tiles[q] = -1;
    for (long long k = 0; k < kend + STAGES; ++k) {
      const int s = (int)(k % STAGES);
      if (k >= STAGES) {
        mbar_wait(&s_empty[s], (unsigned)(((k / STAGES) - 1) & 1));
        long long pt = -1;
#pragma unroll
        for (int q = 0; q < STAGES; ++q)
          if (q == s) pt = prev_tiles[q];
        if (lane == 0) st_release_u64g(sp.jcount + pt, s_jc[s]);
      }
      if (k >= kend) continue;
      const long long tile = tile_at(k);
      if (tile < 0) {
        kend = k;
        continue;
      }
#pragma unroll
      for (int q = 0; q < STAGES; ++q)
        if (q == s) prev_tiles[q] = tile;
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
  if (warp <= 1 + kLookWarps) {
    const int me = warp - 2;
    for (long long k = me;; k += kLookWarps) {
      const long long tile = tile_at(k);
      if (tile < 0) break;
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      // head flags of rows r = j*32 + lane (j < LPR), key columns read from global / L2
      unsigned int hb = 0;  // bit j: row j*32+lane is a head
#pragma unroll 1
      for (int c = 0; c < NKR; ++c) {
        if (NK == 0 && c >= nk) break;
        const long long* col = p.key[c] + start;
        long long prevcarry = (start > 0) ? __ldcg(col - 1) : 0;  // row start-1 (lane 0's predecessor)
        constexpr int CH = LPR < 16 ? LPR : 16;  // rows per lane in flight (register budget)
#pragma unroll 1
        for (int j0 = 0; j0 < LPR; j0 += CH) {
          long long v[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int r = (j0 + j) * 32 + lane;
            v[j] = r < cnt ? __ldcg(col + r) : 0;
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const long long up = __shfl_up_sync(0xffffffffu, v[j], 1);
            const long long last = __shfl_sync(0xffffffffu, v[j], 31);
            const long long prev = lane == 0 ? prevcarry : up;
            if (v[j] != prev) hb |= 1u << (j0 + j);
            prevcarry = last;
          }
        }
      }
      if (start == 0 && lane == 0) hb |= 1u;
      int agg = 0;
#pragma unroll
      for (int j = 0; j < LPR; ++j) {
        const bool head = ((hb >> j) & 1u) && (j * 32 + lane < cnt);
        agg += __popc(__ballot_sync(0xffffffffu, head));
      }
      lookback_publish_agg<LBD>(p.status, tile, (unsigned long long)agg);
      const unsigned long long excl = lookback_wide<LBD>(p.status, tile, (unsigned long long)agg);
      const int slot = (int)(k % kRing);
      if (lane == 0) {  // (slot k % kRing is free: the ticketer waited for its ack before issuing k)
        if (start + cnt == p.n) p.ctr->groups = excl + (unsigned long long)agg;
        s_base[slot] = excl;
        mbar_arrive(&s_based[slot]);
      }
      __syncwarp();
    }
    return;
  }

  // ============================================== pipes ==============================================
  if (warp <= 1 + kLookWarps + kPipes * kPipeWarps) {
    const int pw = warp - 2 - kLookWarps;  // 0 .. kPipes*kPipeWarps-1
    const int pipe = pw / kPipeWarps;
    const int t = (pw % kPipeWarps) * 32 + lane;  // thread within pipe
    const int pwarp = t >> 5;
    const int bar_id = 1 + pipe;
    unsigned int* head = s_head[pipe];
    int* wpref = s_wpref[pipe];
    unsigned long long* med = s_med_all + pipe * kMaxMedium;
    unsigned int flags = 0;
    for (long long k = pipe;; k += kPipes) {
      const long long tile = tile_at(k);
      if (tile < 0) break;
      const int s = (int)(k % STAGES);
      long long* st = stage0 + stage_words * s;
      long long* s_key = st;
      double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
      const long long* s_subk = st + (size_t)(nk + 1) * ROWS;
      const long long* s_prev2 = st + (size_t)ncol * ROWS;
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      const int avail = (int)min((long long)ROWS, p.n - start);
      TKP_START(t_m);
      mbar_wait(&s_full[s], (unsigned)((k / STAGES) & 1));
      if (t == 0) TKP_ADD(0, t_m);

      // ---- w = vals * x[subk]: every gather in flight before any store ----
      if constexpr (SRC == kSrcRaw) {
        double xv[ITER], av[ITER];
#pragma unroll
        for (int j = 0; j < ITER; ++j) {
          const int r = j * NPT + t;
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
          const int r = j * NPT + t;
          if (r < avail) s_a[r] = __dmul_rn(av[j], xv[j]);
        }
      }
      // ---- head bitmask over tile + halo (striped rows) ----
#pragma unroll
      for (int j = 0; j < ITER; ++j) {
        const int r = j * NPT + t;
        bool hd = false;
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
          hd = cmp != 0;
          if (cmp < 0 && r < cnt) flags |= kFlagUnsorted;
        }
        const unsigned int m = __ballot_sync(0xffffffffu, hd);
        const int wi = j * kPipeWarps + pwarp;
        if (lane == 0 && wi < WORDS) head[wi] = m;
      }
      named_bar(bar_id, NPT);  // heads visible
      if (pwarp == 0) {        // exclusive popcount prefix of the tile's words
        unsigned int w = 0;
        if (lane < TWORDS && lane * 32 < cnt) {
          w = head[lane];
          if (lane * 32 + 32 > cnt) w &= (1u << (cnt - lane * 32)) - 1u;
        }
        int incl = __popc(w);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (lane < TWORDS) wpref[lane] = incl - __popc(w);
        if (lane == 31) wpref[TWORDS] = incl;
      }
      named_bar(bar_id, NPT);
      if (t == 0) TKP_ADD(1, t_m);
      TKP_START(t_f);

      // ---- classify groups (striped over threads): fold short ones now ----
      const int nheads = wpref[TWORDS];
      double gval[GPT];
      short grow[GPT];
#pragma unroll
      for (int m = 0; m < GPT; ++m) {
        const int li = t + m * NPT;
        grow[m] = -1;
        gval[m] = 0.0;
        if (li >= nheads) continue;
        int lo = 0, hi = TWORDS - 1;  // word holding the li-th head
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (wpref[mid] <= li) lo = mid;
          else hi = mid - 1;
        }
        const int r = lo * 32 + (int)__fns(head[lo], 0, li - wpref[lo] + 1);
        int end = avail;
        {
          const int q1 = r + 1;
          int wi = q1 >> 5;
          unsigned int wb = (q1 < avail) ? (head[wi] & (0xffffffffu << (q1 & 31))) : 0u;
          while (wb == 0 && (wi + 1) * 32 < avail) wb = head[++wi];
          if (wb) end = min(avail, wi * 32 + __ffs(wb) - 1);
        }
        const bool open = end == avail && start + avail < p.n;
        const int len = end - r;
        if (!open && len <= kShortFold) {
          gval[m] = fold_run(s_a, r + 1, end, s_a[r]);
          grow[m] = (short)r;
        } else if (!open && len <= kShort) {
          const int q = atomicAdd(&s_nmed[pipe], 1);
          med[q] = ((unsigned long long)end << 32) | ((unsigned long long)r << 16) | (unsigned long long)li;
        } else {
          const int j = atomicAdd(&s_njobs[pipe], 1);
          sp.jobs[tile * kJobsPerTile + j] = ((unsigned long long)r << 16) | (unsigned long long)li;
        }
      }
      named_bar(bar_id, NPT);  // medium list complete
      if (t == 0) TKP_ADD(3, t_f);
      TKP_START(t_d);
      const int slot = (int)(k % kRing);
      mbar_wait(&s_based[slot], (unsigned)((k / kRing) & 1));
      const long long base = (long long)s_base[slot];
      if (t == 0) TKP_ADD(4, t_d);
      TKP_START(t_o);
      auto emit_short = [&](long long g, int r, double v) {
        p.out_vals[g] = v;
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
      };
      unsigned int zeros = 0;
      // medium groups: one per lane, packed into the first warps
      const int nmed = s_nmed[pipe];
      for (int q = t; q < nmed; q += NPT) {
        const unsigned long long e = med[q];
        const int li = (int)(e & 0xffff), r = (int)((e >> 16) & 0xffff), end = (int)(e >> 32);
        const double v = fold_run(s_a, r + 1, end, s_a[r]);
        zeros += v == 0.0;
        emit_short(base + li, r, v);
      }
#pragma unroll
      for (int m = 0; m < GPT; ++m) {
        if (grow[m] < 0) continue;
        zeros += gval[m] == 0.0;
        emit_short(base + t + m * NPT, grow[m], gval[m]);
      }
      if (zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
      named_bar(bar_id, NPT);  // slot s consumed, job list complete
      if (t == 0) {
        s_jc[s] = ((unsigned long long)base << 8) | (unsigned long long)(s_njobs[pipe] + 1);
        s_njobs[pipe] = 0;
        s_nmed[pipe] = 0;
        s_ack[slot] = k;
        mbar_arrive(&s_empty[s]);
        TKP_ADD(5, t_o);
        TKP_COUNT(7, 1);
      }
    }
    if (flags) atomicOr(&s_flags, flags);
    named_bar(bar_id, NPT);
    if (t == 0 && s_flags) atomicOr(&p.ctr->flags, s_flags);
    return;
  }

  // ============================================= chain warps =============================================
  double* cbuf = chain_buf + (size_t)(warp - (2 + kLookWarps + kPipes * kPipeWarps)) * kChunk;
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
