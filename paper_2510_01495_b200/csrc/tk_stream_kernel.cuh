// tk_stream_kernel.cuh -- the persistent streaming TTV kernel (see tk_stream.cuh for the roles).
//
// Software pipeline per CTA (iteration i handles tile T_i, ring slot b = i % NB):
//   streamers: [wait TMA T_i] head pass | popcount prefix (registers) | hand (T_i, agg) to the
//              scan warp (arrive FULL_b) | folds T_i | [sync DONE_{b'}] output T_{i-LAG} | refill
//   scan warp: [sync FULL_b] look-back T_i -> base | arrive DONE_b          (fully asynchronous)
// The output of T_i consumes its base LAG iterations later, so the look-back latency (one or
// more L2 round trips) is hidden behind LAG tiles of streaming work, and nothing in the
// streamer loop waits on the scan warp except that deferred output.
#pragma once

#include "tk_stream.cuh"

namespace tk {

template <int TILE, int HALO, int STAGES, int LAG>
constexpr size_t stream_smem_bytes(int ncol, int nk) {
  return ((size_t)ncol * (TILE + HALO) + 2 * nk) * 8 * STAGES + (size_t)kChainWarps * kChunk * 8 +
         (size_t)(LAG + 1) * TILE * 10;
}

__device__ __forceinline__ void named_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int SRC, int NK, int TILE, int HALO, int STAGES, int LAG, int LBD, int MINB>
__global__ void __launch_bounds__(kStreamThreads, MINB) ttv_stream_kernel(StreamParams sp) {
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int TWORDS = TILE / 32;
  constexpr int ITER = (ROWS + 255) / 256;
  constexpr int OWN = TILE / 256;  // rows owned per streamer thread (blocked)
  constexpr int NB = LAG + 1;      // ring slots: fold results, look-back hand-off
  constexpr int NSB = kStreamWarps * 32;
  constexpr int NSS = NSB + 32;    // streamers + scan warp
  constexpr int kFull = 2, kDone = 2 + NB;  // named barrier ids (1 = streamers only)
  static_assert(ROWS % 32 == 0 && TILE % 256 == 0 && TILE <= 1024 && TWORDS <= 32, "tile geometry (job packing: 10-bit local id)");
  static_assert(STAGES >= LAG + 2, "a stage per pending tile plus one in flight");
  static_assert(kDone + NB <= 16, "named barrier ids");
  const SegParams& p = sp.s;
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const size_t stage_words = (size_t)ncol * ROWS + 2 * nk;  // + [nk][2] previous-row words
  long long* stage0 = reinterpret_cast<long long*>(smem_raw);
  double* chain_buf = reinterpret_cast<double*>(stage0 + stage_words * STAGES);
  double* s_val = chain_buf + kChainWarps * kChunk;           // [NB][TILE] folded values by local id
  short* s_row = reinterpret_cast<short*>(s_val + NB * TILE);  // [NB][TILE] head row (-1: chain job)

  __shared__ __align__(8) uint64_t s_full[STAGES];
  __shared__ long long s_stage_tile[STAGES];
  __shared__ int s_stage_bulk[STAGES];
  __shared__ unsigned int s_head[WORDS];
  __shared__ long long s_lb_tile[NB];
  __shared__ int s_nheads[NB];
  __shared__ unsigned long long s_base[NB];
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&s_full[s], 1);
    s_flags = 0;
  }
  __syncthreads();

  if (warp == kScanWarp) {
    // ========================= scan warp: asynchronous look-backs =========================
    for (long long k = 0;; ++k) {
      const int b = (int)(k % NB);
      TKP_START(t_w);
      named_bar(kFull + b, NSS);
      if (lane == 0) TKP_ADD(8, t_w);
      const long long tile = s_lb_tile[b];
      if (tile < 0) break;
      const unsigned long long agg = (unsigned long long)s_nheads[b];
      TKP_START(t_l);
      const unsigned long long excl = lookback_wide<LBD>(p.status, tile, agg);
      if (lane == 0) TKP_ADD(9, t_l);
      if (lane == 0) {
        s_base[b] = excl;
        const long long start = tile * TILE;
        if (start + min((long long)TILE, p.n - start) == p.n) p.ctr->groups = excl + agg;
      }
      __syncwarp();
      named_arrive(kDone + b, NSS);
    }
    return;
  }

  if (warp < kStreamWarps) {
    // ==================================== streamers ====================================
    // Static round-robin tiles (CTA c: c, c+G, c+2G, ...): every CTA processes its k-th tile
    // in the same wave as its neighbours, so a look-back finds its predecessors' aggregates
    // published by CTAs working in lock-step, not by one that prefetched far ahead.
    long long next_tile = blockIdx.x;
    auto acquire_issue = [&](int s) {  // thread 0 only
      const long long t = next_tile;
      next_tile += gridDim.x;
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
    };

    if (tid == 0)
      for (int s = 0; s < STAGES; ++s) acquire_issue(s);
    unsigned int phase = 0;
    unsigned int flags = 0;
    long long hist[LAG];
#pragma unroll
    for (int k = 0; k < LAG; ++k) hist[k] = -1;
    int s = 0;
    long long i = 0;
    for (;; ++i) {
      TKP_START(t_a);
      named_bar(1, NSB);  // (A) stage s descriptor visible; previous tile's smem reads done
      if (tid == 0) TKP_ADD(6, t_a);
      const long long tile = s_stage_tile[s];
      const long long out_tile = hist[LAG - 1];  // tile of iteration i - LAG
      bool any = tile >= 0 || out_tile >= 0;
#pragma unroll
      for (int k = LAG - 1; k > 0; --k) {
        hist[k] = hist[k - 1];
        any = any || hist[k] >= 0;
      }
      hist[0] = tile;
      if (!any) break;
      const int b = (int)(i % NB);

      if (tile >= 0) {
        long long* st = stage0 + stage_words * s;
        long long* s_key = st;
        double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
        const long long* s_subk = st + (size_t)(nk + 1) * ROWS;
        const long long* s_prev2 = st + (size_t)ncol * ROWS;
        const long long start = tile * TILE;
        const int cnt = (int)min((long long)TILE, p.n - start);
        const int avail = (int)min((long long)ROWS, p.n - start);
        TKP_START(t_m);
        if (s_stage_bulk[s]) {
          mbar_wait(&s_full[s], (phase >> s) & 1u);
          phase ^= 1u << s;
          if (tid == 0) TKP_ADD(0, t_m);
        } else {
          for (int r = tid; r < avail; r += NSB) {
            for (int c = 0; c < nk; ++c) s_key[c * ROWS + r] = p.key[c][start + r];
            s_a[r] = p.a[start + r];
            if constexpr (SRC == kSrcRaw) st[(size_t)(nk + 1) * ROWS + r] = p.subk[start + r];
          }
          if (tid < nk && start > 0) st[(size_t)ncol * ROWS + 2 * tid + 1] = p.key[tid][start - 1];
          named_bar(1, NSB);
        }
        // ---- w and head flags (striped rows: conflict-free shared memory) ----
        if constexpr (SRC == kSrcRaw) {
          // all gathers in flight before any store: a store to s_a could alias the
          // later loads for the compiler, which would serialise ITER L2 round trips
          double xv[ITER], av[ITER];
#pragma unroll
          for (int j = 0; j < ITER; ++j) {
            const int r = j * 256 + tid;
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
            const int r = j * 256 + tid;
            if (r < avail) s_a[r] = __dmul_rn(av[j], xv[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < ITER; ++j) {
          const int r = j * 256 + tid;
          bool head = false;
          if (r < avail) {
            int cmp = 0;
#pragma unroll
            for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
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
          const int wi = j * 8 + warp;
          if (lane == 0 && wi < WORDS) s_head[wi] = m;
        }
        if (tid == 0) TKP_ADD(1, t_m);
        TKP_START(t_b);
        named_bar(1, NSB);  // (B) heads visible to all streamer warps
        if (tid == 0) TKP_ADD(2, t_b);
        TKP_START(t_f);

        // ---- popcount prefix over the tile's words, one word per lane, in every warp ----
        unsigned int myword = 0;
        if (lane < TWORDS && lane * 32 < cnt) {
          myword = s_head[lane];
          if (lane * 32 + 32 > cnt) myword &= (1u << (cnt - lane * 32)) - 1u;
        }
        int incl = __popc(myword);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int wpref = incl - __popc(myword);  // exclusive prefix of word `lane`
        const int agg = __shfl_sync(0xffffffffu, incl, 31);
        if (tid == 0) {
          lookback_publish_agg<LBD>(p.status, tile, (unsigned long long)agg);
          s_lb_tile[b] = tile;
          s_nheads[b] = agg;
        }
        named_arrive(kFull + b, NSS);  // hand (tile, agg) to the scan warp

        // ---- folds (blocked row ownership); long / spanning groups -> chain jobs ----
        double* vb = s_val + (size_t)b * TILE;
        short* rb = s_row + (size_t)b * TILE;
        const int r0 = tid * OWN;
        // the OWN rows of this thread lie in word r0 >> 5
        const int wp_own = __shfl_sync(0xffffffffu, wpref, (r0 >> 5) & 31);
#pragma unroll 1
        for (int q = 0; q < OWN; ++q) {
          const int r = r0 + q;
          if (r >= cnt) break;
          const unsigned int word = s_head[r >> 5];
          if (!((word >> (r & 31)) & 1u)) continue;
          const int li = wp_own + __popc(word & ((1u << (r & 31)) - 1u));
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
            vb[li] = fold_run(s_a, r + 1, end, s_a[r]);
            rb[li] = (short)r;
          } else {
            rb[li] = -1;
            // one 64-bit word = the whole job: no fence needed to publish it
            const unsigned long long slot = atomicAdd(&p.ctr->q_tail, 1ull);
            st_relaxed(sp.jobs + slot, job_pack(start + r, li, agg));
          }
        }
        if (tid == 0) TKP_ADD(3, t_f);
      }

      // ---- output of tile T_{i-LAG}: coalesced stores of its short groups ----
      if (out_tile >= 0) {
        const int bo = (int)((i + 1) % NB);  // == (i - LAG) % NB
        const int so = (s - LAG + STAGES) % STAGES;
        TKP_START(t_d);
        named_bar(kDone + bo, NSS);  // wait for its base
        if (tid == 0) TKP_ADD(4, t_d);
        TKP_START(t_o);
        const long long* s_key = stage0 + stage_words * so;
        const int nheads = s_nheads[bo];
        const long long base = (long long)s_base[bo];
        const double* vb = s_val + (size_t)bo * TILE;
        const short* rb = s_row + (size_t)bo * TILE;
        unsigned int zeros = 0;
        for (int li = tid; li < nheads; li += NSB) {
          const int r = rb[li];
          if (r < 0) continue;
          const double v = vb[li];
          p.out_vals[base + li] = v;
          zeros += v == 0.0;
          if constexpr (SRC == kSrcLinKey) {
            long long lin = s_key[r];
            long long* o = p.out_subs + (base + li) * p.out_nk;
            for (int q = p.out_nk - 1; q >= 0; --q) {
              const long long dm = p.dims[q];
              o[q] = lin % dm;
              lin /= dm;
            }
          } else {
#pragma unroll
            for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
              if (NK == 0 && c >= nk) break;
              p.out_subs[(base + li) * p.out_nk + c] = s_key[c * ROWS + r];
            }
          }
        }
        if (zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
        named_bar(1, NSB);  // stage `so` consumed
        if (tid == 0) acquire_issue(so);
        if (tid == 0) TKP_ADD(5, t_o);
        if (tid == 0) TKP_COUNT(7, 1);
      }
      s = (s + 1) % STAGES;
    }
    // stop the scan warp: sentinel in the next ring slot (every earlier slot is drained).
    // Tiles were processed in iterations 0..ntile-1 (tickets are monotonic), so the slot
    // the scan warp waits on is ntile % NB.
    const long long ntile = i - LAG < 0 ? 0 : i - LAG;
    if (tid == 0) s_lb_tile[(int)(ntile % NB)] = -1;
    named_arrive(kFull + (int)(ntile % NB), NSS);
    if (flags) atomicOr(&s_flags, flags);
    named_bar(1, NSB);
    if (tid == 0) {
      if (s_flags) atomicOr(&p.ctr->flags, s_flags);
      __threadfence();
      atomicAdd(&p.ctr->streamers_done, 1u);
    }
    return;
  }

  // ===================================== chain warps =====================================
  // Each warp drains jobs: a job is a group that is long or crosses its tile.  Rows stream in
  // 256-row chunks (8 per lane, coalesced, L2-hot); the x gathers of a chunk are issued
  // together; lane 0 folds the chunk serially from smem while the next chunk is in flight.
  double* cbuf = chain_buf + (size_t)(warp - kScanWarp - 1) * kChunk;
  constexpr int NKR = NK > 0 ? NK : kMaxKeep;
  while (true) {
    long long start = -1;
    unsigned long long job = 0;
    TKP_START(t_idle);
    if (lane == 0) {
      const unsigned long long t = atomicAdd(&p.ctr->q_head, 1ull);
      while (true) {
        if (t < ld_relaxed_u64(&p.ctr->q_tail)) {
          while ((job = ld_relaxed_u64(sp.jobs + t)) == 0) __nanosleep(32);
          sp.jobs[t] = 0;  // self-cleaning queue
          start = (long long)(job >> 21) - 1;
          break;
        }
        if (ld_relaxed_u32(&p.ctr->streamers_done) == gridDim.x) {
          if (t < ld_relaxed_u64(&p.ctr->q_tail)) continue;
          break;
        }
        __nanosleep(512);
      }
    }
    start = __shfl_sync(0xffffffffu, start, 0);
    if (lane == 0) TKP_ADD(10, t_idle);
    if (start < 0) break;
    TKP_START(t_busy);
    job = __shfl_sync(0xffffffffu, job, 0);

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
    // output slot = tile base (its published inclusive prefix minus its aggregate) + local id
    if (lane == 0) {
      const long long tile = start / TILE;
      const unsigned long long li = (job >> 11) & 0x3ff, agg = job & 0x7ff;
      unsigned long long stw;
      while (((stw = ld_relaxed(p.status + tile)) >> 62) != 2) __nanosleep(64);
      const long long g = (long long)((stw & kStVal) - agg + li);
      seg_emit<SRC>(p, g, gk, acc);
      TKP_ADD(11, t_busy);
      TKP_COUNT(12, 1);
    }
  }
}

}  // namespace tk
