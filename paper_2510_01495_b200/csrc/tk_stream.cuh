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

// job record: start row + 1 (0 = empty slot; written last, with release semantics) and
// (tile, local group index, tile head count) packed into one word.
struct StreamJob {
  unsigned long long start_p1;
  unsigned long long meta;  // tile << 24 | local << 12 | agg   (TILE <= 4096)
};

struct StreamParams {
  SegParams s;          // stream description + outputs + status/ctr
  StreamJob* jobs;      // self-cleaning: all-zero on entry and on exit
  long long ntiles;
};

constexpr int kStreamWarps = 8;
constexpr int kScanWarp = 8;
constexpr int kChainWarps = 4;
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

// Look-back with a 4-deep window per lane (128 predecessors per round).
__device__ __forceinline__ unsigned long long lookback_wide(unsigned long long* status, long long tile,
                                                            unsigned long long agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed(status, kStPre | agg);
    return 0;
  }
  if (lane == 0) st_relaxed(status + tile, kStAgg | agg);
  unsigned long long excl = 0;
  long long look = tile - 1;
  while (true) {
    unsigned long long s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long t = look - (lane * 4 + i);
      s[i] = t >= 0 ? ld_relaxed(status + t) : kStPre;
    }
    bool pending = true;
    while (pending) {
      bool mine = false;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((s[i] >> 62) == 0) {
          s[i] = ld_relaxed(status + (look - (lane * 4 + i)));
          mine = mine || (s[i] >> 62) == 0;
        }
      pending = __any_sync(0xffffffffu, mine);
    }
    // first (nearest) prefix in lane-major order: element e = lane*4 + i
    int first_pre = 1 << 30;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if ((s[i] >> 62) == 2 && first_pre == (1 << 30)) first_pre = lane * 4 + i;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first_pre = min(first_pre, __shfl_xor_sync(0xffffffffu, first_pre, o));
    unsigned long long v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane * 4 + i <= first_pre) v += s[i] & kStVal;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (first_pre < (1 << 30)) break;
    look -= 128;
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

template <int TILE, int HALO, int STAGES>
constexpr size_t stream_smem_bytes(int ncol, int nk) {
  return ((size_t)ncol * (TILE + HALO) + 2 * nk) * 8 * STAGES + (size_t)kChainWarps * kChunk * 8 + (size_t)TILE * 10;
}

template <int SRC, int NK, int TILE, int HALO, int STAGES, int MINB>
__global__ void __launch_bounds__(kStreamThreads, MINB) ttv_stream_kernel(StreamParams sp) {
  constexpr int ROWS = TILE + HALO;
  constexpr int WORDS = ROWS / 32;
  constexpr int TWORDS = TILE / 32;
  constexpr int ITER = (ROWS + 255) / 256;
  constexpr int OWN = TILE / 256;  // rows owned per streamer thread (blocked)
  static_assert(ROWS % 32 == 0 && TILE % 256 == 0 && TILE < 4096, "tile geometry");
  const SegParams& p = sp.s;
  const int nk = seg_nk<SRC, NK>(p);
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);  // keys | a | subk
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const size_t stage_words = (size_t)ncol * ROWS + 2 * nk;  // + [nk][2] previous-row words
  long long* stage0 = reinterpret_cast<long long*>(smem_raw);
  double* chain_buf = reinterpret_cast<double*>(stage0 + stage_words * STAGES);
  double* s_val = chain_buf + kChainWarps * kChunk;            // [TILE] folded values by local id
  short* s_row = reinterpret_cast<short*>(s_val + TILE);        // [TILE] head row of local id (-1: chain)

  __shared__ __align__(8) uint64_t s_full[STAGES];
  __shared__ long long s_stage_tile[STAGES];
  __shared__ int s_stage_bulk[STAGES];
  __shared__ unsigned int s_head[WORDS];
  __shared__ int s_wpref[TWORDS];
  __shared__ int s_nheads;
  __shared__ unsigned long long s_base;
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&s_full[s], 1);
    s_flags = 0;
  }
  __syncthreads();

  if (warp <= kScanWarp) {
    // ====================== streamer warps + scan warp (shared tile loop) ======================
    const bool scan = warp == kScanWarp;
    auto acquire_issue = [&](int s) {  // streamer thread 0 only
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
    int s = 0;
    while (true) {
      named_bar(2, 288);  // (A) stage s descriptor visible
      const long long tile = s_stage_tile[s];
      if (tile < 0) break;
      long long* st = stage0 + stage_words * s;
      long long* s_key = st;
      double* s_a = reinterpret_cast<double*>(st + (size_t)nk * ROWS);
      const long long* s_subk = st + (size_t)(nk + 1) * ROWS;
      const long long* s_prev2 = st + (size_t)ncol * ROWS;
      const long long start = tile * TILE;
      const int cnt = (int)min((long long)TILE, p.n - start);
      const int avail = (int)min((long long)ROWS, p.n - start);

      if (!scan) {
        if (s_stage_bulk[s]) {
          mbar_wait(&s_full[s], (phase >> s) & 1u);
        } else {
          for (int r = tid; r < avail; r += kStreamWarps * 32) {
            for (int c = 0; c < nk; ++c) s_key[c * ROWS + r] = p.key[c][start + r];
            s_a[r] = p.a[start + r];
            if constexpr (SRC == kSrcRaw) st[(size_t)(nk + 1) * ROWS + r] = p.subk[start + r];
          }
          if (tid < nk && start > 0) st[(size_t)ncol * ROWS + 2 * tid + 1] = p.key[tid][start - 1];
          named_bar(1, 256);
        }
        // ---- w and head flags (striped rows: conflict-free shared memory) ----
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
            const long long* prevp = r == 0 ? s_prev2 + 1 : nullptr;
#pragma unroll
            for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c) {
              if (NK == 0 && c >= nk) break;
              const long long va = s_key[c * ROWS + r];
              const long long vb = r ? s_key[c * ROWS + r - 1] : prevp[2 * c];
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
      }
      if (s_stage_bulk[s]) phase ^= 1u << s;
      named_bar(2, 288);  // (B) heads ready

      if (scan) {
        // popcount prefix over the tile's words, publish, look back (overlaps the folds)
        constexpr int PL = (TWORDS + 31) / 32;
        int cw[PL];
        int mine = 0;
#pragma unroll
        for (int i = 0; i < PL; ++i) {
          const int wi = lane * PL + i;
          unsigned int word = 0;
          if (wi < TWORDS && wi * 32 < cnt) {
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
        for (int i = 0; i < PL; ++i) {
          const int wi = lane * PL + i;
          if (wi < TWORDS) s_wpref[wi] = run;
          run += cw[i];
        }
        const int agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) s_nheads = agg;
        __syncwarp();
        named_bar(3, 288);  // (C) local ids ready
        const unsigned long long excl = lookback_wide(p.status, tile, (unsigned long long)agg);
        if (lane == 0) {
          s_base = excl;
          if (start + cnt == p.n) p.ctr->groups = excl + (unsigned long long)agg;
        }
      } else {
        named_bar(3, 288);  // (C)
        const int nheads = s_nheads;
        // ---- folds (blocked row ownership); long / spanning groups -> chain jobs ----
        const int r0 = tid * OWN;
#pragma unroll 1
        for (int i = 0; i < OWN; ++i) {
          const int r = r0 + i;
          if (r >= cnt) break;
          const unsigned int word = s_head[r >> 5];
          if (!((word >> (r & 31)) & 1u)) continue;
          const int li = s_wpref[r >> 5] + __popc(word & ((1u << (r & 31)) - 1u));
          int end = avail;
          {
            const int q = r + 1;
            int wi = q >> 5;
            unsigned int wb = (q < avail) ? (s_head[wi] & (0xffffffffu << (q & 31))) : 0u;
            while (wb == 0 && (wi + 1) * 32 < avail) wb = s_head[++wi];
            if (wb) end = min(avail, wi * 32 + __ffs(wb) - 1);
          }
          const bool open = end == avail && start + avail < p.n;
          if (!open && end - r <= kShort) {
            s_val[li] = fold_run(s_a, r + 1, end, s_a[r]);
            s_row[li] = (short)r;
          } else {
            s_row[li] = -1;
            const unsigned long long slot = atomicAdd(&p.ctr->q_tail, 1ull);
            StreamJob* jb = sp.jobs + slot;
            jb->meta = ((unsigned long long)tile << 24) | ((unsigned long long)li << 12) | (unsigned long long)nheads;
            st_release_u64(&jb->start_p1, (unsigned long long)(start + r) + 1ull);
          }
        }
      }
      named_bar(2, 288);  // (D) folds staged, base known
      if (!scan) {
        // ---- coalesced output of the short groups ----
        const int nheads = s_nheads;
        const long long base = (long long)s_base;
        unsigned int zeros = 0;
        for (int li = tid; li < nheads; li += 256) {
          const int r = s_row[li];
          if (r < 0) continue;
          const double v = s_val[li];
          p.out_vals[base + li] = v;
          zeros += v == 0.0;
          if constexpr (SRC == kSrcLinKey) {
            long long kv[1] = {s_key[r]};
            write_key<SRC>(p, base + li, 0, 0, kv);
          } else {
            for (int c = 0; c < nk; ++c) p.out_subs[(base + li) * p.out_nk + c] = s_key[c * ROWS + r];
          }
        }
        if (zeros) atomicAdd(&p.ctr->zeros, (unsigned long long)zeros);
        named_bar(1, 256);  // stage s consumed
        if (tid == 0) acquire_issue(s);
      }
      s = (s + 1) % STAGES;
    }
    if (!scan) {
      if (flags) atomicOr(&s_flags, flags);
      named_bar(1, 256);
      if (tid == 0) {
        if (s_flags) atomicOr(&p.ctr->flags, s_flags);
        __threadfence();
        atomicAdd(&p.ctr->streamers_done, 1u);
      }
    }
    return;
  }

  // ===================================== chain warps =====================================
  double* cbuf = chain_buf + (size_t)(warp - kScanWarp - 1) * kChunk;
  while (true) {
    unsigned long long t = 0;
    long long start = -1;
    unsigned long long meta = 0;
    if (lane == 0) {
      t = atomicAdd(&p.ctr->q_head, 1ull);
      while (true) {
        if (t < ld_relaxed_u64(&p.ctr->q_tail)) {
          unsigned long long sp1;
          while ((sp1 = ld_relaxed_u64(&sp.jobs[t].start_p1)) == 0) __nanosleep(32);
          start = (long long)(sp1 - 1);
          meta = ld_relaxed_u64(&sp.jobs[t].meta);
          sp.jobs[t].start_p1 = 0;  // self-cleaning queue
          break;
        }
        if (ld_relaxed_u32(&p.ctr->streamers_done) == gridDim.x) {
          if (t < ld_relaxed_u64(&p.ctr->q_tail)) continue;
          break;
        }
        __nanosleep(256);
      }
    }
    start = __shfl_sync(0xffffffffu, start, 0);
    if (start < 0) break;
    meta = __shfl_sync(0xffffffffu, meta, 0);
    long long gk[NK > 0 ? NK : kMaxKeep];
#pragma unroll
    for (int c = 0; c < (NK > 0 ? NK : kMaxKeep); ++c)
      if (NK > 0 || c < nk) gk[c] = __ldcg(p.key[c] + start);

    double acc = 0.0;
    bool first = true;
    long long pos = start;
    double av[8];
    long long sk[8];
    bool same[8];
    auto load_chunk = [&](long long b) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const long long r = b + i * 32 + lane;
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
        if (first) {
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
    // output slot: tile base (from the tile's published inclusive prefix) + local id
    if (lane == 0) {
      const long long tile = (long long)(meta >> 24);
      const unsigned long long li = (meta >> 12) & 0xfff, agg = meta & 0xfff;
      unsigned long long stw;
      while (((stw = ld_relaxed(p.status + tile)) >> 62) != 2) __nanosleep(64);
      const long long g = (long long)((stw & kStVal) - agg + li);
      seg_emit<SRC>(p, g, gk, acc);
    }
  }
}

}  // namespace tk
