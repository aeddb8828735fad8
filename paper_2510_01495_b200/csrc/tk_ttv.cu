// tk_ttv.cu -- sparse TTV orchestration (sparse result and dense multi-vector result).
//
// Paths:
//   fast    : contracted mode is the trailing mode of a canonical tensor -> the kept
//             tuples are already sorted; one fused streaming kernel (seg_ttv_kernel<Raw>).
//   general : any other mode / unsorted input -> w and a linearised kept key per row,
//             stable device radix sort of (key, w), then the same segmented kernel
//             (<LinKey>).  Garbage kept indices or keys wider than 62 bits: LSD radix
//             passes over the kept columns (signed int64) carrying a permutation, then
//             <KeysW>.  Both sorts are stable, so every group is folded in ascending
//             original-row order, exactly like the reference (pyx:229-295).
//   dense   : multi-vector TTV to a dense vector (BASELINE config 4): one streaming
//             kernel with a deterministic block-level segmented reduction and a tiny
//             ordered fix-up for runs that cross tiles; chained single-mode TTV otherwise.
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "tk_host.h"
#include "tk_tile_kernel.cuh"
#include "tk_ttv_kernels.cuh"

namespace tk {

// ============================================================================================
// helper kernels
// ============================================================================================

struct KeepCols {
  const long long* col[kMaxKeep];
  long long dims[kMaxKeep];
};

__global__ void prep_linkey_kernel2(long long n, int nk, KeepCols kc, const long long* __restrict__ subk,
                                    const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                    long long* __restrict__ key, double* __restrict__ w, Counters* ctr) {
  unsigned int flags = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long idx = subk[r];
    double wr = 0.0;
    if (idx < 0 || idx >= nx) flags |= kFlagIndex;
    else wr = __dmul_rn(vals[r], __ldg(x + idx));
    long long lin = 0;
    for (int c = 0; c < nk; ++c) {
      const long long v = kc.col[c][r];
      if (v < 0 || v >= kc.dims[c]) flags |= kFlagKeptOob;
      lin = lin * kc.dims[c] + v;
    }
    key[r] = lin;
    w[r] = wr;
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

__global__ void iota_kernel(long long n, long long* out) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    out[r] = r;
}

__global__ void gather_i64_kernel(long long n, const long long* __restrict__ src, const long long* __restrict__ idx,
                                  long long* __restrict__ dst) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x)
    dst[r] = src[idx[r]];
}

__global__ void gather_w_kernel(long long n, const long long* __restrict__ perm, const long long* __restrict__ subk,
                                const double* __restrict__ vals, const double* __restrict__ x, long long nx,
                                double* __restrict__ w, Counters* ctr) {
  unsigned int flags = 0;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long o = perm[r];
    const long long idx = subk[o];
    double wr = 0.0;
    if (idx < 0 || idx >= nx) flags |= kFlagIndex;
    else wr = __dmul_rn(vals[o], __ldg(x + idx));
    w[r] = wr;
  }
  if (flags) atomicOr(&ctr->flags, flags);
}

__global__ void aos_to_soa_kernel(long long n, int d, const long long* __restrict__ aos, long long* __restrict__ soa,
                                  long long pitch) {
  const long long total = n * d;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / d;
    const int m = (int)(e - r * d);
    soa[m * pitch + r] = __ldcs(aos + e);
  }
}

// ---- zero-group compaction (runs only when some group summed to exactly 0.0) -----------------
constexpr int kCompItems = 8;
constexpr int kCompTile = 256 * kCompItems;

__global__ void nz_count_kernel(long long n, const double* __restrict__ v, long long* __restrict__ blk) {
  using Reduce = cub::BlockReduce<int, 256>;
  __shared__ typename Reduce::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kCompTile;
  int c = 0;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + threadIdx.x * kCompItems + i;
    if (e < n && v[e] != 0.0) ++c;
  }
  const int tot = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) blk[blockIdx.x] = tot;
}

__global__ void scan_blocks_kernel(long long nblk, long long* __restrict__ blk) {
  // single block, exclusive scan in place (sequential chunks of 256)
  using Scan = cub::BlockScan<long long, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (long long off = 0; off < nblk; off += 256) {
    const long long i = off + threadIdx.x;
    long long v = i < nblk ? blk[i] : 0, ex, agg;
    Scan(tmp).ExclusiveSum(v, ex, agg);
    if (i < nblk) blk[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += agg;
    __syncthreads();
  }
}

__global__ void nz_scatter_kernel(long long n, int nk, const double* __restrict__ v, const long long* __restrict__ s,
                                  const long long* __restrict__ blk, double* __restrict__ v2, long long* __restrict__ s2) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  const long long base = (long long)blockIdx.x * kCompTile + threadIdx.x * kCompItems;
  int c = 0;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + i;
    if (e < n && v[e] != 0.0) ++c;
  }
  int ex;
  Scan(tmp).ExclusiveSum(c, ex);
  long long o = blk[blockIdx.x] + ex;
  for (int i = 0; i < kCompItems; ++i) {
    const long long e = base + i;
    if (e < n && v[e] != 0.0) {
      v2[o] = v[e];
      for (int q = 0; q < nk; ++q) s2[o * nk + q] = s[e * nk + q];
      ++o;
    }
  }
}

// ============================================================================================
// dense-result multi-vector kernel
// ============================================================================================

struct DenseParams {
  long long n;
  int d, keep;
  const long long* col[kMaxOrder];
  const double* vals;
  const double* vec[kMaxOrder];
  long long dims[kMaxOrder];
  double* out;
  double* c_first;
  double* c_last;
  long long* c_lastkey;
  int* c_flags;
  Counters* ctr;
  int bulk_ok;
};

struct SegPair {
  int f;
  double v;
};
// (a then b): a run head in b restarts the sum; otherwise b continues a's run.
__device__ __forceinline__ SegPair seg_combine(SegPair a, SegPair b) {
  return {a.f | b.f, b.f ? b.v : __dadd_rn(a.v, b.v)};
}

template <int kItems, int D>  // D: tensor order when 3..5 (gathers batched), 0: any order
__global__ void __launch_bounds__(256) dense_ttv_kernel(DenseParams p) {
  constexpr int TILE = kItems * 256;
  constexpr int NW = TILE / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  long long* s_col = reinterpret_cast<long long*>(smem_raw);   // [d][TILE]
  double* s_v = reinterpret_cast<double*>(s_col + (size_t)p.d * TILE);
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ unsigned int s_head[NW];
  __shared__ long long s_prev, s_next;
  __shared__ int s_has_prev, s_has_next;
  __shared__ SegPair s_warp[8];
  __shared__ unsigned int s_flags;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long tile = blockIdx.x;
  const long long start = tile * TILE;
  const int cnt = (int)min((long long)TILE, p.n - start);
  const int keep = p.keep;
  const long long* s_key = s_col + (size_t)keep * TILE;

  const bool bulk = p.bulk_ok && cnt == TILE;
  if (tid == 0) s_flags = 0;
  if (bulk) {
    if (tid == 0) {
      mbar_init(&s_bar, 1);
      const uint32_t col_bytes = TILE * 8u;
      mbar_arrive_expect_tx(&s_bar, col_bytes * (p.d + 1));
      const uint64_t pol = l2_evict_first_policy();
      for (int m = 0; m < p.d; ++m) bulk_g2s(s_col + (size_t)m * TILE, p.col[m] + start, col_bytes, &s_bar, pol);
      bulk_g2s(s_v, p.vals + start, col_bytes, &s_bar, pol);
    }
  } else {
    for (int j = 0; j < kItems; ++j) {
      const int r = j * 256 + tid;
      if (r < cnt) {
        for (int m = 0; m < p.d; ++m) s_col[m * TILE + r] = p.col[m][start + r];
        s_v[r] = p.vals[start + r];
      }
    }
  }
  if (tid == 32) {
    s_has_prev = start > 0;
    s_has_next = start + cnt < p.n;
    if (start > 0) s_prev = p.col[keep][start - 1];
    if (start + cnt < p.n) s_next = p.col[keep][start + cnt];
  }
  __syncthreads();
  if (bulk) mbar_wait(&s_bar, 0);

  // w = ((vals * x_{d-1}) * x_{d-2}) ... (descending modes: the chained-TTV association)
  unsigned int flags = 0;
  const long long nkeep = p.dims[keep];
  // every gather of the tile in flight before the first multiply (D known at compile time)
  double xg[D > 0 ? kItems : 1][D > 0 ? D : 1];
  if constexpr (D > 0) {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int r = j * 256 + tid;
      const int rc = min(r, cnt - 1);
#pragma unroll
      for (int m = 0; m < D; ++m) {
        xg[j][m] = 1.0;
        if (m != keep) {
          const long long idx = s_col[m * TILE + rc];
          const bool bad = (unsigned long long)idx >= (unsigned long long)p.dims[m];
          if (bad && r < cnt) flags |= kFlagIndex;  // the call raises; the value is never used
          xg[j][m] = __ldg(p.vec[m] + (bad ? 0 : idx));
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const int r = j * 256 + tid;
    bool head = false;
    if (r < cnt) {
      double w = s_v[r];
      if constexpr (D > 0) {
#pragma unroll
        for (int m = D - 1; m >= 0; --m)
          if (m != keep) w = __dmul_rn(w, xg[j][m]);
      } else {
        for (int m = p.d - 1; m >= 0; --m) {
          if (m == keep) continue;
          const long long idx = s_col[m * TILE + r];
          if (idx < 0 || idx >= p.dims[m]) { flags |= kFlagIndex; w = 0.0; }
          else w = __dmul_rn(w, __ldg(p.vec[m] + idx));
        }
      }
      s_v[r] = w;
      const long long key = s_key[r];
      if (key < 0 || key >= nkeep) flags |= kFlagKeptOob;
      if (r == 0) head = !s_has_prev || key != s_prev, flags |= (s_has_prev && key < s_prev) ? kFlagUnsorted : 0u;
      else {
        const long long pk = s_key[r - 1];
        head = key != pk;
        if (key < pk) flags |= kFlagUnsorted;
      }
    }
    const unsigned int m = __ballot_sync(0xffffffffu, head);
    if (lane == 0) s_head[j * 8 + warp] = m;
  }
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();

  // blocked per-thread segmented fold
  const int r0 = tid * kItems;
  double first = 0.0, cur = 0.0;
  int hh = 0;
  long long curkey = 0;
  for (int i = 0; i < kItems; ++i) {
    const int r = r0 + i;
    if (r >= cnt) break;
    if ((s_head[r >> 5] >> (r & 31)) & 1u) {
      if (hh) {
        if (curkey >= 0 && curkey < nkeep) p.out[curkey] = cur;  // run wholly inside this thread
      } else {
        first = cur;
        hh = 1;
      }
      cur = s_v[r];
      curkey = s_key[r];
    } else {
      cur = (i == 0) ? s_v[r] : __dadd_rn(cur, s_v[r]);
    }
  }
  // block segmented scan over threads of (has_head, last-run partial)
  SegPair mine{hh, cur};
  SegPair inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    SegPair up{__shfl_up_sync(0xffffffffu, inc.f, o), __shfl_up_sync(0xffffffffu, inc.v, o)};
    if (lane >= o) inc = seg_combine(up, inc);
  }
  SegPair exc{__shfl_up_sync(0xffffffffu, inc.f, 1), __shfl_up_sync(0xffffffffu, inc.v, 1)};
  if (lane == 0) exc = {0, 0.0};
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  SegPair wpre{0, 0.0};
  for (int q = 0; q < warp; ++q) wpre = seg_combine(wpre, s_warp[q]);
  exc = lane == 0 ? wpre : seg_combine(wpre, exc);
  inc = seg_combine(wpre, inc);

  if (hh) {  // the run open at this thread's start closes at its first head
    const double closing = __dadd_rn(exc.v, first);
    if (exc.f) {
      const long long k = s_key[r0 - 1];
      if (k >= 0 && k < nkeep) p.out[k] = closing;
    } else {
      p.c_first[tile] = closing;
    }
  }
  if (tid == 255) {
    const long long lastkey = s_key[cnt - 1];
    const bool last_open = s_has_next && s_next == lastkey;
    if (inc.f) {
      if (last_open) {
        p.c_last[tile] = inc.v;
        p.c_lastkey[tile] = lastkey;
      } else if (lastkey >= 0 && lastkey < nkeep) {
        p.out[lastkey] = inc.v;
      }
    } else {
      p.c_first[tile] = inc.v;
    }
    p.c_flags[tile] = (inc.f ? 1 : 0) | (last_open ? 2 : 0);
    if (s_flags) atomicOr(&p.ctr->flags, s_flags);
  }
}

__global__ void dense_fixup_kernel(long long ntiles, const double* __restrict__ c_first,
                                   const double* __restrict__ c_last, const long long* __restrict__ c_lastkey,
                                   const int* __restrict__ c_flags, long long nkeep, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= ntiles || (c_flags[t] & 3) != 3) return;
  double s = c_last[t];
  for (long long t2 = t + 1; t2 < ntiles; ++t2) {
    s = __dadd_rn(s, c_first[t2]);
    const int f2 = c_flags[t2];
    if ((f2 & 1) || !(f2 & 2)) break;
  }
  const long long k = c_lastkey[t];
  if (k >= 0 && k < nkeep) out[k] = s;
}

// ============================================================================================
// host orchestration
// ============================================================================================

namespace {

// Opt a kernel in to >48 KB of dynamic shared memory, once per (kernel, device).
template <class K>
void set_smem_once(K kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{reinterpret_cast<const void*>(kernel), dev}];
  if (bytes > have) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    // all shared memory: eight tile CTAs need ~216 KB; x's hot entries still fit the rest of L1
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    have = bytes;
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(long long n, int per_thread = 4) {
  long long want = (n + 256LL * per_thread - 1) / (256LL * per_thread);
  long long cap = (long long)num_sms() * 16;
  return (int)std::max(1LL, std::min(want, cap));
}

template <int SRC, int NK>
int launch_stream_t(SegParams& p, cudaStream_t st, Counters* host_ctr) {
  // one CTA per tile, eight CTAs per SM (~19 KB shared memory each: L1 keeps x resident)
#ifndef TK_TILE_LAG
#define TK_TILE_LAG 1024  // tiles between a tile's count and its fold
#endif
#ifndef TK_TILE_ROWS
#define TK_TILE_ROWS 768
#endif
  constexpr int TILE = NK > 0 ? TK_TILE_ROWS : 256;
  constexpr int HALO = 32;
  const int nk = SRC == kSrcLinKey ? 1 : p.nk;
  const int ncol = nk + 1 + (SRC == kSrcRaw ? 1 : 0);
  const size_t smem = tile_total_smem<SRC, TILE, HALO>(ncol, nk);
  auto kern = ttv_tile_kernel<SRC, NK, TILE, HALO>;
  set_smem_once(kern, smem);
  const long long ntiles = (p.n + TILE - 1) / TILE;
  const size_t status_b = ((size_t)ntiles * 8 + 255) & ~size_t(255);
  DevBuf scratch;
  if (int rc = scratch.alloc(status_b + 256, st)) return rc;
  char* b = scratch.as<char>();
  p.status = reinterpret_cast<unsigned long long*>(b);
  p.ctr = reinterpret_cast<Counters*>(b + status_b);
  TK_CUDA(cudaMemsetAsync(b, 0, status_b + 256, st));
  DevBuf prof;
#ifdef TK_TRACE
  const char* trace_file = getenv("TK_TRACE_FILE");
  const unsigned nblk = (unsigned)(ntiles + std::min<long long>(TK_TILE_LAG, ntiles) + 1);
  if (trace_file) {
    if (int rc = prof.alloc((size_t)nblk * 64, st)) return rc;
    TK_CUDA(cudaMemsetAsync(prof.get(), 0, (size_t)nblk * 64, st));
    p.prof = prof.as<unsigned long long>();
  }
#endif
  ktimer_begin(st);
  // block 0: the prefix scanner; block b counts tile b-1 and folds tile b-1-lag
  p.lag = std::min<long long>(TK_TILE_LAG, ntiles);
  p.out_v2 = p.out_nk == 2 && aligned16(p.out_subs);
  kern<<<(unsigned)(ntiles + p.lag + 1), kTileThreads, smem, st>>>(p);
  ktimer_end(st);
  count_launch();
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaMemcpyAsync(host_ctr, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  if (host_ctr->flags & kFlagStall)
    return fail(TK_ECUDA, "internal error: tile pipeline wait gave up (site " +
                              std::to_string(host_ctr->grab_ticket) + ", tile " +
                              std::to_string(host_ctr->tile_ticket) + ")");
#ifdef TK_TRACE
  if (trace_file) {
    std::vector<unsigned long long> h((size_t)nblk * 8);
    TK_CUDA(cudaMemcpy(h.data(), prof.get(), h.size() * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_file, "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
    p.prof = nullptr;
  }
#endif
  return TK_OK;
}

template <int SRC>
int launch_stream(SegParams& p, cudaStream_t st, Counters* host_ctr) {
  const int nk = SRC == kSrcLinKey ? 1 : p.nk;
  switch (nk) {
    case 1: return launch_stream_t<SRC, 1>(p, st, host_ctr);
    case 2: return launch_stream_t<SRC, 2>(p, st, host_ctr);
    case 3: return launch_stream_t<SRC, 3>(p, st, host_ctr);
    default: return launch_stream_t<SRC, 0>(p, st, host_ctr);
  }
}

// Run one segmented pass over a sorted stream; returns groups/zeros/flags in host_ctr.
int run_seg(int src, SegParams& p, cudaStream_t st, Counters* host_ctr) {
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  int rc = src == kSrcRaw     ? launch_stream<kSrcRaw>(p, st, hc)
           : src == kSrcKeysW ? launch_stream<kSrcKeysW>(p, st, hc)
                              : launch_stream<kSrcLinKey>(p, st, hc);
  if (rc) return rc;
  *host_ctr = *hc;
  return TK_OK;
}

int compact_zeros(long long groups, int nk, long long* out_subs, double* out_vals, cudaStream_t st) {
  const long long nblk = (groups + kCompTile - 1) / kCompTile;
  DevBuf blk, v2, s2;
  if (int rc = blk.alloc(nblk * 8, st)) return rc;
  if (int rc = v2.alloc(groups * 8, st)) return rc;
  if (int rc = s2.alloc(groups * 8 * std::max(nk, 1), st)) return rc;
  nz_count_kernel<<<(unsigned)nblk, 256, 0, st>>>(groups, out_vals, blk.as<long long>());
  scan_blocks_kernel<<<1, 256, 0, st>>>(nblk, blk.as<long long>());
  nz_scatter_kernel<<<(unsigned)nblk, 256, 0, st>>>(groups, nk, out_vals, out_subs, blk.as<long long>(),
                                                    v2.as<double>(), s2.as<long long>());
  count_launch(3);
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaMemcpyAsync(out_vals, v2.get(), groups * 8, cudaMemcpyDeviceToDevice, st));
  TK_CUDA(cudaMemcpyAsync(out_subs, s2.get(), groups * 8 * nk, cudaMemcpyDeviceToDevice, st));
  return TK_OK;
}

int finish(const Counters& c, int k, long long nx, int nk, long long* out_subs, double* out_vals,
           int64_t* out_nnz, cudaStream_t st, bool keep_zeros = false) {
  if (c.flags & kFlagIndex) {
    char buf[160];
    snprintf(buf, sizeof buf, "ttv: mode-%d index out of range for a vector of length %lld", k, nx);
    return fail(TK_EINDEX, buf);
  }
  if (keep_zeros) {
    *out_nnz = (int64_t)c.groups;
    return TK_OK;
  }
  if (c.zeros) {
    if (int rc = compact_zeros((long long)c.groups, nk, out_subs, out_vals, st)) return rc;
    TK_CUDA(cudaStreamSynchronize(st));
  }
  *out_nnz = (int64_t)(c.groups - c.zeros);
  return TK_OK;
}

// keys of kept modes must fit a signed 63-bit linear index
int lin_bits(const std::vector<long long>& dims) {
  unsigned __int128 prod = 1;
  for (long long dm : dims) {
    prod *= (unsigned __int128)dm;
    if (prod > ((unsigned __int128)1 << 62)) return -1;
  }
  int bits = 0;
  while (bits < 63 && ((unsigned __int128)1 << bits) < prod) ++bits;
  return std::max(bits, 1);
}

int ttv_general(int d, const int64_t* shape, long long nnz, const int64_t* const* cols, const double* vals,
                const double* x, long long nx, int k, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                cudaStream_t st, bool keep_zeros) {
  const int nk = d - 1;
  std::vector<long long> dims;
  KeepCols kc{};
  for (int m = 0, c = 0; m < d; ++m)
    if (m != k) {
      kc.col[c] = reinterpret_cast<const long long*>(cols[m]);
      kc.dims[c] = shape[m];
      dims.push_back(shape[m]);
      ++c;
    }
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  const int bits = lin_bits(dims);
  const int g = grid_for(nnz);

  DevBuf keys, keys2, w, w2, ctrbuf, temp;
  if (int rc = ctrbuf.alloc(sizeof(Counters), st)) return rc;
  Counters* dctr = ctrbuf.as<Counters>();
  TK_CUDA(cudaMemsetAsync(dctr, 0, sizeof(Counters), st));
  if (int rc = keys.alloc(nnz * 8, st)) return rc;
  if (int rc = keys2.alloc(nnz * 8, st)) return rc;
  if (int rc = w.alloc(nnz * 8, st)) return rc;
  if (int rc = w2.alloc(nnz * 8, st)) return rc;

  bool linear = bits > 0;
  if (linear) {
    prep_linkey_kernel2<<<g, 256, 0, st>>>(nnz, nk, kc, reinterpret_cast<const long long*>(cols[k]), vals, x, nx,
                                           keys.as<long long>(), w.as<double>(), dctr);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (hc->flags & kFlagIndex) return finish(*hc, k, nx, nk, nullptr, nullptr, out_nnz, st);
    if (hc->flags & kFlagKeptOob) linear = false;
  }

  Counters res{};
  if (linear) {
    cub::DoubleBuffer<long long> kb(keys.as<long long>(), keys2.as<long long>());
    cub::DoubleBuffer<double> vb(w.as<double>(), w2.as<double>());
    size_t tb = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)nnz, 0, bits, st));
    if (int rc = temp.alloc(tb, st)) return rc;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kb, vb, (int)nnz, 0, bits, st));
    SegParams p{};
    p.n = nnz;
    p.nk = 1;
    p.key[0] = kb.Current();
    p.a = vb.Current();
    p.out_nk = nk;
    for (int c = 0; c < nk; ++c) p.dims[c] = dims[c];
    p.out_subs = reinterpret_cast<long long*>(out_subs);
    p.out_vals = out_vals;
    p.bulk_ok = aligned16(p.key[0]) && aligned16(p.a);
    if (int rc = run_seg(kSrcLinKey, p, st, &res)) return rc;
    return finish(res, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
  }

  // LSD over kept columns, last column first, signed 64-bit keys, carrying the row permutation
  DevBuf perm, perm2, sorted_cols;
  if (int rc = perm.alloc(nnz * 8, st)) return rc;
  if (int rc = perm2.alloc(nnz * 8, st)) return rc;
  iota_kernel<<<g, 256, 0, st>>>(nnz, perm.as<long long>());
  cub::DoubleBuffer<long long> pb(perm.as<long long>(), perm2.as<long long>());
  {
    size_t tb = 0;
    cub::DoubleBuffer<long long> kb(keys.as<long long>(), keys2.as<long long>());
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, pb, (int)nnz, 0, 64, st));
    if (int rc = temp.alloc(tb, st)) return rc;
    for (int c = nk - 1; c >= 0; --c) {
      cub::DoubleBuffer<long long> kc2(keys.as<long long>(), keys2.as<long long>());
      gather_i64_kernel<<<g, 256, 0, st>>>(nnz, kc.col[c], pb.Current(), kc2.Current());
      TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kc2, pb, (int)nnz, 0, 64, st));
    }
  }
  if (int rc = sorted_cols.alloc((size_t)nnz * 8 * nk, st)) return rc;
  SegParams p{};
  p.n = nnz;
  p.nk = nk;
  for (int c = 0; c < nk; ++c) {
    long long* dst = sorted_cols.as<long long>() + (size_t)c * nnz;
    gather_i64_kernel<<<g, 256, 0, st>>>(nnz, kc.col[c], pb.Current(), dst);
    p.key[c] = dst;
  }
  gather_w_kernel<<<g, 256, 0, st>>>(nnz, pb.Current(), reinterpret_cast<const long long*>(cols[k]), vals, x, nx,
                                     w.as<double>(), dctr);
  TK_CUDA(cudaGetLastError());
  p.a = w.as<double>();
  p.out_nk = nk;
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  p.bulk_ok = 0;  // per-column offsets c*nnz need not be 16-byte aligned
  if (int rc = run_seg(kSrcKeysW, p, st, &res)) return rc;
  TK_CUDA(cudaMemcpyAsync(hc, dctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  res.flags |= hc->flags;
  return finish(res, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
}

}  // namespace

int ttv_prefix_try(int d, int64_t nnz, const int64_t* const* cols, const double* vals, const double* x, int64_t nx,
                   int64_t* out_subs, double* out_vals, int64_t* out_nnz, bool* unsorted, cudaStream_t st) {
  *out_nnz = 0;
  *unsorted = false;
  if (nnz == 0) return TK_OK;
  const int nk = d - 1, k = d - 1;
  SegParams p{};
  p.n = nnz;
  p.nk = nk;
  for (int c = 0; c < nk; ++c) p.key[c] = reinterpret_cast<const long long*>(cols[c]);
  p.subk = reinterpret_cast<const long long*>(cols[k]);
  p.a = vals;
  p.x = x;
  p.nx = nx;
  p.out_nk = nk;
  p.out_subs = reinterpret_cast<long long*>(out_subs);
  p.out_vals = out_vals;
  bool al = aligned16(vals) && aligned16(p.subk);
  for (int c = 0; c < nk; ++c) al = al && aligned16(p.key[c]);
  p.bulk_ok = al;
  Counters c{};
  if (int rc = run_seg(kSrcRaw, p, st, &c)) return rc;
  if ((c.flags & kFlagUnsorted) && !(c.flags & kFlagIndex)) {
    *unsorted = true;
    return TK_OK;
  }
  return finish(c, k, nx, nk, p.out_subs, out_vals, out_nnz, st);
}

int ttv_sparse_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                      const double* x, int64_t nx, int k, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                      cudaStream_t st, bool keep_zeros) {
  *out_nnz = 0;
  if (nnz == 0) return TK_OK;
  const int nk = d - 1;
  if (k == d - 1) {  // kept modes form a prefix: canonical input streams in sorted order
    SegParams p{};
    p.n = nnz;
    p.nk = nk;
    for (int c = 0; c < nk; ++c) p.key[c] = reinterpret_cast<const long long*>(cols[c]);
    p.subk = reinterpret_cast<const long long*>(cols[k]);
    p.a = vals;
    p.x = x;
    p.nx = nx;
    p.out_nk = nk;
    p.out_subs = reinterpret_cast<long long*>(out_subs);
    p.out_vals = out_vals;
    bool al = aligned16(vals) && aligned16(p.subk);
    for (int c = 0; c < nk; ++c) al = al && aligned16(p.key[c]);
    p.bulk_ok = al;
    Counters c{};
    if (int rc = run_seg(kSrcRaw, p, st, &c)) return rc;
    if (!(c.flags & kFlagUnsorted) || (c.flags & kFlagIndex))
      return finish(c, k, nx, nk, p.out_subs, out_vals, out_nnz, st, keep_zeros);
    // not canonical after all: fall through to the sort path
  }
  return ttv_general(d, shape, nnz, cols, vals, x, nx, k, out_subs, out_vals, out_nnz, st, keep_zeros);
}

int aos_to_soa(int64_t nnz, int d, const int64_t* aos, int64_t* soa, int64_t pitch, cudaStream_t st) {
  if (nnz == 0) return TK_OK;
  aos_to_soa_kernel<<<grid_for(nnz * d), 256, 0, st>>>(nnz, d, reinterpret_cast<const long long*>(aos),
                                                        reinterpret_cast<long long*>(soa), pitch);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

__global__ void scatter_dense_kernel(long long n, const long long* __restrict__ idx, const double* __restrict__ v,
                                     double* __restrict__ out, long long nout) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
    const long long i = idx[r];
    if (i >= 0 && i < nout) out[i] = v[r];
  }
}

int scatter_dense(long long n, const int64_t* idx, const double* v, double* out, long long nout, cudaStream_t st) {
  scatter_dense_kernel<<<grid_for(n), 256, 0, st>>>(n, reinterpret_cast<const long long*>(idx), v, out, nout);
  TK_CUDA(cudaGetLastError());
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

int ttv_dense_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                     int keep, const double* const* vecs, double* out, cudaStream_t st) {
  const long long nkeep = shape[keep];
  TK_CUDA(cudaMemsetAsync(out, 0, (size_t)nkeep * 8, st));
  if (nnz == 0) return TK_OK;
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  if (keep == 0) {
    constexpr int kItems = 4, TILE = kItems * 256;
    const long long ntiles = (nnz + TILE - 1) / TILE;
    DevBuf scratch;
    const size_t per = (size_t)ntiles * 8;
    if (int rc = scratch.alloc(per * 4 + 512, st)) return rc;
    DenseParams p{};
    p.n = nnz;
    p.d = d;
    p.keep = keep;
    bool al = aligned16(vals);
    for (int m = 0; m < d; ++m) {
      p.col[m] = reinterpret_cast<const long long*>(cols[m]);
      p.vec[m] = vecs[m];
      p.dims[m] = shape[m];
      al = al && aligned16(cols[m]);
    }
    p.vals = vals;
    p.out = out;
    char* b = scratch.as<char>();
    p.c_first = reinterpret_cast<double*>(b);
    p.c_last = reinterpret_cast<double*>(b + per);
    p.c_lastkey = reinterpret_cast<long long*>(b + 2 * per);
    p.c_flags = reinterpret_cast<int*>(b + 3 * per);
    p.ctr = reinterpret_cast<Counters*>(b + 4 * per + 128);
    p.bulk_ok = al;
    TK_CUDA(cudaMemsetAsync(p.ctr, 0, sizeof(Counters), st));
    const size_t smem = (size_t)(d + 1) * TILE * 8;
    auto kern = d == 3 ? dense_ttv_kernel<kItems, 3> : d == 4 ? dense_ttv_kernel<kItems, 4>
                : d == 5 ? dense_ttv_kernel<kItems, 5> : dense_ttv_kernel<kItems, 0>;
    set_smem_once(kern, smem);
    ktimer_begin(st);
    kern<<<(unsigned)ntiles, 256, smem, st>>>(p);
    ktimer_end(st);
    count_launch(2);
    dense_fixup_kernel<<<(unsigned)((ntiles + 255) / 256), 256, 0, st>>>(ntiles, p.c_first, p.c_last, p.c_lastkey,
                                                                         p.c_flags, nkeep, out);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaMemcpyAsync(hc, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    if (hc->flags & kFlagIndex) return fail(TK_EINDEX, "ttv: contracted-mode index out of range for its vector");
    if (hc->flags & kFlagKeptOob) return fail(TK_EDIM, "index out of bounds for shape");
    if (!(hc->flags & kFlagUnsorted)) return TK_OK;
    TK_CUDA(cudaMemsetAsync(out, 0, (size_t)nkeep * 8, st));
  }
  // chained single-mode TTV on the device, descending modes (the oracle's definition)
  std::vector<int64_t> cur_shape(shape, shape + d);
  std::vector<const int64_t*> cur_cols(cols, cols + d);
  const double* cur_vals = vals;
  long long cur_nnz = nnz;
  int cur_d = d, cur_keep = keep;
  DevBuf bufs[2][2];  // [ping][subs|vals]
  DevBuf soa;
  int ping = 0;
  for (int m = d - 1; m >= 0; --m) {
    if (m == keep) continue;
    const int nk = cur_d - 1;
    DevBuf& bs = bufs[ping][0];
    DevBuf& bv = bufs[ping][1];
    bs.reset();
    bv.reset();
    if (int rc = bs.alloc((size_t)std::max(cur_nnz, 1LL) * 8 * nk, st)) return rc;
    if (int rc = bv.alloc((size_t)std::max(cur_nnz, 1LL) * 8, st)) return rc;
    int64_t u = 0;
    if (int rc = ttv_sparse_device(cur_d, cur_shape.data(), cur_nnz, cur_cols.data(), cur_vals, vecs[m],
                                   shape[m], m, bs.as<int64_t>(), bv.as<double>(), &u, st))
      return rc;
    // row-major (u, nk) -> SoA for the next stage
    DevBuf nsoa;
    if (int rc = nsoa.alloc((size_t)std::max<int64_t>(u, 1) * 8 * nk, st)) return rc;
    if (int rc = aos_to_soa(u, nk, bs.as<int64_t>(), nsoa.as<int64_t>(), u, st)) return rc;
    soa.reset();
    std::swap(soa, nsoa);
    cur_shape.erase(cur_shape.begin() + m);
    cur_cols.clear();
    for (int c = 0; c < nk; ++c) cur_cols.push_back(soa.as<int64_t>() + (size_t)c * u);
    cur_vals = bv.as<double>();
    cur_nnz = u;
    cur_d = nk;
    if (m < cur_keep) --cur_keep;
    ping ^= 1;
  }
  // order-1 sparse result -> dense
  return cur_nnz ? scatter_dense(cur_nnz, cur_cols[0], cur_vals, out, nkeep, st) : TK_OK;
}

}  // namespace tk
