// tk_mttkrp.cu -- sparse MTTKRP (matricised tensor times Khatri-Rao product) for sm_100a.
//
// M(i_n, r) = sum over nonzeros of  val * prod_{m != n} U_m(i_m, r)     (M: shape[n] x R, row-major)
//
// The R-column generalisation of the dense multi-vector TTV (column r of M is the TTV of every
// mode but n with the vectors U_m(:, r)); the paper names it as TTV's consumer (PAPER.md:18, 156,
// 273).  The reference has no MTTKRP, so the oracle is the reference's own chained
// single-mode ttv_raw per column (oracle/oracle.py mttkrp).
//
// Layout: factor matrices row-major (n_m x R), so one nonzero's gather U_m(i_m, 0:R) is R*8
// contiguous bytes -- a coalesced warp load, unlike the TTV's 8-byte random gathers.
//
// Kernel: one warp per span of kMtSpan rows in the kept mode's sorted order (canonical order when
// n == 0; otherwise a stable device radix sort of the row ids by subs[:, n] supplies `perm`).  A
// lane owns columns lane, lane+32, ... (RPL per lane).  The warp stages 32 rows' indices and values
// in shared memory (coalesced loads), then walks them in row order: broadcast reads, R-wide
// gathers, w = ((val * U_{d-1}) * ...) * U_1 in descending modes (the chained-TTV association), and
// a per-lane accumulator per column that is flushed at every key change.  Every column is thus a
// serial left fold in row order (deterministic).  Runs cut by span boundaries go to per-span
// carries, folded in span order by mttkrp_fixup_kernel (one writer per output element).
#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "tk_host.h"
#include "tk_common.cuh"

namespace tk {

namespace {

#ifndef TK_MT_SPAN
#define TK_MT_SPAN 1024
#endif
#ifndef TK_MT_BATCH
#define TK_MT_BATCH 4  // gathers issued per batch, in groups of rows (8: R=16 3.77 ms; 4: 3.28 ms; 2, 1: slower)
#endif
constexpr int kMtSpan = TK_MT_SPAN;  // rows per warp span (carry unit)
#ifndef TK_MT_THREADS
#define TK_MT_THREADS 256
#endif
constexpr int kMtThreads = TK_MT_THREADS;  // warps per CTA x 32
constexpr int kMtWarps = kMtThreads / 32;

struct MtParams {
  long long n;                     // rows
  int d;                           // order
  int mode;                        // kept mode n in the caller's numbering (column 0 here)
  long long R;                     // rank (columns)
  const long long* col[kMaxOrder];  // col[0]: the kept mode; col[1..d-1]: the others, ascending
  const double* vals;
  const long long* perm;           // row order (nullptr: identity, keys already sorted)
  const double* fac[kMaxOrder];    // U_m, row-major (dims[m] x R); fac[mode] unused
  long long dims[kMaxOrder];
  double* out;                     // shape[n] x R, zeroed by the host
  double* c_first;                 // [nspans][R]  leading piece of each span
  double* c_last;                  // [nspans][R]  trailing open piece
  long long* c_lastkey;            // [nspans]
  int* c_flags;                    // [nspans] bit0: span has a head, bit1: last run continues
  Counters* ctr;
};

// D: tensor order (2..5, gathers unrolled) or 0 (any order).  RP: lanes per row (a power of two
// >= R for R <= 32, so a warp step covers G = 32/RP rows); RPL: columns per lane (R > 32, RP = 32).
// Slot s = lane / RP handles rows j0+s of each G-row group and keeps its own partial of the open
// run; a group with a head reduces the slot partials (xor butterfly over the slot bits) and walks
// the group's rows in order, so each column is folded in a fixed order (deterministic).
template <int D, int RP, int RPL, bool PERM>
__global__ void __launch_bounds__(kMtThreads) mttkrp_kernel(MtParams p, long long nspans) {
  constexpr int DM = D > 0 ? D : kMaxOrder;
  constexpr int G = 32 / RP;
  // groups per gather batch (narrow rows, RP <= 4: twice as many -- a group is only 4 gathers wide)
  constexpr int BT = RP <= 4 ? 2 * TK_MT_BATCH : TK_MT_BATCH;
  constexpr int B = BT / RPL > 0 ? BT / RPL : 1;
  static_assert(RP == 32 || RPL == 1, "several columns per lane only with full-warp rows");
  __shared__ long long s_off[kMtWarps][DM][32];  // factor-row offsets idx*R (column 0 unused)
  __shared__ long long s_key[kMtWarps][32];
  __shared__ double s_val[kMtWarps][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int slot = lane / RP, cl = lane % RP;
  const int d = D > 0 ? D : p.d;
  const long long R = p.R;
  const unsigned long long nkeep = (unsigned long long)p.dims[0];  // the kept mode is column 0
  const long long W = ((long long)gridDim.x * blockDim.x) >> 5;
  unsigned int flags = 0;
  auto row_of = [&](long long q) { return PERM ? p.perm[q] : q; };
  auto reduce_slots = [&](double v) {
#pragma unroll
    for (int o = RP; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;  // identical in every slot (RN addition commutes)
  };

  for (long long sp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sp < nspans; sp += W) {
    const long long s0 = sp * kMtSpan, s1 = min(s0 + kMtSpan, p.n);
    long long curkey = s0 > 0 ? p.col[0][row_of(s0 - 1)] : 0;
    double acc[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) acc[q] = 0.0;
    bool seen = false;
    // a run closes at a head: the span's first closing before any head is its leading carry
    auto flush = [&](long long key, const double* tot) {
      if (slot != 0) return;
      if (!seen) {
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const long long c = cl + 32 * q;
          if (c < R) p.c_first[sp * R + c] = tot[q];
        }
      } else if ((unsigned long long)key < nkeep) {
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
          const long long c = cl + 32 * q;
          if (c < R) p.out[key * R + c] = tot[q];
        }
      }
    };
    for (long long b = s0; b < s1; b += 32) {
      // stage 32 rows (coalesced loads; the permuted path reads through perm).  Per row, once:
      // the factor-row offsets idx*R (bounds-checked: an out-of-range index raises and is never
      // read), the head bit (key change) and the order / kept-bounds checks.
      const long long q0 = b + lane;
      const bool ok = q0 < s1;
      long long key = curkey;
      if (ok) {
        const long long row = row_of(q0);
        key = p.col[0][row];
#pragma unroll
        for (int m = 1; m < DM; ++m) {
          if (D == 0 && m >= d) break;
          const long long idx = p.col[m][row];
          const bool bad = (unsigned long long)idx >= (unsigned long long)p.dims[m];
          if (bad) flags |= kFlagIndex;
          s_off[wib][m][lane] = (bad ? 0 : idx) * R;
        }
        s_val[wib][lane] = p.vals[row];
      }
      long long prev = __shfl_up_sync(0xffffffffu, key, 1);
      if (lane == 0) prev = curkey;
      const bool head = ok && (q0 == 0 || key != prev);
      if (head && q0 > 0 && key < prev) flags |= kFlagUnsorted;
      if (head && (unsigned long long)key >= nkeep) flags |= kFlagKeptOob;
      const unsigned int hmask = __ballot_sync(0xffffffffu, head);
      s_key[wib][lane] = key;
      __syncwarp();
      const int cnt = (int)min(32LL, s1 - b);
      for (int j0 = 0; j0 < cnt; j0 += B * G) {
        // every gather of the batch (B groups of G rows) in flight before the first product
        double g[B][RPL][DM];
#pragma unroll
        for (int bb = 0; bb < B; ++bb) {
          const int j = min(j0 + bb * G + slot, cnt - 1);  // past the block: a repeated row, unused
#pragma unroll
          for (int m = 1; m < DM; ++m) {
            if (D == 0 && m >= d) break;
            const double* row = p.fac[m] + s_off[wib][m][j];
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
              const long long c = cl + 32 * q;
              g[bb][q][m] = c < R ? __ldg(row + c) : 0.0;
            }
          }
        }
#pragma unroll
        for (int bb = 0; bb < B; ++bb) {
          const int jg = j0 + bb * G;  // first row of the group
          if (jg >= cnt) break;
          const int j = jg + slot;
          const double v = j < cnt ? s_val[wib][j] : 0.0;
          double w[RPL];
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            w[q] = v;
#pragma unroll
            for (int m = DM - 1; m >= 1; --m) {  // descending modes: the chained-TTV association
              if (D == 0 && m >= d) continue;
              w[q] = __dmul_rn(w[q], g[bb][q][m]);
            }
          }
          const unsigned int gm = (hmask >> jg) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
          if (gm == 0) {
#pragma unroll
            for (int q = 0; q < RPL; ++q) acc[q] = __dadd_rn(acc[q], w[q]);
            continue;
          }
          // the group holds a head: slot partials -> one total, then the rows in order
          double tot[RPL];
#pragma unroll
          for (int q = 0; q < RPL; ++q) tot[q] = reduce_slots(acc[q]);
#pragma unroll
          for (int s = 0; s < G; ++s) {
            if (jg + s >= cnt) break;
            double ws[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q) ws[q] = __shfl_sync(0xffffffffu, w[q], s * RP + cl);
            if ((gm >> s) & 1u) {
              flush(curkey, tot);
              seen = true;
              curkey = s_key[wib][jg + s];
#pragma unroll
              for (int q = 0; q < RPL; ++q) tot[q] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < RPL; ++q) tot[q] = __dadd_rn(tot[q], ws[q]);
          }
#pragma unroll
          for (int q = 0; q < RPL; ++q) acc[q] = slot == 0 ? tot[q] : 0.0;
        }
      }
      curkey = s_key[wib][cnt - 1];
      __syncwarp();
    }
    // span end: the trailing run is closed here unless the next row continues it
    double tot[RPL];
#pragma unroll
    for (int q = 0; q < RPL; ++q) tot[q] = reduce_slots(acc[q]);
    const bool last_open = s1 < p.n && p.col[0][row_of(s1)] == curkey;
    if (!seen || !last_open) {
      flush(curkey, tot);  // !seen: the whole span continues the run open at its start
    } else if (slot == 0) {
#pragma unroll
      for (int q = 0; q < RPL; ++q) {
        const long long c = cl + 32 * q;
        if (c < R) p.c_last[sp * R + c] = tot[q];
      }
      if (lane == 0) p.c_lastkey[sp] = curkey;
    }
    if (lane == 0) p.c_flags[sp] = (seen ? 1 : 0) | (last_open ? 2 : 0);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0 && flags) atomicOr(&p.ctr->flags, flags);
}

// One thread per (span, column): a span whose last run stays open sums the leading pieces of the
// following spans, in span order, until the run closes.
__global__ void mttkrp_fixup_kernel(long long nspans, long long R, const double* __restrict__ c_first,
                                    const double* __restrict__ c_last, const long long* __restrict__ c_lastkey,
                                    const int* __restrict__ c_flags, long long nkeep, double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nspans * R) return;
  const long long sp = t / R, c = t % R;
  if ((c_flags[sp] & 3) != 3) return;
  double s = c_last[sp * R + c];
  for (long long s2 = sp + 1; s2 < nspans; ++s2) {
    s = __dadd_rn(s, c_first[s2 * R + c]);
    const int f2 = c_flags[s2];
    if ((f2 & 1) || !(f2 & 2)) break;
  }
  const long long k = c_lastkey[sp];
  if (k >= 0 && k < nkeep) out[k * R + c] = s;
}

__global__ void iota_kernel(long long n, long long* __restrict__ v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] = i;
}

template <int D, int RP, int RPL>
void* pick_mt(bool perm) {
  return perm ? reinterpret_cast<void*>(mttkrp_kernel<D, RP, RPL, true>)
              : reinterpret_cast<void*>(mttkrp_kernel<D, RP, RPL, false>);
}

// rank -> (lanes per row, columns per lane) instance for an order-D tensor
template <int D>
void* pick_mt_r(long long R, bool perm) {
  if (R > 64) return pick_mt<D, 32, 4>(perm);
  if (R > 32) return pick_mt<D, 32, 2>(perm);
  if (D == 0 || R > 16) return pick_mt<D, 32, 1>(perm);
  if (R > 8) return pick_mt<D == 0 ? 2 : D, 16, 1>(perm);
  if (R > 4) return pick_mt<D == 0 ? 2 : D, 8, 1>(perm);
  return pick_mt<D == 0 ? 2 : D, 4, 1>(perm);
}

int launch_mttkrp(MtParams& p, bool perm, cudaStream_t st, unsigned int* flags_out) {
  const long long nspans = (p.n + kMtSpan - 1) / kMtSpan;
  const size_t per = ((size_t)nspans * p.R * 8 + 255) & ~size_t(255);
  const size_t perk = ((size_t)nspans * 8 + 255) & ~size_t(255);
  DevBuf scratch;
  if (int rc = scratch.alloc(2 * per + 2 * perk + 256, st)) return rc;
  char* b = scratch.as<char>();
  p.c_first = reinterpret_cast<double*>(b);
  p.c_last = reinterpret_cast<double*>(b + per);
  p.c_lastkey = reinterpret_cast<long long*>(b + 2 * per);
  p.c_flags = reinterpret_cast<int*>(b + 2 * per + perk);
  p.ctr = reinterpret_cast<Counters*>(b + 2 * per + 2 * perk);
  TK_CUDA(cudaMemsetAsync(p.ctr, 0, sizeof(Counters), st));
  void* kern = p.d == 2 ? pick_mt_r<2>(p.R, perm) : p.d == 3 ? pick_mt_r<3>(p.R, perm)
               : p.d == 4 ? pick_mt_r<4>(p.R, perm) : p.d == 5 ? pick_mt_r<5>(p.R, perm)
                                                     : pick_mt_r<0>(p.R, perm);
  const long long warps = std::min(nspans, (long long)num_sms() * 8 * kMtWarps);
  const unsigned blocks = (unsigned)((warps + kMtWarps - 1) / kMtWarps);
  void* args[] = {&p, const_cast<long long*>(&nspans)};
  ktimer_begin(st);
  TK_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(kMtThreads), args, 0, st));
  const long long nfix = nspans * p.R;
  mttkrp_fixup_kernel<<<(unsigned)((nfix + 255) / 256), 256, 0, st>>>(nspans, p.R, p.c_first, p.c_last,
                                                                       p.c_lastkey, p.c_flags, p.dims[0], p.out);
  ktimer_end(st);
  count_launch(2);
  TK_CUDA(cudaGetLastError());
  Counters* hc = static_cast<Counters*>(pinned_scratch(sizeof(Counters)));
  TK_CUDA(cudaMemcpyAsync(hc, p.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  *flags_out = hc->flags;
  return TK_OK;
}

}  // namespace

int mttkrp_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals, int mode,
                  int64_t R, const double* const* factors, double* out, cudaStream_t st) {
  TK_CUDA(cudaMemsetAsync(out, 0, (size_t)shape[mode] * R * 8, st));
  if (nnz == 0 || R == 0) return TK_OK;
  MtParams p{};
  p.n = nnz;
  p.d = d;
  p.mode = mode;
  p.R = R;
  // kept mode first, then the others in ascending order: the kernel's descending walk over
  // columns 1..d-1 is then the chained-TTV association (descending modes, skipping n)
  for (int m = 0, c = 1; m < d; ++m) {
    const int q = m == mode ? 0 : c++;
    p.col[q] = reinterpret_cast<const long long*>(cols[m]);
    p.fac[q] = factors[m];
    p.dims[q] = shape[m];
  }
  p.vals = vals;
  p.out = out;
  unsigned int flags = 0;
  DevBuf keys_s, perm_in, perm_s, temp;
  if (mode == 0) {  // canonical tensors stream in kept-key order: no sort
    if (int rc = launch_mttkrp(p, false, st, &flags)) return rc;
  } else {
    flags = kFlagUnsorted;
  }
  if (flags & kFlagIndex) return fail(TK_EINDEX, "mttkrp: factor row index out of range for its factor matrix");
  if ((flags & kFlagUnsorted) && !(flags & kFlagKeptOob)) {
    // stable radix sort of the row ids by the kept mode (original row order inside each key)
    TK_CUDA(cudaMemsetAsync(out, 0, (size_t)shape[mode] * R * 8, st));
    int bits = 1;
    while (bits < 63 && (1LL << bits) < shape[mode]) ++bits;
    if (int rc = keys_s.alloc((size_t)nnz * 8, st)) return rc;
    if (int rc = perm_in.alloc((size_t)nnz * 8, st)) return rc;
    if (int rc = perm_s.alloc((size_t)nnz * 8, st)) return rc;
    iota_kernel<<<std::max(1, std::min((int)((nnz + 255) / 256), num_sms() * 8)), 256, 0, st>>>(
        nnz, perm_in.as<long long>());
    count_launch();
    size_t tb = 0;
    const unsigned long long* kin = reinterpret_cast<const unsigned long long*>(cols[mode]);
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin, keys_s.as<unsigned long long>(),
                                            perm_in.as<long long>(), perm_s.as<long long>(), (int)nnz, 0, bits, st));
    if (int rc = temp.alloc(tb, st)) return rc;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kin, keys_s.as<unsigned long long>(),
                                            perm_in.as<long long>(), perm_s.as<long long>(), (int)nnz, 0, bits, st));
    count_launch();
    p.perm = perm_s.as<long long>();
    if (int rc = launch_mttkrp(p, true, st, &flags)) return rc;
    if (flags & kFlagIndex) return fail(TK_EINDEX, "mttkrp: factor row index out of range for its factor matrix");
  }
  if (flags & kFlagKeptOob) return fail(TK_EDIM, "index out of bounds for shape");
  return TK_OK;
}

}  // namespace tk
