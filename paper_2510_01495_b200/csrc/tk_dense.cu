// tk_dense.cu -- dot and row-major matvec for sm_100a (FP64, HBM-bound streams).
//
// Reference: _dot_impl / _matvec_impl, pkg/src/tenkern/_ckernels.pyx:40-56 (one scalar
// accumulator, left to right).  A single dependency chain over 1e6 adds cannot use a GPU,
// so both kernels reduce in a fixed tree order: grid-stride 128-bit loads, per-thread
// partial sums, warp-shuffle butterflies, a fixed-order block and grid combine.  The
// result is deterministic run to run and within 1e-12 relative of the reference's
// left-to-right sum (north-star tolerance; exact on the reference's pinned examples).
// Products and sums are explicit __dmul_rn / __dadd_rn (no FMA contraction), as in the
// reference build (pkg/setup.py:4-13).
#include <algorithm>

#include "tk_host.h"
#include "tk_common.cuh"

namespace tk {

namespace {
constexpr int kDotThreads = 256;
#ifndef TK_DOT_UNROLL
#define TK_DOT_UNROLL 8  // 16-byte load pairs in flight per thread (config 1: 245 CTAs; 2 and 4: 12.9 us, 8-16: 10.9 us)
#endif
constexpr int kDotUnroll = TK_DOT_UNROLL;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double block_sum(double v, double* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) s_warp[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in warp 0
}
}  // namespace

// Single pass: every CTA streams its grid-stride share with all kDotUnroll 16-byte load pairs in
// flight, reduces it (warp butterflies, fixed warp order), stores its partial and takes a ticket;
// the last CTA to finish sums the partials in CTA-index order (thread t takes t, t+256, ...; then
// the same block tree), so the result does not depend on which CTA finished when.  The ticket
// word is zeroed by the host (cudaMemsetAsync) before the launch.
__global__ void __launch_bounds__(kDotThreads) dot_kernel(const double* __restrict__ x,
                                                          const double* __restrict__ y, long long n,
                                                          double* __restrict__ partial,
                                                          unsigned int* __restrict__ ticket,
                                                          double* __restrict__ out, int vec2) {
  __shared__ double s_warp[kDotThreads / 32];
  __shared__ bool s_last;
  double acc = 0.0;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (vec2) {
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* y2 = reinterpret_cast<const double2*>(y);
    const long long n2 = n >> 1;
    long long i = tid;
    for (; i + (kDotUnroll - 1) * stride < n2; i += kDotUnroll * stride) {
      double2 a[kDotUnroll], b[kDotUnroll];
#pragma unroll
      for (int u = 0; u < kDotUnroll; ++u) {
        a[u] = __ldcs(x2 + i + u * stride);
        b[u] = __ldcs(y2 + i + u * stride);
      }
#pragma unroll
      for (int u = 0; u < kDotUnroll; ++u) {
        acc = __dadd_rn(acc, __dmul_rn(a[u].x, b[u].x));
        acc = __dadd_rn(acc, __dmul_rn(a[u].y, b[u].y));
      }
    }
    {  // remainder: fewer than kDotUnroll strides left, still all loads first
      double2 a[kDotUnroll - 1], b[kDotUnroll - 1];
#pragma unroll
      for (int u = 0; u < kDotUnroll - 1; ++u) {
        const bool ok = i + u * stride < n2;
        a[u] = ok ? __ldcs(x2 + i + u * stride) : make_double2(0.0, 0.0);
        b[u] = ok ? __ldcs(y2 + i + u * stride) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kDotUnroll - 1; ++u) {
        if (i + u * stride < n2) {
          acc = __dadd_rn(acc, __dmul_rn(a[u].x, b[u].x));
          acc = __dadd_rn(acc, __dmul_rn(a[u].y, b[u].y));
        }
      }
    }
    if ((n & 1) && tid == 0) acc = __dadd_rn(acc, __dmul_rn(x[n - 1], y[n - 1]));
  } else {
    for (long long i = tid; i < n; i += stride) acc = __dadd_rn(acc, __dmul_rn(x[i], y[i]));
  }
  const double s = block_sum(acc, s_warp);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = s;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) t = __dadd_rn(t, __ldcg(partial + b));
  __syncthreads();  // s_warp reuse
  const double r = block_sum(t, s_warp);
  if (threadIdx.x == 0) *out = r;
}

// One warp per row; 128-bit loads of the row (streamed), x through the read-only path (L1
// resident after the first rows).  The warp butterfly fixes the combine order.
#ifndef TK_MV_UNROLL
#define TK_MV_UNROLL 8
#endif
#ifndef TK_MV_WARPS
#define TK_MV_WARPS 8
#endif
constexpr int kMvWarps = TK_MV_WARPS;
constexpr int kMvUnroll = TK_MV_UNROLL;

__global__ void __launch_bounds__(kMvWarps * 32) matvec_kernel(const double* __restrict__ a, long long rows,
                                                                long long cols, const double* __restrict__ x,
                                                                double* __restrict__ y, int vec2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long row = (long long)blockIdx.x * kMvWarps + warp;
  if (row >= rows) return;
  const double* ar = a + row * cols;
  double acc = 0.0;
  if (vec2) {
    const double2* a2 = reinterpret_cast<const double2*>(ar);
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const long long c2 = cols >> 1;
    long long j = lane;
    for (; j + (kMvUnroll - 1) * 32 < c2; j += kMvUnroll * 32) {
      double2 av[kMvUnroll], xv[kMvUnroll];
#pragma unroll
      for (int u = 0; u < kMvUnroll; ++u) {
        av[u] = __ldcs(a2 + j + u * 32);
        xv[u] = __ldg(x2 + j + u * 32);
      }
#pragma unroll
      for (int u = 0; u < kMvUnroll; ++u) {
        acc = __dadd_rn(acc, __dmul_rn(av[u].x, xv[u].x));
        acc = __dadd_rn(acc, __dmul_rn(av[u].y, xv[u].y));
      }
    }
    for (; j < c2; j += 32) {
      const double2 av = __ldcs(a2 + j), xv = __ldg(x2 + j);
      acc = __dadd_rn(acc, __dmul_rn(av.x, xv.x));
      acc = __dadd_rn(acc, __dmul_rn(av.y, xv.y));
    }
    if ((cols & 1) && lane == 0) acc = __dadd_rn(acc, __dmul_rn(ar[cols - 1], x[cols - 1]));
  } else {
    for (long long j = lane; j < cols; j += 32) acc = __dadd_rn(acc, __dmul_rn(ar[j], __ldg(x + j)));
  }
  acc = warp_sum(acc);
  if (lane == 0) y[row] = acc;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int dot_blocks(long long n) {
  // one grid-stride round of kDotUnroll 16-byte load pairs per thread when that fits eight
  // 256-thread CTAs per SM (config 1: 245 CTAs, every load of the call in flight at once)
  const long long want = (n + 2LL * kDotThreads * kDotUnroll - 1) / (2LL * kDotThreads * kDotUnroll);
  return (int)std::max(1LL, std::min(want, (long long)num_sms() * 8));
}

int dot_device(const double* x, const double* y, int64_t n, double* out, cudaStream_t st) {
  if (n == 0) {
    TK_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    return TK_OK;
  }
  const int nblk = dot_blocks(n);
  DevBuf part;  // [ticket (8 B) | partials]
  if (int rc = part.alloc((size_t)(nblk + 1) * sizeof(double), st)) return rc;
  TK_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double), st));
  const int vec2 = al16(x) && al16(y);
  ktimer_begin(st);
  dot_kernel<<<nblk, kDotThreads, 0, st>>>(x, y, n, part.as<double>() + 1, part.as<unsigned int>(), out, vec2);
  ktimer_end(st);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

// Measurement floor (not a reference kernel): read n doubles with the dot kernel's access pattern
// and launch shape -- every 16-byte load of the call in flight at once, a per-thread sum, one store
// per CTA, no cross-CTA combine.  Timed under the same L2 flush as dot / matvec / the small TTV,
// it is the cold-read time of those byte counts on this GPU (bench.py secondary "floor").
__global__ void __launch_bounds__(kDotThreads) read_floor_kernel(const double2* __restrict__ p, long long n2,
                                                                 double* __restrict__ sink) {
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long i = tid; i < n2; i += kDotUnroll * stride) {
    double2 a[kDotUnroll];
#pragma unroll
    for (int u = 0; u < kDotUnroll; ++u) a[u] = i + u * stride < n2 ? __ldcs(p + i + u * stride) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < kDotUnroll; ++u) acc = __dadd_rn(acc, __dadd_rn(a[u].x, a[u].y));
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc == 1.2345e300) sink[blockIdx.x] = acc;  // keeps the loads alive
}

int read_floor_device(const double* p, int64_t n, double* sink, cudaStream_t st) {
  if (n < 2) return TK_OK;
  const long long n2 = n >> 1;
  const long long want = (n2 + (long long)kDotThreads * kDotUnroll - 1) / ((long long)kDotThreads * kDotUnroll);
  const int nblk = (int)std::max(1LL, std::min(want, (long long)num_sms() * 8));
  ktimer_begin(st);
  read_floor_kernel<<<nblk, kDotThreads, 0, st>>>(reinterpret_cast<const double2*>(p), n2, sink);
  ktimer_end(st);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

int matvec_device(const double* a, int64_t rows, int64_t cols, const double* x, double* y, cudaStream_t st) {
  if (rows == 0) return TK_OK;
  const int vec2 = al16(a) && al16(x) && (cols % 2 == 0);
  const long long nblk = (rows + kMvWarps - 1) / kMvWarps;
  ktimer_begin(st);
  matvec_kernel<<<(unsigned)nblk, kMvWarps * 32, 0, st>>>(a, rows, cols, x, y, vec2);
  ktimer_end(st);
  count_launch();
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

}  // namespace tk
