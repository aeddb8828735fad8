// tk_scan.cuh -- warp/block prefix sums and a device-wide exclusive scan (no library code).
#pragma once

#include "tk_common.cuh"

namespace tk {

template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exclusive prefix of v over the block's threads (in thread order); *total = block sum.
// `ws` is shared scratch of at least 33 elements.  Every thread of the block must call it.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T* ws, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const T inc = warp_incl_scan(v);
  if (lane == 31) ws[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const T t = lane < nw ? ws[lane] : T(0);
    const T ti = warp_incl_scan(t);
    if (lane < nw) ws[lane] = ti - t;
    if (lane == nw - 1) ws[32] = ti;
  }
  __syncthreads();
  const T r = ws[warp] + inc - v;
  *total = ws[32];
  __syncthreads();
  return r;
}

// Device-wide exclusive scan of n int64 values: out[i] = sum(in[0..i)), out[n] = total
// (out may alias in).  Three launches: block sums, one-block scan of the sums, block scans.
int scan_excl_i64(const long long* in, long long* out, long long n, cudaStream_t st);

}  // namespace tk
