// tk_gen.cu -- synthetic COO operands generated on the device (measurement inputs).
//
// BASELINE configs 4 and 5 (1e8 / 4e8 distinct coordinates) are far outside what the
// reference's host generator (numpy, synth.py:103-143) can produce inside a bench run, so
// they are generated here with the same exact-nnz semantics:
//   * draw i (i = 0, 1, 2, ...) is a d-tuple whose mode-m coordinate comes from a
//     counter-based Philox4x32-10 stream (key = seed, counter = (i, m)): uniform on
//     {0..n_m-1}, or truncated Zipf(s) (P(v) ~ (v+1)^-s, v < n_m) by inverse CDF;
//   * the tensor is the set of the FIRST nnz DISTINCT tuples of that sequence, i.e.
//     sampling without replacement until the count is exact -- the reference's top-up
//     protocol ("draw, dedupe, top up until exactly nnz", synth.py:124-131);
//   * coordinates are emitted in canonical (lexicographic) order as SoA columns;
//   * values are a function of the coordinate (Philox keyed by seed^kValSalt): uniform
//     [0,1) or N(0,1) (Box-Muller), exact zeros redrawn (synth.py:133-138).
// Implementation: M draws -> stable radix sort of (linear key, draw index) -> first
// occurrence of each key -> if fewer than nnz distinct, grow M and redraw (deterministic);
// else keep the keys whose first draw index is among the nnz smallest.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "tk_common.cuh"
#include "tk_host.h"

namespace tk {

namespace {

constexpr uint64_t kValSalt = 0x9E3779B97F4A7C15ull;

struct Philox {
  __device__ __forceinline__ static uint4 round10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const unsigned int hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
      const unsigned int hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

// 53-bit uniform in [0,1) from two 32-bit words
__device__ __forceinline__ double u53(unsigned int a, unsigned int b) {
  const unsigned long long v = ((unsigned long long)a << 21) ^ (unsigned long long)(b >> 11);
  return (double)(v & ((1ull << 53) - 1)) * 0x1.0p-53;
}

struct GenParams {
  int d;
  long long dims[kMaxOrder];
  long long stride[kMaxOrder];
  const double* cdf[kMaxOrder];  // nullptr -> uniform mode
  uint2 key;
};

__device__ __forceinline__ long long draw_coord(const GenParams& p, unsigned long long i, int m) {
  const uint4 c = Philox::round10(make_uint4((unsigned)i, (unsigned)(i >> 32), (unsigned)m, 0x7A11u), p.key);
  const double u = u53(c.x, c.y);
  const long long n = p.dims[m];
  if (p.cdf[m] == nullptr) {
    long long v = (long long)(u * (double)n);
    return v < n ? v : n - 1;
  }
  // first index with cdf[idx] > u
  const double* cdf = p.cdf[m];
  long long lo = 0, hi = n - 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (__ldg(cdf + mid) > u) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__global__ void draw_kernel(GenParams p, unsigned long long m0, long long count, unsigned long long* __restrict__ keys,
                            unsigned int* __restrict__ idx) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    const unsigned long long i = m0 + t;
    unsigned long long lin = 0;
    for (int m = 0; m < p.d; ++m) lin += (unsigned long long)draw_coord(p, i, m) * (unsigned long long)p.stride[m];
    keys[t] = lin;
    idx[t] = (unsigned int)i;
  }
}

__global__ void first_flag_kernel(long long n, const unsigned long long* __restrict__ keys,
                                  unsigned char* __restrict__ flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    flag[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1 : 0;
}

__global__ void le_flag_kernel(long long n, const unsigned int* __restrict__ idx, const unsigned int* __restrict__ thr,
                               unsigned char* __restrict__ flag) {
  const unsigned int T = *thr;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    flag[t] = idx[t] <= T ? 1 : 0;
}

struct ColPtrs {
  long long* col[kMaxOrder];
};

// ---- N(0,1) values from exactly-rounded operations only -----------------------------------
// Box-Muller with its own ln and cos built from IEEE +, -, *, / and sqrt, each an explicit
// round-to-nearest intrinsic (no FMA contraction, no libdevice approximation).  The host twin of
// this generator (oracle/tk_gen_host.cpp) performs the same operation sequence, so device- and
// host-generated tensors are byte-identical (tests/test_gen_twin.py).
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }

// ln(x), x in [2^-53, 1]: x = 2^e m, m in [sqrt(1/2), sqrt(2)); ln m = 2 atanh(f) with
// f = (m - 1) / (m + 1) (|f| <= 0.172), odd series to f^23.
__device__ double gen_ln(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((long long)((b & 0xFFFFFFFFFFFFFull) | (1023ull << 52)));
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = rn_mul(m, 0.5);
    e += 1;
  }
  const double f = __ddiv_rn(rn_sub(m, 1.0), rn_add(m, 1.0));
  const double s = rn_mul(f, f);
  double q = 0x1.642c8590b2164p-5;                  // 1/23
  q = rn_add(0x1.8618618618618p-5, rn_mul(s, q));   // 1/21
  q = rn_add(0x1.af286bca1af28p-5, rn_mul(s, q));   // 1/19
  q = rn_add(0x1.e1e1e1e1e1e1ep-5, rn_mul(s, q));   // 1/17
  q = rn_add(0x1.1111111111111p-4, rn_mul(s, q));   // 1/15
  q = rn_add(0x1.3b13b13b13b14p-4, rn_mul(s, q));   // 1/13
  q = rn_add(0x1.745d1745d1746p-4, rn_mul(s, q));   // 1/11
  q = rn_add(0x1.c71c71c71c71cp-4, rn_mul(s, q));   // 1/9
  q = rn_add(0x1.2492492492492p-3, rn_mul(s, q));   // 1/7
  q = rn_add(0x1.999999999999ap-3, rn_mul(s, q));   // 1/5
  q = rn_add(0x1.5555555555555p-2, rn_mul(s, q));   // 1/3
  const double f2 = rn_add(f, f);
  const double lm = rn_add(f2, rn_mul(rn_mul(f2, s), q));
  return rn_add(rn_mul((double)e, 0x1.62e42fefa39efp-1), lm);  // e ln 2 + ln m
}

// cos y and sin y for y in [0, pi/4]: Taylor to y^16 / y^17, Horner in z = y^2
__device__ double gen_cos_q(double y) {
  const double z = rn_mul(y, y);
  double q = 0x1.ae7f3e733b81fp-45;                 // 1/16!
  q = rn_sub(0x1.93974a8c07c9dp-37, rn_mul(z, q));  // 1/14!
  q = rn_sub(0x1.1eed8eff8d898p-29, rn_mul(z, q));  // 1/12!
  q = rn_sub(0x1.27e4fb7789f5cp-22, rn_mul(z, q));  // 1/10!
  q = rn_sub(0x1.a01a01a01a01ap-16, rn_mul(z, q));  // 1/8!
  q = rn_sub(0x1.6c16c16c16c17p-10, rn_mul(z, q));  // 1/6!
  q = rn_sub(0x1.5555555555555p-5, rn_mul(z, q));   // 1/4!
  q = rn_sub(0.5, rn_mul(z, q));                    // 1/2!
  return rn_sub(1.0, rn_mul(z, q));
}
__device__ double gen_sin_q(double y) {
  const double z = rn_mul(y, y);
  double q = 0x1.952c77030ad4ap-49;                 // 1/17!
  q = rn_sub(0x1.ae7f3e733b81fp-41, rn_mul(z, q));  // 1/15!
  q = rn_sub(0x1.6124613a86d09p-33, rn_mul(z, q));  // 1/13!
  q = rn_sub(0x1.ae64567f544e4p-26, rn_mul(z, q));  // 1/11!
  q = rn_sub(0x1.71de3a556c734p-19, rn_mul(z, q));  // 1/9!
  q = rn_sub(0x1.a01a01a01a01ap-13, rn_mul(z, q));  // 1/7!
  q = rn_sub(0x1.1111111111111p-7, rn_mul(z, q));   // 1/5!
  q = rn_sub(0x1.5555555555555p-3, rn_mul(z, q));   // 1/3!
  return rn_sub(y, rn_mul(rn_mul(y, z), q));
}

// cos(2 pi t), t in [0, 1): exact reductions (Sterbenz) to t in [0, 1/8] or [1/8, 1/4], then the
// cosine or sine polynomial
__device__ double gen_cos2pi(double t) {
  double sign = 1.0;
  if (t > 0.5) t = rn_sub(1.0, t);
  if (t > 0.25) {
    t = rn_sub(0.5, t);
    sign = -1.0;
  }
  const double c = t > 0.125 ? gen_sin_q(rn_mul(0x1.921fb54442d18p+2, rn_sub(0.25, t)))
                             : gen_cos_q(rn_mul(0x1.921fb54442d18p+2, t));
  return rn_mul(sign, c);
}

__global__ void unravel_vals_kernel(GenParams p, long long n, const unsigned long long* __restrict__ keys,
                                    int normal_vals, ColPtrs cp, double* __restrict__ vals) {
  const uint2 vk = make_uint2(p.key.x ^ (unsigned)kValSalt, p.key.y ^ (unsigned)(kValSalt >> 32));
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    unsigned long long lin = keys[t];
    for (int m = p.d - 1; m >= 0; --m) {
      const unsigned long long dm = (unsigned long long)p.dims[m];
      cp.col[m][t] = (long long)(lin % dm);
      lin /= dm;
    }
    const unsigned long long key = keys[t];
    double v = 0.0;
    for (unsigned int attempt = 0; v == 0.0; ++attempt) {
      const uint4 c = Philox::round10(make_uint4((unsigned)key, (unsigned)(key >> 32), attempt, 0xBA15u), vk);
      if (!normal_vals) {
        v = u53(c.x, c.y);
      } else {
        const double u1 = rn_sub(1.0, u53(c.x, c.y));  // (0, 1], exact
        const double u2 = u53(c.z, c.w);
        v = rn_mul(__dsqrt_rn(rn_mul(-2.0, gen_ln(u1))), gen_cos2pi(u2));
      }
    }
    vals[t] = v;
  }
}

__global__ void uniform_kernel(long long n, uint2 key, double* __restrict__ out) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const uint4 c = Philox::round10(make_uint4((unsigned)t, (unsigned)(t >> 32), 0x5EEDu, 0u), key);
    out[t] = u53(c.x, c.y);
  }
}

int gen_grid(long long n) {
  return (int)std::max(1LL, std::min((n + 255) / 256, (long long)num_sms() * 32));
}

}  // namespace

int gen_coo(int d, const int64_t* shape, int64_t nnz, double zipf_s, int normal_vals, uint64_t seed,
            int64_t* const* cols, double* vals, cudaStream_t st) {
  GenParams p{};
  p.d = d;
  p.key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  unsigned __int128 total = 1;
  for (int m = d - 1; m >= 0; --m) {
    p.dims[m] = shape[m];
    p.stride[m] = (long long)total;
    total *= (unsigned __int128)shape[m];
    if (total > ((unsigned __int128)1 << 62)) return fail(TK_EARG, "gen: index space exceeds 2^62");
  }
  if ((unsigned __int128)nnz > total) return fail(TK_EARG, "gen: nnz exceeds the number of cells");
  if (nnz == 0) return TK_OK;
  int bits = 1;
  while (bits < 63 && ((unsigned __int128)1 << bits) < total) ++bits;

  // truncated Zipf CDF tables (host-built, summed smallest index first)
  std::vector<DevBuf> cdfs(d);
  if (zipf_s > 0) {
    for (int m = 0; m < d; ++m) {
      const long long n = shape[m];
      std::vector<double> h(n);
      double acc = 0.0;
      for (long long i = 0; i < n; ++i) {
        acc += std::pow((double)(i + 1), -zipf_s);
        h[i] = acc;
      }
      for (long long i = 0; i < n; ++i) h[i] /= acc;
      h[n - 1] = 2.0;  // every u < 1 maps inside the support
      if (int rc = cdfs[m].alloc(n * 8, st)) return rc;
      TK_CUDA(cudaMemcpyAsync(cdfs[m].get(), h.data(), n * 8, cudaMemcpyHostToDevice, st));
      TK_CUDA(cudaStreamSynchronize(st));
      p.cdf[m] = cdfs[m].as<double>();
    }
  }

  long long M = zipf_s > 0 ? (long long)(nnz * 3.6) + 4096 : nnz + nnz / 64 + 4096;
  unsigned int* h_cnt = static_cast<unsigned int*>(pinned_scratch(16));
  while (true) {
    if (M > 0xFFFFFFF0LL) return fail(TK_EARG, "gen: more than 2^32 draws needed");
    DevBuf keys, keys2, idx, idx2, flag, temp, dkeys, didx, nsel;
    if (int rc = keys.alloc(M * 8, st)) return rc;
    if (int rc = keys2.alloc(M * 8, st)) return rc;
    if (int rc = idx.alloc(M * 4, st)) return rc;
    if (int rc = idx2.alloc(M * 4, st)) return rc;
    draw_kernel<<<gen_grid(M), 256, 0, st>>>(p, 0, M, keys.as<unsigned long long>(), idx.as<unsigned int>());
    TK_CUDA(cudaGetLastError());
    cub::DoubleBuffer<unsigned long long> kb(keys.as<unsigned long long>(), keys2.as<unsigned long long>());
    cub::DoubleBuffer<unsigned int> vb(idx.as<unsigned int>(), idx2.as<unsigned int>());
    size_t tb = 0;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)M, 0, bits, st));
    size_t tb2 = 0;
    TK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, kb.Current(), (unsigned char*)nullptr, kb.Alternate(),
                                       (int*)nullptr, (int)M, st));
    tb = std::max(tb, tb2);
    if (int rc = temp.alloc(tb, st)) return rc;
    TK_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, kb, vb, (int)M, 0, bits, st));
    if (int rc = flag.alloc(M, st)) return rc;
    if (int rc = nsel.alloc(16, st)) return rc;
    first_flag_kernel<<<gen_grid(M), 256, 0, st>>>(M, kb.Current(), flag.as<unsigned char>());
    // distinct keys (ascending) and their first draw index
    unsigned long long* ukeys = kb.Alternate();
    unsigned int* uidx = vb.Alternate();
    TK_CUDA(cub::DeviceSelect::Flagged(temp.get(), tb, kb.Current(), flag.as<unsigned char>(), ukeys,
                                       nsel.as<int>(), (int)M, st));
    TK_CUDA(cub::DeviceSelect::Flagged(temp.get(), tb, vb.Current(), flag.as<unsigned char>(), uidx,
                                       nsel.as<int>() + 1, (int)M, st));
    TK_CUDA(cudaMemcpyAsync(h_cnt, nsel.get(), 8, cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    const long long D = h_cnt[0];
    if (D < nnz) {
      // grow M by the observed acceptance ratio (deterministic: draws depend only on i)
      const double ratio = (double)D / (double)M;
      long long need = (long long)((double)nnz / std::max(ratio, 1e-3) * 1.08) + 4096;
      M = std::max(need, M + M / 4);
      continue;
    }
    // threshold T = nnz-th smallest first-draw index among distinct keys
    unsigned int* sidx = vb.Current();  // scratch (same size)
    {
      size_t tb3 = 0;
      TK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb3, uidx, sidx, (int)D, 0, 32, st));
      if (tb3 > tb) {
        temp.reset();
        if (int rc = temp.alloc(tb3, st)) return rc;
        tb = tb3;
      }
      TK_CUDA(cub::DeviceRadixSort::SortKeys(temp.get(), tb, uidx, sidx, (int)D, 0, 32, st));
    }
    le_flag_kernel<<<gen_grid(D), 256, 0, st>>>(D, uidx, sidx + (nnz - 1), flag.as<unsigned char>());
    unsigned long long* fkeys = kb.Current();
    TK_CUDA(cub::DeviceSelect::Flagged(temp.get(), tb, ukeys, flag.as<unsigned char>(), fkeys, nsel.as<int>(),
                                       (int)D, st));
    ColPtrs cp{};
    for (int m = 0; m < d; ++m) cp.col[m] = reinterpret_cast<long long*>(cols[m]);
    unravel_vals_kernel<<<gen_grid(nnz), 256, 0, st>>>(p, nnz, fkeys, normal_vals, cp, vals);
    TK_CUDA(cudaGetLastError());
    TK_CUDA(cudaStreamSynchronize(st));
    return TK_OK;
  }
}

int gen_uniform(int64_t n, uint64_t seed, double* out, cudaStream_t st) {
  if (n == 0) return TK_OK;
  uniform_kernel<<<gen_grid(n), 256, 0, st>>>(n, make_uint2((unsigned)seed, (unsigned)(seed >> 32)), out);
  TK_CUDA(cudaGetLastError());
  return TK_OK;
}

}  // namespace tk
