// tk_gen_host.cpp -- host twin of the device operand generator.  TEST / BASELINE
// INFRASTRUCTURE ONLY: used by tests/ (to check the device generator byte for byte) and by
// bench.py's reference arm (which must build the config-4/5 tensors without touching the
// product library).  Never linked into or loaded by paper_2510_01495_b200/.
//
// It restates paper_2510_01495_b200/csrc/tk_gen.cu operation for operation:
//   * draw i is a d-tuple; mode m's coordinate comes from Philox4x32-10 (key = seed, counter =
//     (i lo, i hi, m, 0x7A11)) as a 53-bit uniform u, mapped to {0..n-1} by floor(u*n) (uniform
//     mode) or by the first index with cdf > u of a truncated Zipf(s) CDF table (built with the
//     same host code as tk_gen.cu);
//   * the tensor is the set of the FIRST nnz DISTINCT tuples of the draw sequence -- the
//     reference's exact-nnz top-up protocol (/root/reference/pkg/src/tenkern/synth.py:124-131);
//   * rows are emitted in canonical (lexicographic) order, row-major (nnz, d) int64 -- the
//     reference's SparseCooTensor layout (sparse.py:48-107);
//   * values are keyed by the linear coordinate (Philox, key = seed ^ salt, counter = (key lo,
//     key hi, attempt, 0xBA15)): uniform [0,1) or N(0,1) by Box-Muller with ln/cos made of IEEE
//     +,-,*,/,sqrt only, exact zeros redrawn (synth.py:133-138).
// Compiled with -ffp-contract=off (no FMA), so every double operation rounds exactly like the
// device's explicit __d*_rn intrinsics.
//
// Algorithm on the host (16 threads on the GPU box): draws -> radix partition by the top key
// bits (buckets stay in draw order) -> per-bucket sort by (key, draw) -> first occurrence per
// key -> threshold T = nnz-th smallest first-draw index (histogram + nth_element) -> keep keys
// whose first draw is <= T, in bucket (= key) order.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace {

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define TKG_T(label) if (std::getenv("TKG_TIMING")) std::fprintf(stderr, "tkg %-10s %.3f s\n", label, now_s() - t_start)

constexpr uint64_t kValSalt = 0x9E3779B97F4A7C15ull;

struct U4 {
  uint32_t x, y, z, w;
};

inline uint32_t mulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }

inline U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

inline double u53(uint32_t a, uint32_t b) {
  const uint64_t v = ((uint64_t)a << 21) ^ (uint64_t)(b >> 11);
  return (double)(v & ((1ull << 53) - 1)) * 0x1.0p-53;
}

// ---- ln / cos from exactly rounded operations (tk_gen.cu gen_ln / gen_cos2pi) ------------------
double gen_ln(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  const uint64_t mb = (b & 0xFFFFFFFFFFFFFull) | (1023ull << 52);
  double m;
  std::memcpy(&m, &mb, 8);
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    e += 1;
  }
  const double f = (m - 1.0) / (m + 1.0);
  const double s = f * f;
  double q = 0x1.642c8590b2164p-5;
  q = 0x1.8618618618618p-5 + s * q;
  q = 0x1.af286bca1af28p-5 + s * q;
  q = 0x1.e1e1e1e1e1e1ep-5 + s * q;
  q = 0x1.1111111111111p-4 + s * q;
  q = 0x1.3b13b13b13b14p-4 + s * q;
  q = 0x1.745d1745d1746p-4 + s * q;
  q = 0x1.c71c71c71c71cp-4 + s * q;
  q = 0x1.2492492492492p-3 + s * q;
  q = 0x1.999999999999ap-3 + s * q;
  q = 0x1.5555555555555p-2 + s * q;
  const double f2 = f + f;
  const double lm = f2 + (f2 * s) * q;
  return (double)e * 0x1.62e42fefa39efp-1 + lm;
}

double gen_cos_q(double y) {
  const double z = y * y;
  double q = 0x1.ae7f3e733b81fp-45;
  q = 0x1.93974a8c07c9dp-37 - z * q;
  q = 0x1.1eed8eff8d898p-29 - z * q;
  q = 0x1.27e4fb7789f5cp-22 - z * q;
  q = 0x1.a01a01a01a01ap-16 - z * q;
  q = 0x1.6c16c16c16c17p-10 - z * q;
  q = 0x1.5555555555555p-5 - z * q;
  q = 0.5 - z * q;
  return 1.0 - z * q;
}

double gen_sin_q(double y) {
  const double z = y * y;
  double q = 0x1.952c77030ad4ap-49;
  q = 0x1.ae7f3e733b81fp-41 - z * q;
  q = 0x1.6124613a86d09p-33 - z * q;
  q = 0x1.ae64567f544e4p-26 - z * q;
  q = 0x1.71de3a556c734p-19 - z * q;
  q = 0x1.a01a01a01a01ap-13 - z * q;
  q = 0x1.1111111111111p-7 - z * q;
  q = 0x1.5555555555555p-3 - z * q;
  return y - (y * z) * q;
}

double gen_cos2pi(double t) {
  double sign = 1.0;
  if (t > 0.5) t = 1.0 - t;
  if (t > 0.25) {
    t = 0.5 - t;
    sign = -1.0;
  }
  const double c = t > 0.125 ? gen_sin_q(0x1.921fb54442d18p+2 * (0.25 - t)) : gen_cos_q(0x1.921fb54442d18p+2 * t);
  return sign * c;
}

double value_of(uint64_t key, uint32_t vk0, uint32_t vk1, int normal_vals) {
  double v = 0.0;
  for (uint32_t attempt = 0; v == 0.0; ++attempt) {
    const U4 c = philox10(U4{(uint32_t)key, (uint32_t)(key >> 32), attempt, 0xBA15u}, vk0, vk1);
    if (!normal_vals) {
      v = u53(c.x, c.y);
    } else {
      const double u1 = 1.0 - u53(c.x, c.y);
      const double u2 = u53(c.z, c.w);
      v = std::sqrt(-2.0 * gen_ln(u1)) * gen_cos2pi(u2);
    }
  }
  return v;
}

// ---- threading -----------------------------------------------------------------------------------
template <class F>
void parallel_for(int nthreads, F&& f) {  // f(thread index)
  std::vector<std::thread> th;
  for (int t = 1; t < nthreads; ++t) th.emplace_back(f, t);
  f(0);
  for (auto& x : th) x.join();
}

struct Mode {
  int64_t n;
  uint64_t stride;
  const double* cdf;          // nullptr: uniform
  const int32_t* guide;       // G + 1 entries
  int64_t G;
};

// first index with cdf[idx] > u (the device's binary search), narrowed by a guide table
inline int64_t zipf_index(const Mode& md, double u) {
  const double* cdf = md.cdf;
  int64_t j = (int64_t)(u * (double)md.G);
  int64_t lo = md.guide[j > 0 ? j - 1 : 0];
  int64_t hi = md.guide[j + 1 < md.G ? j + 1 : md.G];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  if (!(cdf[lo] > u) || (lo > 0 && cdf[lo - 1] > u)) {  // guide miss (never expected): full search
    lo = 0;
    hi = md.n - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] > u) hi = mid;
      else lo = mid + 1;
    }
  }
  return lo;
}

inline uint64_t draw_key(const std::vector<Mode>& modes, uint32_t k0, uint32_t k1, uint64_t i) {
  uint64_t lin = 0;
  for (size_t m = 0; m < modes.size(); ++m) {
    const U4 c = philox10(U4{(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)m, 0x7A11u}, k0, k1);
    const double u = u53(c.x, c.y);
    const Mode& md = modes[m];
    int64_t v;
    if (md.cdf == nullptr) {
      v = (int64_t)(u * (double)md.n);
      if (v >= md.n) v = md.n - 1;
    } else {
      v = zipf_index(md, u);
    }
    lin += (uint64_t)v * md.stride;
  }
  return lin;
}

// draw_key for draws i0 .. i0+n-1 (n <= 16): all uniforms first, then the guide-table lines of
// every Zipf lookup prefetched, so the cache misses of the 16 draws overlap
inline void draw_keys16(const std::vector<Mode>& modes, uint32_t k0, uint32_t k1, uint64_t i0, int n,
                        uint64_t* out) {
  const int d = (int)modes.size();
  double u[16][8];
  for (int t = 0; t < n; ++t) {
    const uint64_t i = i0 + t;
    for (int m = 0; m < d; ++m) {
      const U4 c = philox10(U4{(uint32_t)i, (uint32_t)(i >> 32), (uint32_t)m, 0x7A11u}, k0, k1);
      u[t][m] = u53(c.x, c.y);
      const Mode& md = modes[m];
      if (md.cdf) __builtin_prefetch(md.guide + (int64_t)(u[t][m] * (double)md.G));
    }
  }
  for (int t = 0; t < n; ++t) {
    uint64_t lin = 0;
    for (int m = 0; m < d; ++m) {
      const Mode& md = modes[m];
      int64_t v;
      if (md.cdf == nullptr) {
        v = (int64_t)(u[t][m] * (double)md.n);
        if (v >= md.n) v = md.n - 1;
      } else {
        v = zipf_index(md, u[t][m]);
      }
      lin += (uint64_t)v * md.stride;
    }
    out[t] = lin;
  }
}

#pragma pack(push, 4)
struct Rec {
  uint64_t key;
  uint32_t idx;
};
#pragma pack(pop)

}  // namespace

extern "C" {

int tkg_version(void) { return 1; }

// The Zipf CDF table of tk_gen.cu (host-built there too): cdf[i] = sum_{j<=i} (j+1)^-s / total,
// cdf[n-1] = 2.0.
void tkg_zipf_cdf(int64_t n, double s, double* h) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += std::pow((double)(i + 1), -s);
    h[i] = acc;
  }
  for (int64_t i = 0; i < n; ++i) h[i] /= acc;
  h[n - 1] = 2.0;
}

// gen_uniform (tk_gen.cu uniform_kernel): out[t] = u53 of Philox(key = seed, counter = (t, 0x5EED, 0))
void tkg_gen_uniform(int64_t n, uint64_t seed, double* out) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t t = 0; t < n; ++t) {
    const U4 c = philox10(U4{(uint32_t)t, (uint32_t)((uint64_t)t >> 32), 0x5EEDu, 0u}, k0, k1);
    out[t] = u53(c.x, c.y);
  }
}

// exposed for the unit test of the exact-op normal transform
double tkg_ln(double x) { return gen_ln(x); }
double tkg_cos2pi(double t) { return gen_cos2pi(t); }

// gen_coo (tk_gen.cu gen_coo): row-major subs (nnz, d) int64 in canonical order + vals.
// Returns 0, or 8 (TK_EARG) for an index space over 2^62 / nnz over the cell count / >2^32 draws.
int tkg_gen_coo(int d, const int64_t* shape, int64_t nnz, double zipf_s, int normal_vals, uint64_t seed,
                int nthreads, int64_t* subs, double* vals) {
  if (nthreads < 1) nthreads = 1;
  const double t_start = now_s();
  std::vector<Mode> modes(d);
  unsigned __int128 total = 1;
  for (int m = d - 1; m >= 0; --m) {
    modes[m].n = shape[m];
    modes[m].stride = (uint64_t)total;
    modes[m].cdf = nullptr;
    total *= (unsigned __int128)shape[m];
    if (total > ((unsigned __int128)1 << 62)) return 8;
  }
  if ((unsigned __int128)nnz > total) return 8;
  if (nnz == 0) return 0;

  std::vector<std::vector<double>> cdfs(d);
  std::vector<std::vector<int32_t>> guides(d);
  if (zipf_s > 0) {
    for (int m = 0; m < d; ++m) {
      const int64_t n = shape[m];
      cdfs[m].resize(n);
      tkg_zipf_cdf(n, zipf_s, cdfs[m].data());
      const int64_t G = std::max<int64_t>(1, std::min<int64_t>(2 * n, 1 << 22));
      guides[m].resize(G + 1);
      int64_t idx = 0;
      for (int64_t j = 0; j <= G; ++j) {
        const double t = j == G ? 1.0 : (double)j / (double)G;
        while (idx < n - 1 && !(cdfs[m][idx] > t)) ++idx;
        guides[m][j] = (int32_t)idx;
      }
      modes[m].cdf = cdfs[m].data();
      modes[m].guide = guides[m].data();
      modes[m].G = G;
    }
  }
  TKG_T("cdf");
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  constexpr int HB = 12;  // hash buckets 2^HB for the dedup stage
  constexpr int64_t NB = 1 << HB;
  auto hmix = [](uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return k;
  };

  int64_t M = zipf_s > 0 ? (int64_t)(nnz * 3.6) + 4096 : nnz + nnz / 64 + 4096;
  while (true) {
    if (M > 0xFFFFFFF0ll) return 8;
    // 1. draws, in per-thread draw-order chunks; a draw whose key a small direct-mapped cache has
    //    already seen earlier in the same chunk is dropped (its first occurrence is kept), which
    //    removes most repeats of the Zipf head cheaply
    std::vector<std::vector<Rec>> local(nthreads);
    std::vector<int64_t> hist((size_t)nthreads * NB, 0);
    parallel_for(nthreads, [&](int t) {
      const int64_t a = M * t / nthreads, b = M * (t + 1) / nthreads;
      constexpr int CB = 16;
      std::vector<uint64_t> cache((size_t)1 << CB, ~0ull);
      std::vector<Rec>& out = local[t];
      out.reserve((size_t)((b - a) / 2 + 1024));
      int64_t* h = hist.data() + (size_t)t * NB;
      uint64_t kb[16];
      for (int64_t i0 = a; i0 < b; i0 += 16) {
        const int nb = (int)std::min<int64_t>(16, b - i0);
        if (d <= 8) draw_keys16(modes, k0, k1, (uint64_t)i0, nb, kb);
        else
          for (int t = 0; t < nb; ++t) kb[t] = draw_key(modes, k0, k1, (uint64_t)(i0 + t));
        for (int t = 0; t < nb; ++t) {
          const uint64_t k = kb[t];
          const uint64_t hk = hmix(k);
          uint64_t& c = cache[hk & ((1u << CB) - 1)];
          if (c == k) continue;
          c = k;
          out.push_back(Rec{k, (uint32_t)(i0 + t)});
          ++h[hk >> (64 - HB)];
        }
      }
    });
    TKG_T("draws");
    // 2. scatter into hash buckets (bucket-major, thread-minor)
    std::vector<int64_t> boff(NB + 1, 0), toff((size_t)nthreads * NB);
    {
      int64_t run = 0;
      for (int64_t bkt = 0; bkt < NB; ++bkt) {
        boff[bkt] = run;
        for (int t = 0; t < nthreads; ++t) {
          toff[(size_t)t * NB + bkt] = run;
          run += hist[(size_t)t * NB + bkt];
        }
      }
      boff[NB] = run;
    }
    std::vector<Rec> recs(boff[NB]);
    parallel_for(nthreads, [&](int t) {
      int64_t* o = toff.data() + (size_t)t * NB;
      for (const Rec& r : local[t]) recs[o[hmix(r.key) >> (64 - HB)]++] = r;
      std::vector<Rec>().swap(local[t]);
    });
    TKG_T("scatter");
    // 3. per bucket: sort by (key, draw), keep each key's first draw, compact in place
    std::vector<int64_t> dcount(NB, 0);
    std::atomic<int64_t> next{0};
    parallel_for(nthreads, [&](int) {
      for (int64_t bkt; (bkt = next.fetch_add(1)) < NB;) {
        Rec* r = recs.data() + boff[bkt];
        const int64_t n = boff[bkt + 1] - boff[bkt];
        std::sort(r, r + n, [](const Rec& x, const Rec& y) { return x.key < y.key || (x.key == y.key && x.idx < y.idx); });
        int64_t w = 0;
        for (int64_t i = 0; i < n; ++i)
          if (i == 0 || r[i].key != r[i - 1].key) r[w++] = r[i];
        dcount[bkt] = w;
      }
    });
    TKG_T("dedup");
    int64_t D = 0;
    for (int64_t bkt = 0; bkt < NB; ++bkt) D += dcount[bkt];
    if (D < nnz) {
      const double ratio = (double)D / (double)M;
      const int64_t need = (int64_t)((double)nnz / std::max(ratio, 1e-3) * 1.08) + 4096;
      M = std::max(need, M + M / 4);
      continue;
    }
    // 4. T = the nnz-th smallest first-draw index among the D distinct keys
    const int HS = 16;
    const int64_t NH = (M >> HS) + 1;
    std::vector<int64_t> h2((size_t)nthreads * NH, 0);
    parallel_for(nthreads, [&](int t) {
      int64_t* h = h2.data() + (size_t)t * NH;
      for (int64_t bkt = NB * t / nthreads; bkt < NB * (t + 1) / nthreads; ++bkt) {
        const Rec* r = recs.data() + boff[bkt];
        for (int64_t i = 0; i < dcount[bkt]; ++i) ++h[r[i].idx >> HS];
      }
    });
    int64_t below = 0, bin = 0;
    for (; bin < NH; ++bin) {
      int64_t c = 0;
      for (int t = 0; t < nthreads; ++t) c += h2[(size_t)t * NH + bin];
      if (below + c >= nnz) break;
      below += c;
    }
    std::vector<uint32_t> inbin;
    for (int64_t bkt = 0; bkt < NB; ++bkt) {
      const Rec* r = recs.data() + boff[bkt];
      for (int64_t i = 0; i < dcount[bkt]; ++i)
        if ((int64_t)(r[i].idx >> HS) == bin) inbin.push_back(r[i].idx);
    }
    const int64_t kth = nnz - below - 1;
    std::nth_element(inbin.begin(), inbin.begin() + kth, inbin.end());
    const uint32_t T = inbin[kth];
    TKG_T("threshold");
    // 5. the kept keys (exactly nnz, all distinct), into `keys`
    std::vector<int64_t> kept(NB + 1, 0);
    parallel_for(nthreads, [&](int t) {
      for (int64_t bkt = NB * t / nthreads; bkt < NB * (t + 1) / nthreads; ++bkt) {
        const Rec* r = recs.data() + boff[bkt];
        int64_t c = 0;
        for (int64_t i = 0; i < dcount[bkt]; ++i) c += r[i].idx <= T;
        kept[bkt + 1] = c;
      }
    });
    for (int64_t bkt = 0; bkt < NB; ++bkt) kept[bkt + 1] += kept[bkt];
    std::vector<uint64_t> keys(nnz);
    parallel_for(nthreads, [&](int t) {
      for (int64_t bkt = NB * t / nthreads; bkt < NB * (t + 1) / nthreads; ++bkt) {
        const Rec* r = recs.data() + boff[bkt];
        int64_t o = kept[bkt];
        for (int64_t i = 0; i < dcount[bkt]; ++i)
          if (r[i].idx <= T) keys[o++] = r[i].key;
      }
    });
    std::vector<Rec>().swap(recs);
    // 6. canonical order: splitter partition of the distinct keys (sampled, so the Zipf head does
    //    not pile into one range), then every range sorted on its own
    const int64_t P = std::max<int64_t>(1, std::min<int64_t>(nnz / 4096, 4096));
    std::vector<uint64_t> spl;
    {
      std::vector<uint64_t> smp;
      const int64_t ns = std::min<int64_t>(nnz, P * 32);
      for (int64_t i = 0; i < ns; ++i) smp.push_back(keys[(uint64_t)i * 0x9E3779B97F4A7C15ull % (uint64_t)nnz]);
      std::sort(smp.begin(), smp.end());
      for (int64_t j = 1; j < P; ++j) spl.push_back(smp[ns * j / P]);
    }
    std::vector<int64_t> ph((size_t)nthreads * (P + 1), 0);
    auto part_of = [&](uint64_t k) { return (int64_t)(std::upper_bound(spl.begin(), spl.end(), k) - spl.begin()); };
    parallel_for(nthreads, [&](int t) {
      int64_t* h = ph.data() + (size_t)t * (P + 1);
      for (int64_t i = nnz * t / nthreads; i < nnz * (t + 1) / nthreads; ++i) ++h[part_of(keys[i])];
    });
    std::vector<int64_t> poff(P + 1, 0), tpo((size_t)nthreads * P);
    {
      int64_t run = 0;
      for (int64_t q = 0; q < P; ++q) {
        poff[q] = run;
        for (int t = 0; t < nthreads; ++t) {
          tpo[(size_t)t * P + q] = run;
          run += ph[(size_t)t * (P + 1) + q];
        }
      }
      poff[P] = run;
    }
    std::vector<uint64_t> sorted(nnz);
    parallel_for(nthreads, [&](int t) {
      int64_t* o = tpo.data() + (size_t)t * P;
      for (int64_t i = nnz * t / nthreads; i < nnz * (t + 1) / nthreads; ++i) sorted[o[part_of(keys[i])]++] = keys[i];
    });
    std::vector<uint64_t>().swap(keys);
    next = 0;
    parallel_for(nthreads, [&](int) {
      for (int64_t q; (q = next.fetch_add(1)) < P;) std::sort(sorted.begin() + poff[q], sorted.begin() + poff[q + 1]);
    });
    TKG_T("sort");
    // 7. unravel + values
    const uint32_t vk0 = k0 ^ (uint32_t)kValSalt, vk1 = k1 ^ (uint32_t)(kValSalt >> 32);
    parallel_for(nthreads, [&](int t) {
      for (int64_t row = nnz * t / nthreads; row < nnz * (t + 1) / nthreads; ++row) {
        uint64_t lin = sorted[row];
        for (int m = d - 1; m >= 0; --m) {
          const uint64_t dm = (uint64_t)shape[m];
          subs[row * d + m] = (int64_t)(lin % dm);
          lin /= dm;
        }
        vals[row] = value_of(sorted[row], vk0, vk1, normal_vals);
      }
    });
    TKG_T("emit");
    return 0;
  }
}

// Split points [0 = b0 <= ... <= b_parts = n] of row-major canonical subs (nnz, d) such that no
// run of equal kept-mode prefixes (the first `nkeep` columns) spans two parts: b_i is the first
// row >= i*n/parts whose prefix differs from row (target - 1)'s -- the shards' concatenated TTV
// results are the one-call result.
void tkg_shard_bounds(const int64_t* subs, int64_t n, int d, int nkeep, int parts, int64_t* bounds) {
  auto same = [&](int64_t a, int64_t b) {
    for (int c = 0; c < nkeep; ++c)
      if (subs[a * d + c] != subs[b * d + c]) return false;
    return true;
  };
  bounds[0] = 0;
  for (int i = 1; i < parts; ++i) {
    const int64_t t = n * i / parts;
    int64_t b;
    if (t <= 0) b = 0;
    else if (t >= n) b = n;
    else {  // rows [t-1, b) share row t-1's prefix (sorted input): gallop then bisect
      int64_t lo = t, step = 1, hi = t;
      while (hi < n && same(hi, t - 1)) {
        lo = hi + 1;
        hi = std::min(n, hi + step);
        step *= 2;
      }
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (same(mid, t - 1)) lo = mid + 1;
        else hi = mid;
      }
      b = lo;
    }
    bounds[i] = std::max(b, bounds[i - 1]);
  }
  bounds[parts] = n;
}

}  // extern "C"
