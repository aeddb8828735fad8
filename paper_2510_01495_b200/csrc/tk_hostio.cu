// tk_hostio.cu -- the host side of the host-buffer C-ABI calls (tk_*_host).
//
// A reference caller hands the kernel module pageable, read-only numpy arrays
// (SparseCooTensor's subs/vals, sparse.py:101-107; BoundKernelSet passes them through without a
// copy, bindings.py:19-37).  cudaMemcpy from pageable memory goes through the driver's
// single-threaded bounce buffer (11 GB/s measured on the B200 box vs 55 GB/s pinned), so the
// library stages pageable buffers itself:
//   * HostPool -- persistent worker threads (one per host core) for parallel host copies;
//   * per-device pinned staging arenas, reused across calls (allocated once, grown on demand);
//   * h2d / d2h -- chunked copies through the arena: the parallel host copy of chunk i+1
//     overlaps the DMA of chunk i;
//   * the packed row format for tensors: when every index of a row fits its dimension, the d int64
//     coordinates travel as one 64-bit word of bit fields (config 5: 20+17+14 bits), halving the
//     PCIe bytes of the reference layout's 32 B per nonzero; the device unpacks into SoA columns.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <unordered_map>

#include <unistd.h>
#include <thread>
#include <vector>

#include <emmintrin.h>

#include "tk_host.h"

namespace tk {

namespace {

// Copy with non-temporal (streaming) stores: the destination of a large host copy here is either a
// pinned staging buffer the DMA engine reads next or a caller's multi-GB result, never re-read
// from cache soon, so skipping the read-for-ownership of each destination line saves a third of
// the memory traffic (SSE2: baseline x86-64, no target flags).
void nt_copy(void* dst, const void* src, size_t bytes) {
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const size_t head = std::min(bytes, (size_t)((16 - ((uintptr_t)d & 15)) & 15));
  memcpy(d, s, head);
  d += head, s += head, bytes -= head;
  size_t i = 0;
  for (; i + 64 <= bytes; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
  }
  memcpy(d + i, s + i, bytes - i);
  _mm_sfence();
}

class HostPool {
 public:
  HostPool() {
    unsigned n = std::thread::hardware_concurrency();
    n = std::max(1u, std::min(n, 64u));
    for (unsigned i = 1; i < n; ++i) th_.emplace_back([this] { loop(); });
    size_ = (int)n;
  }
  int size() const { return size_; }
  // fn(i) for i in [0, n) on the workers and the caller; returns when every part is done
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || size_ == 1 || in_job_) {  // nested use from inside a job runs inline
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> one(run_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      n_ = n;
      next_.store(0);
      pending_ = n;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      in_job_ = true;
      (*job_)(i);
      in_job_ = false;
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin briefly before sleeping: a staged copy issues its chunk copies back to back, and a
      // condition-variable wake-up costs tens of microseconds
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(200)) {
      }
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
      }
      {
        std::lock_guard<std::mutex> lk(mu_);  // job_ / n_ of the new generation are published
        seen = gen_.load(std::memory_order_acquire);
      }
      work();
    }
  }
  static thread_local bool in_job_;
  std::vector<std::thread> th_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0, pending_ = 0, size_ = 1;
  std::atomic<int> next_{0};
  std::atomic<uint64_t> gen_{0};
};

thread_local bool HostPool::in_job_ = false;

HostPool& pool() {
  static HostPool* p = new HostPool();  // never destroyed: workers may outlive static teardown
  return *p;
}

constexpr size_t kDirectBytes = 1u << 20;   // below this a pageable copy goes straight to the driver
constexpr size_t kChunkBytes = 32u << 20;   // generic staged-copy chunk (largest)
constexpr size_t kMinChunkBytes = 2u << 20;  // smallest chunk: the host copy of chunk i+1 overlaps the DMA of i

struct Arena {  // per-device pinned staging, two halves used alternately
  std::mutex mu;
  char* buf = nullptr;
  size_t half = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // last DMA that read / wrote each half
  int ensure(size_t half_bytes) {
    if (!ev[0]) {
      TK_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
      TK_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    }
    if (half_bytes <= half) return TK_OK;
    TK_CUDA(cudaEventSynchronize(ev[0]));
    TK_CUDA(cudaEventSynchronize(ev[1]));
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    half = 0;
    half_bytes = (half_bytes + 4095) & ~size_t(4095);
    TK_CUDA(cudaMallocHost(&buf, 2 * half_bytes));
    half = half_bytes;
    return TK_OK;
  }
  char* part(int b) const { return buf + (size_t)b * half; }
};

Arena& arena(int which) {  // 0: inputs, 1: outputs
  static Arena a[64][2];
  int dev = 0;
  cudaGetDevice(&dev);
  return a[dev & 63][which];
}

// Cached pinned blocks for host-call RESULTS (tk_host_alloc / tk_host_free): a caller that drops
// the previous result gets its block back on the next call, so the D2H lands in the final array
// (no copy-out through staging, no first-touch faults of a fresh multi-GB array).
struct ResultPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> live_;
  size_t total = 0, cap = 0;
  ResultPool() {
    if (const char* e = getenv("TK_HOST_POOL_MB")) {
      cap = (size_t)atoll(e) << 20;
    } else {
      const long pages = sysconf(_SC_PHYS_PAGES), psz = sysconf(_SC_PAGESIZE);
      cap = pages > 0 && psz > 0 ? (size_t)pages * (size_t)psz / 4 : 0;  // a quarter of host RAM
    }
  }
  void* get(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= 2 * bytes) {  // at most 2x slack
      void* p = it->second;
      live_[p] = it->first;
      free_.erase(it);
      return p;
    }
    while (total + bytes > cap && !free_.empty()) {  // evict cached blocks, largest first
      auto last = std::prev(free_.end());
      cudaFreeHost(last->second);
      total -= last->first;
      free_.erase(last);
    }
    if (total + bytes > cap) return nullptr;
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    total += bytes;
    live_[p] = bytes;
    return p;
  }
  bool put(void* p) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = live_.find(p);
    if (it == live_.end()) return false;
    free_.emplace(it->second, p);
    live_.erase(it);
    return true;
  }
  void trim() {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : free_) {
      cudaFreeHost(kv.second);
      total -= kv.first;
    }
    free_.clear();
  }
};

ResultPool& result_pool() {
  static ResultPool* rp = new ResultPool();  // never destroyed: blocks may be returned at exit
  return *rp;
}

}  // namespace

void* host_result_alloc(size_t bytes) { return bytes ? result_pool().get(bytes) : nullptr; }
bool host_result_free(void* p) { return result_pool().put(p); }
void host_result_trim() { result_pool().trim(); }

int host_threads() { return pool().size(); }

void parallel_for(int n, const std::function<void(int)>& fn) { pool().run(n, fn); }

void pmemcpy(void* dst, const void* src, size_t bytes) {
  if (bytes < (512u << 10)) {
    memcpy(dst, src, bytes);
    return;
  }
  const int parts = (int)std::min<size_t>(pool().size(), bytes / (256u << 10));
  const size_t step = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
  pool().run(parts, [&](int i) {
    const size_t a = std::min(bytes, (size_t)i * step), b = std::min(bytes, a + step);
    if (b > a) nt_copy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  });
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return TK_OK;
  if (bytes < kDirectBytes || host_is_pinned(src)) {
    TK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return TK_OK;
  }
  Arena& a = arena(0);
  std::lock_guard<std::mutex> lk(a.mu);
  if (int rc = a.ensure(std::max(a.half, std::min(bytes, kChunkBytes)))) return rc;
  const size_t chunk = std::min(a.half, std::max(kMinChunkBytes, std::min(kChunkBytes, bytes / 8)));
  int b = 0;
  for (size_t off = 0; off < bytes; off += chunk, b ^= 1) {
    const size_t n = std::min(chunk, bytes - off);
    TK_CUDA(cudaEventSynchronize(a.ev[b]));  // the DMA that last read this half is done
    pmemcpy(a.part(b), static_cast<const char*>(src) + off, n);
    TK_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, a.part(b), n, cudaMemcpyHostToDevice, st));
    TK_CUDA(cudaEventRecord(a.ev[b], st));
  }
  return TK_OK;
}

int d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return TK_OK;
  if (bytes < kDirectBytes || host_is_pinned(dst)) {
    TK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaStreamSynchronize(st));
    return TK_OK;
  }
  Arena& a = arena(1);
  std::lock_guard<std::mutex> lk(a.mu);
  if (int rc = a.ensure(std::max(a.half, std::min(bytes, kChunkBytes)))) return rc;
  const size_t chunk = std::min(a.half, std::max(kMinChunkBytes, std::min(kChunkBytes, bytes / 8)));
  const size_t nch = (bytes + chunk - 1) / chunk;
  auto issue = [&](size_t i) -> int {
    const size_t off = i * chunk, n = std::min(chunk, bytes - off);
    TK_CUDA(cudaMemcpyAsync(a.part((int)(i & 1)), static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, st));
    TK_CUDA(cudaEventRecord(a.ev[i & 1], st));
    return TK_OK;
  };
  if (int rc = issue(0)) return rc;
  for (size_t i = 0; i < nch; ++i) {
    if (i + 1 < nch)
      if (int rc = issue(i + 1)) return rc;  // its half was copied out in iteration i-1
    TK_CUDA(cudaEventSynchronize(a.ev[i & 1]));
    const size_t off = i * chunk;
    pmemcpy(static_cast<char*>(dst) + off, a.part((int)(i & 1)), std::min(chunk, bytes - off));
  }
  return TK_OK;
}

// ---- packed tensor rows -----------------------------------------------------------------------

bool row_pack_plan(int d, const int64_t* shape, RowPack* p) {
  p->d = d;
  int total = 0;
  for (int m = d - 1; m >= 0; --m) {
    if (shape[m] <= 0) return false;
    const uint64_t top = (uint64_t)shape[m] - 1;
    const int bits = top == 0 ? 0 : 64 - __builtin_clzll(top);
    p->shift[m] = total;
    p->dim[m] = (uint64_t)shape[m];
    total += bits;
  }
  return total <= 64;
}

namespace {
template <int D>
bool pack_part(const RowPack& p, const int64_t* subs, int64_t n, uint64_t* out) {
  const int d = D > 0 ? D : p.d;
  bool ok = true;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t* s = subs + r * d;
    uint64_t w = 0;
    for (int m = 0; m < d; ++m) {
      const uint64_t v = (uint64_t)s[m];
      ok &= v < p.dim[m];
      w |= v << p.shift[m];
    }
    _mm_stream_si64(reinterpret_cast<long long*>(out + r), (long long)w);  // see nt_copy
  }
  _mm_sfence();
  return ok;
}
}  // namespace

bool pack_rows(const RowPack& p, const int64_t* subs, const double* vals, int64_t n, uint64_t* packed,
               double* vals_out) {
  std::atomic<bool> ok{true};
  const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(pool().size(), n / 65536));
  pool().run(parts, [&](int i) {
    const int64_t a = n * i / parts, b = n * (i + 1) / parts;
    bool o;
    switch (p.d) {
      case 2: o = pack_part<2>(p, subs + a * 2, b - a, packed + a); break;
      case 3: o = pack_part<3>(p, subs + a * 3, b - a, packed + a); break;
      case 4: o = pack_part<4>(p, subs + a * 4, b - a, packed + a); break;
      default: o = pack_part<0>(p, subs + a * p.d, b - a, packed + a); break;
    }
    if (!o) ok.store(false, std::memory_order_relaxed);
    nt_copy(vals_out + a, vals + a, (size_t)(b - a) * 8);
  });
  return ok.load();
}

}  // namespace tk
