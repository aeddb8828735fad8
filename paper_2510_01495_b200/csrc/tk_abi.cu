// tk_abi.cu -- extern "C" surface of libtk_b200.so (declared in include/tk_b200.h).
//
// Argument validation mirrors the reference's structural guards, which stay on even
// for unchecked calls (_check_ttv, pkg/src/tenkern/_ckernels.pyx:298-310): order >= 2,
// 0 <= k < d, len(x) == shape[k]; messages use the reference's wording so the Python
// layer can raise the same exception text.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tk_host.h"

namespace tk {

int gen_coo(int d, const int64_t* shape, int64_t nnz, double zipf_s, int normal_vals, uint64_t seed,
            int64_t* const* cols, double* vals, cudaStream_t st);
int gen_uniform(int64_t n, uint64_t seed, double* out, cudaStream_t st);

namespace {
thread_local std::string g_err;
thread_local void* g_pinned = nullptr;
thread_local size_t g_pinned_bytes = 0;
thread_local cudaStream_t g_stream[64] = {};
thread_local cudaEvent_t g_ev[64][2] = {};
std::mutex g_mu;
bool g_pool_ready[64] = {};
int g_sms[64] = {};

int cur_dev() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}

cudaStream_t lib_stream() {
  const int dev = cur_dev();
  if (!g_stream[dev]) cudaStreamCreateWithFlags(&g_stream[dev], cudaStreamNonBlocking);
  return g_stream[dev];
}

std::string fmt(const char* f, long long a, long long b = 0, long long c = 0) {
  char buf[256];
  snprintf(buf, sizeof buf, f, a, b, c);
  return buf;
}

int check_ttv_args(int d, const int64_t* shape, int k, int64_t nx) {
  if (d < 2) return fail(TK_EORDER, fmt("ttv: tensor order must be at least 2, got %lld", d));
  if (k < 0 || k >= d) return fail(TK_EMODE, fmt("ttv: mode %lld out of range for order-%lld tensor", k, d));
  if (d > TK_MAX_ORDER) return fail(TK_EARG, fmt("ttv: tensor order %lld exceeds TK_MAX_ORDER (%lld)", d, TK_MAX_ORDER));
  if (shape == nullptr) return fail(TK_EARG, "ttv: shape is NULL");
  if (nx != shape[k])
    return fail(TK_EDIM, fmt("ttv: vector length %lld does not match shape[%lld] == %lld", nx, k, shape[k]));
  return TK_OK;
}

int64_t pitch_of(int64_t n) { return (n + 1) & ~int64_t(1); }  // keep SoA columns 16-byte aligned

// Native-side monotonic clock around each *_host call, like the reference's _monotonic()
// around its kernels (_ckernels.pyx:30-33, 98-122, 377-388): excludes the FFI crossing.
thread_local double g_last_call_s = 0.0;
thread_local cudaEvent_t g_kev[64][2] = {};
thread_local bool g_kev_used[64] = {};
std::atomic<long long> g_launches{0};
struct CallClock {
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~CallClock() {
    g_last_call_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};
}  // namespace

void set_error(const std::string& msg) { g_err = msg; }
int fail(int status, const std::string& msg) {
  set_error(msg);
  return status;
}
int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")");
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? TK_ENOMEM : TK_ECUDA;
}

void prepare_pool() {
  const int dev = cur_dev();
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_pool_ready[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  g_pool_ready[dev] = true;
}

int DevBuf::alloc(size_t bytes, cudaStream_t st) {
  reset();
  prepare_pool();
  if (bytes == 0) bytes = 256;
  cudaError_t e = cudaMallocAsync(&ptr_, bytes, st);
  if (e != cudaSuccess) {
    ptr_ = nullptr;
    return cuda_fail(e, "cudaMallocAsync");
  }
  bytes_ = bytes;
  st_ = st;
  return TK_OK;
}

void DevBuf::reset() {
  if (ptr_) cudaFreeAsync(ptr_, st_);
  ptr_ = nullptr;
  bytes_ = 0;
}

void* pinned_scratch(size_t bytes) {
  if (bytes > g_pinned_bytes) {
    if (g_pinned) cudaFreeHost(g_pinned);
    g_pinned = nullptr;
    g_pinned_bytes = 0;
    if (cudaMallocHost(&g_pinned, std::max<size_t>(bytes, 4096)) == cudaSuccess)
      g_pinned_bytes = std::max<size_t>(bytes, 4096);
  }
  return g_pinned;
}

void ktimer_begin(cudaStream_t st) {
  const int dev = cur_dev();
  for (int i = 0; i < 2; ++i)
    if (!g_kev[dev][i]) cudaEventCreate(&g_kev[dev][i]);
  cudaEventRecord(g_kev[dev][0], st);
  g_kev_used[dev] = false;
}

void ktimer_end(cudaStream_t st) {
  const int dev = cur_dev();
  cudaEventRecord(g_kev[dev][1], st);
  g_kev_used[dev] = true;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  const int dev = cur_dev();
  if (!g_sms[dev]) cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return g_sms[dev] ? g_sms[dev] : 148;
}

}  // namespace tk

using namespace tk;

extern "C" {

const char* tk_last_error(void) { return g_err.c_str(); }

int tk_version(void) { return 100; }

double tk_last_call_seconds(void) { return g_last_call_s; }

double tk_last_kernel_ms(void) {
  const int dev = cur_dev();
  if (!g_kev_used[dev]) return -1.0;
  float ms = -1.f;
  if (cudaEventSynchronize(g_kev[dev][1]) != cudaSuccess) return -1.0;
  if (cudaEventElapsedTime(&ms, g_kev[dev][0], g_kev[dev][1]) != cudaSuccess) return -1.0;
  return ms;
}

long long tk_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int tk_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *n = c;
  return TK_OK;
}

// ---- dense ------------------------------------------------------------------------------------

int tk_dot_f64_device(const double* x, const double* y, int64_t n, double* out, void* stream) {
  if (n < 0) return fail(TK_EARG, "dot: negative length");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = dot_device(x, y, n, out, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

int tk_dot_f64_host(const double* x, const double* y, int64_t n, double* out) {
  CallClock clock_;
  if (n < 0) return fail(TK_EARG, "dot: negative length");
  cudaStream_t st = lib_stream();
  const int64_t pn = pitch_of(n);
  DevBuf b;
  if (int rc = b.alloc((size_t)(2 * pn + 2) * 8, st)) return rc;
  double* dx = b.as<double>();
  double* dy = dx + pn;
  double* dout = dy + pn;
  if (n) {
    if (int rc = h2d(dx, x, n * 8, st)) return rc;
    if (int rc = h2d(dy, y, n * 8, st)) return rc;
  }
  if (int rc = dot_device(dx, dy, n, dout, st)) return rc;
  double* h = static_cast<double*>(pinned_scratch(8));
  TK_CUDA(cudaMemcpyAsync(h, dout, 8, cudaMemcpyDeviceToHost, st));
  TK_CUDA(cudaStreamSynchronize(st));
  *out = *h;
  return TK_OK;
}

int tk_read_floor_f64_device(const double* p, int64_t n, double* sink, void* stream) {
  if (n < 0 || (!p && n > 0) || !sink) return fail(TK_EARG, "read_floor: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = read_floor_device(p, n, sink, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

int tk_matvec_f64_device(const double* a, int64_t rows, int64_t cols, const double* x, double* y, void* stream) {
  if (rows < 0 || cols < 0) return fail(TK_EARG, "matvec: negative shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = matvec_device(a, rows, cols, x, y, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

int tk_matvec_f64_host(const double* a, int64_t rows, int64_t cols, const double* x, double* y) {
  CallClock clock_;
  if (rows < 0 || cols < 0) return fail(TK_EARG, "matvec: negative shape");
  if (rows == 0) return TK_OK;
  cudaStream_t st = lib_stream();
  const size_t na = (size_t)rows * cols, pa = (na + 1) & ~size_t(1), px = ((size_t)cols + 1) & ~size_t(1);
  DevBuf b;
  if (int rc = b.alloc((pa + px + rows + 2) * 8, st)) return rc;
  double* da = b.as<double>();
  double* dx = da + pa;
  double* dy = dx + px;
  if (int rc = h2d(da, a, na * 8, st)) return rc;
  if (int rc = h2d(dx, x, (size_t)cols * 8, st)) return rc;
  if (int rc = matvec_device(da, rows, cols, dx, dy, st)) return rc;
  if (int rc = d2h(y, dy, (size_t)rows * 8, st)) return rc;
  return TK_OK;
}

// ---- sparse -----------------------------------------------------------------------------------

int tk_ttv_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const int64_t* subs,
                      const double* vals, const double* x, int64_t nx, int32_t k, int64_t* out_subs,
                      double* out_vals, int64_t* out_nnz, void* stream) {
  if (int rc = check_ttv_args(d, shape, k, nx)) return rc;
  if (nnz < 0 || out_nnz == nullptr) return fail(TK_EARG, "ttv: bad nnz / out_nnz");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  *out_nnz = 0;
  if (nnz == 0) return TK_OK;
  DevBuf soa;
  std::vector<const int64_t*> cp(d);
  if (cols) {
    for (int m = 0; m < d; ++m) cp[m] = cols[m];
  } else {
    if (!subs) return fail(TK_EARG, "ttv: neither cols nor subs given");
    const int64_t pitch = pitch_of(nnz);
    if (int rc = soa.alloc((size_t)pitch * d * 8, st)) return rc;
    if (int rc = aos_to_soa(nnz, d, subs, soa.as<int64_t>(), pitch, st)) return rc;
    for (int m = 0; m < d; ++m) cp[m] = soa.as<int64_t>() + (size_t)m * pitch;
  }
  return ttv_sparse_device(d, shape, nnz, cp.data(), vals, x, nx, k, out_subs, out_vals, out_nnz, st);
}

constexpr int64_t kPipeRows = 8ll << 20;  // rows per chunk of the pipelined host TTV
constexpr int kPipeDeclined = -1;          // the pipelined path does not apply: use the one-shot path

cudaStream_t side_stream(int which) {  // 0: host->device copies, 1: device->host copies
  static cudaStream_t s[64][2] = {};
  const int dev = cur_dev();
  if (!s[dev][which]) cudaStreamCreateWithFlags(&s[dev][which], cudaStreamNonBlocking);
  return s[dev][which];
}

// kept key (first d-1 coordinates) of host rows i and j: -1 / 0 / +1 (lexicographic)
int key_cmp(const int64_t* subs, int d, int64_t i, int64_t j) {
  for (int c = 0; c < d - 1; ++c) {
    const int64_t a = subs[i * d + c], b = subs[j * d + c];
    if (a != b) return a < b ? -1 : 1;
  }
  return 0;
}

// Pinned host staging shared by the pipelined TTV calls of one device (inputs and outputs; two
// halves each, reused across calls, grown on demand).
struct PipeStage {
  std::mutex mu;
  char* in = nullptr;
  char* out = nullptr;
  size_t in_half = 0, out_half = 0;
  int ensure(size_t in_b, size_t out_b) {
    if (in_b > in_half) {
      if (in) cudaFreeHost(in);
      in = nullptr;
      in_half = 0;
      TK_CUDA(cudaMallocHost(&in, 2 * in_b));
      in_half = in_b;
    }
    if (out_b > out_half) {
      if (out) cudaFreeHost(out);
      out = nullptr;
      out_half = 0;
      TK_CUDA(cudaMallocHost(&out, 2 * out_b));
      out_half = out_b;
    }
    return TK_OK;
  }
};
PipeStage& pipe_stage() {
  static PipeStage s[64];
  return s[cur_dev()];
}

// Host-buffer TTV with k == d-1, pipelined over chunks cut at kept-key changes: the copy of chunk
// i+1 in, the TTV of chunk i and the copy of chunk i-1's result out overlap (PCIe is full duplex).
// Each chunk is a complete set of groups, so the result is the concatenation of the chunk results.
// Pinned caller buffers are DMA'd directly.  Pageable ones (the reference caller's numpy arrays)
// go through pinned staging: the host packs chunk i+1's rows (RowPack: one 64-bit word per row
// when every index fits its dimension, else the raw int64 rows) with the thread pool while the
// DMA of chunk i runs, and copies chunk i-1's result out of its staging half in parallel.
// Declines (kPipeDeclined) if the input is not in kept-key order -- the one-shot path then sorts.
// TK_PIPE_TIMING=1: where the host time of one pipelined call goes (stderr; diagnostics only).
struct PipeTimes {
  using clk = std::chrono::steady_clock;
  bool on = getenv("TK_PIPE_TIMING") != nullptr;
  double t[6] = {0, 0, 0, 0, 0, 0};  // wait_in, pack, wait_free, copy_out, final_sync, total
  clk::time_point t0 = clk::now();
  struct Span {
    PipeTimes* p;
    int i;
    clk::time_point s = clk::now();
    ~Span() {
      if (p->on) p->t[i] += std::chrono::duration<double>(clk::now() - s).count();
    }
  };
  Span span(int i) { return Span{this, i}; }
  ~PipeTimes() {
    if (!on) return;
    t[5] = std::chrono::duration<double>(clk::now() - t0).count();
    fprintf(stderr, "[tk pipe] wait_in %.1f pack %.1f wait_free %.1f copy_out %.1f final_sync %.1f total %.1f ms\n",
            t[0] * 1e3, t[1] * 1e3, t[2] * 1e3, t[3] * 1e3, t[4] * 1e3, t[5] * 1e3);
  }
};

int ttv_host_pipelined(int d, const int64_t* shape, int64_t nnz, const int64_t* subs, const double* vals,
                       const double* x, int64_t nx, int64_t* out_subs, double* out_vals, int64_t* out_nnz) {
  PipeTimes pt;
  const int nk = d - 1;
  std::vector<int64_t> cut{0};
  while (cut.back() < nnz) {
    int64_t e = std::min(nnz, cut.back() + kPipeRows);
    while (e < nnz && key_cmp(subs, d, e - 1, e) == 0) ++e;  // never split a group
    if (e < nnz && key_cmp(subs, d, e - 1, e) > 0) return kPipeDeclined;
    cut.push_back(e);
  }
  const int nchunk = (int)cut.size() - 1;
  int64_t rows = 0;
  for (int i = 0; i < nchunk; ++i) rows = std::max(rows, cut[i + 1] - cut[i]);
  const int64_t pitch = pitch_of(rows);
  const bool pin_in = host_is_pinned(subs) && host_is_pinned(vals);
  const bool pin_out = host_is_pinned(out_subs) && host_is_pinned(out_vals);
  RowPack rp;
  const bool packable = !pin_in && row_pack_plan(d, shape, &rp);
  cudaStream_t sc = lib_stream(), si = side_stream(0), so = side_stream(1);
  std::unique_lock<std::mutex> stage_lock;
  PipeStage* ps = nullptr;
  if (!pin_in || !pin_out) {
    ps = &pipe_stage();
    stage_lock = std::unique_lock<std::mutex>(ps->mu);
    if (int rc = ps->ensure(pin_in ? 0 : (size_t)rows * (d + 1) * 8, pin_out ? 0 : (size_t)rows * (nk + 1) * 8))
      return rc;
  }
  DevBuf b_x, b_aos[2], b_soa[2], b_vals[2], b_os[2], b_ov[2];
  if (int rc = b_x.alloc((size_t)std::max<int64_t>(nx, 1) * 8, sc)) return rc;
  for (int b = 0; b < 2; ++b) {
    if (int rc = b_aos[b].alloc((size_t)rows * d * 8, sc)) return rc;
    if (int rc = b_soa[b].alloc((size_t)pitch * d * 8, sc)) return rc;
    if (int rc = b_vals[b].alloc((size_t)rows * 8, sc)) return rc;
    if (int rc = b_os[b].alloc((size_t)rows * nk * 8, sc)) return rc;
    if (int rc = b_ov[b].alloc((size_t)rows * 8, sc)) return rc;
  }
  if (nx) TK_CUDA(cudaMemcpyAsync(b_x.get(), x, (size_t)nx * 8, cudaMemcpyHostToDevice, sc));
  cudaEvent_t ev_in[2], ev_done[2], ev_free[2];
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_free[b], cudaEventDisableTiming);
  }
  struct Cleanup {
    cudaEvent_t* e;
    ~Cleanup() {
      for (int i = 0; i < 6; ++i) cudaEventDestroy(e[i]);
    }
  };
  cudaEvent_t all[6] = {ev_in[0], ev_in[1], ev_done[0], ev_done[1], ev_free[0], ev_free[1]};
  Cleanup cleanup_{all};
  struct Drain {  // on every exit: the side streams are done before the buffers go back to the pool
    cudaStream_t a, b;
    ~Drain() {
      cudaStreamSynchronize(a);
      cudaStreamSynchronize(b);
    }
  } drain_{si, so};
  // the pool allocations above are stream-ordered on sc: the side streams start after them
  TK_CUDA(cudaEventRecord(ev_done[0], sc));
  TK_CUDA(cudaStreamWaitEvent(si, ev_done[0], 0));
  TK_CUDA(cudaStreamWaitEvent(so, ev_done[0], 0));
  bool packed[2] = {false, false};
  auto copy_in = [&](int i) -> int {
    const int b = i & 1;
    const int64_t n = cut[i + 1] - cut[i];
    if (pin_in) {
      TK_CUDA(cudaMemcpyAsync(b_aos[b].get(), subs + cut[i] * d, (size_t)n * d * 8, cudaMemcpyHostToDevice, si));
      TK_CUDA(cudaMemcpyAsync(b_vals[b].get(), vals + cut[i], (size_t)n * 8, cudaMemcpyHostToDevice, si));
    } else {
      {
        auto sp = pt.span(0);
        TK_CUDA(cudaEventSynchronize(ev_in[b]));  // the DMA that last read this staging half is done
      }
      auto sp = pt.span(1);
      char* stg = ps->in + (size_t)b * ps->in_half;
      double* sv = reinterpret_cast<double*>(stg + (size_t)rows * d * 8);
      packed[b] = packable && pack_rows(rp, subs + cut[i] * d, vals + cut[i], n, reinterpret_cast<uint64_t*>(stg), sv);
      if (!packed[b]) {  // an index outside its dimension (or too many bits): raw rows
        pmemcpy(stg, subs + cut[i] * d, (size_t)n * d * 8);
        pmemcpy(sv, vals + cut[i], (size_t)n * 8);
      }
      TK_CUDA(cudaMemcpyAsync(b_aos[b].get(), stg, (size_t)n * (packed[b] ? 1 : d) * 8, cudaMemcpyHostToDevice, si));
      TK_CUDA(cudaMemcpyAsync(b_vals[b].get(), sv, (size_t)n * 8, cudaMemcpyHostToDevice, si));
    }
    TK_CUDA(cudaEventRecord(ev_in[b], si));
    return TK_OK;
  };
  std::vector<int64_t> offs(nchunk + 1, 0), us(nchunk, 0);
  auto copy_out_host = [&](int i) -> int {  // pageable outputs: staging half -> caller, in parallel
    const int b = i & 1;
    {
      auto sp = pt.span(2);
      TK_CUDA(cudaEventSynchronize(ev_free[b]));
    }
    auto sp = pt.span(3);
    const int64_t u = us[i];
    char* stg = ps->out + (size_t)b * ps->out_half;
    pmemcpy(out_subs + offs[i] * nk, stg, (size_t)u * nk * 8);
    pmemcpy(out_vals + offs[i], stg + (size_t)rows * nk * 8, (size_t)u * 8);
    return TK_OK;
  };
  if (int rc = copy_in(0)) return rc;
  for (int i = 0; i < nchunk; ++i) {
    const int b = i & 1;
    const int64_t n = cut[i + 1] - cut[i];
    if (i + 1 < nchunk) {  // the other buffer set is free once chunk i-1's TTV has run (host-synced)
      if (int rc = copy_in(i + 1)) return rc;
    }
    TK_CUDA(cudaStreamWaitEvent(sc, ev_in[b], 0));
    if (i >= 2) TK_CUDA(cudaStreamWaitEvent(sc, ev_free[b], 0));  // chunk i-2's result copied out
    if (packed[b] && !pin_in) {
      if (int rc = unpack_rows(rp, n, b_aos[b].as<uint64_t>(), b_soa[b].as<int64_t>(), pitch, sc)) return rc;
    } else {
      if (int rc = aos_to_soa(n, d, b_aos[b].as<int64_t>(), b_soa[b].as<int64_t>(), pitch, sc)) return rc;
    }
    std::vector<const int64_t*> cp(d);
    for (int m = 0; m < d; ++m) cp[m] = b_soa[b].as<int64_t>() + (size_t)m * pitch;
    int64_t u = 0;
    bool unsorted = false;
    if (int rc = ttv_prefix_try(d, n, cp.data(), b_vals[b].as<double>(), b_x.as<double>(), nx, b_os[b].as<int64_t>(),
                                b_ov[b].as<double>(), &u, &unsorted, sc))
      return rc;
    if (unsorted) return kPipeDeclined;
    us[i] = u;
    offs[i + 1] = offs[i] + u;
    TK_CUDA(cudaEventRecord(ev_done[b], sc));
    TK_CUDA(cudaStreamWaitEvent(so, ev_done[b], 0));
    if (u) {
      if (pin_out) {
        TK_CUDA(cudaMemcpyAsync(out_subs + offs[i] * nk, b_os[b].get(), (size_t)u * nk * 8, cudaMemcpyDeviceToHost, so));
        TK_CUDA(cudaMemcpyAsync(out_vals + offs[i], b_ov[b].get(), (size_t)u * 8, cudaMemcpyDeviceToHost, so));
      } else {
        char* stg = ps->out + (size_t)b * ps->out_half;
        TK_CUDA(cudaMemcpyAsync(stg, b_os[b].get(), (size_t)u * nk * 8, cudaMemcpyDeviceToHost, so));
        TK_CUDA(cudaMemcpyAsync(stg + (size_t)rows * nk * 8, b_ov[b].get(), (size_t)u * 8, cudaMemcpyDeviceToHost, so));
      }
    }
    TK_CUDA(cudaEventRecord(ev_free[b], so));
    if (!pin_out && i >= 1)
      if (int rc = copy_out_host(i - 1)) return rc;
  }
  {
    auto sp = pt.span(4);
    TK_CUDA(cudaStreamSynchronize(so));
    TK_CUDA(cudaStreamSynchronize(sc));
  }
  if (!pin_out && nchunk >= 1)
    if (int rc = copy_out_host(nchunk - 1)) return rc;
  *out_nnz = offs[nchunk];
  return TK_OK;
}

int tk_ttv_f64_host(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* subs, const double* vals,
                    const double* x, int64_t nx, int32_t k, int64_t* out_subs, double* out_vals, int64_t* out_nnz) {
  CallClock clock_;
  if (int rc = check_ttv_args(d, shape, k, nx)) return rc;
  if (nnz < 0 || out_nnz == nullptr) return fail(TK_EARG, "ttv: bad nnz / out_nnz");
  *out_nnz = 0;
  if (nnz == 0) return TK_OK;
  if (k == d - 1 && nnz >= 2 * kPipeRows) {
    const int rc = ttv_host_pipelined(d, shape, nnz, subs, vals, x, nx, out_subs, out_vals, out_nnz);
    if (rc != kPipeDeclined) return rc;
    *out_nnz = 0;
  }
  cudaStream_t st = lib_stream();
  const int64_t pitch = pitch_of(nnz);
  const int nk = d - 1;
  DevBuf b_aos, b_soa, b_vals, b_x, b_os, b_ov;
  if (int rc = b_aos.alloc((size_t)nnz * d * 8, st)) return rc;
  if (int rc = b_soa.alloc((size_t)pitch * d * 8, st)) return rc;
  if (int rc = b_vals.alloc((size_t)nnz * 8, st)) return rc;
  if (int rc = b_x.alloc((size_t)std::max<int64_t>(nx, 1) * 8, st)) return rc;
  if (int rc = b_os.alloc((size_t)nnz * nk * 8, st)) return rc;
  if (int rc = b_ov.alloc((size_t)nnz * 8, st)) return rc;
  if (int rc = h2d(b_aos.get(), subs, (size_t)nnz * d * 8, st)) return rc;
  if (int rc = h2d(b_vals.get(), vals, (size_t)nnz * 8, st)) return rc;
  if (int rc = h2d(b_x.get(), x, (size_t)nx * 8, st)) return rc;
  if (int rc = aos_to_soa(nnz, d, b_aos.as<int64_t>(), b_soa.as<int64_t>(), pitch, st)) return rc;
  b_aos.reset();
  std::vector<const int64_t*> cp(d);
  for (int m = 0; m < d; ++m) cp[m] = b_soa.as<int64_t>() + (size_t)m * pitch;
  int64_t u = 0;
  if (int rc = ttv_sparse_device(d, shape, nnz, cp.data(), b_vals.as<double>(), b_x.as<double>(), nx, k,
                                 b_os.as<int64_t>(), b_ov.as<double>(), &u, st))
    return rc;
  if (int rc = d2h(out_subs, b_os.get(), (size_t)u * nk * 8, st)) return rc;
  if (int rc = d2h(out_vals, b_ov.get(), (size_t)u * 8, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  *out_nnz = u;
  return TK_OK;
}

int tk_group_sum_f64_host(int64_t n, int32_t m, const int64_t* keys, const double* weights, int64_t* out_keys,
                          double* out_sums, int64_t* out_u) {
  CallClock clock_;
  if (n < 0 || m < 1 || m + 1 > TK_MAX_ORDER || !out_u) return fail(TK_EARG, "group_sum: bad arguments");
  *out_u = 0;
  if (n == 0) return TK_OK;
  cudaStream_t st = lib_stream();
  const int d = m + 1;
  const int64_t pitch = pitch_of(n);
  DevBuf b_aos, b_soa, b_w, b_one, b_os, b_ov;
  if (int rc = b_aos.alloc((size_t)n * m * 8, st)) return rc;
  if (int rc = b_soa.alloc((size_t)pitch * d * 8, st)) return rc;
  if (int rc = b_w.alloc((size_t)n * 8, st)) return rc;
  if (int rc = b_one.alloc(16, st)) return rc;
  if (int rc = b_os.alloc((size_t)n * m * 8, st)) return rc;
  if (int rc = b_ov.alloc((size_t)n * 8, st)) return rc;
  static const double one = 1.0;
  if (int rc = h2d(b_aos.get(), keys, (size_t)n * m * 8, st)) return rc;
  if (int rc = h2d(b_w.get(), weights, (size_t)n * 8, st)) return rc;
  TK_CUDA(cudaMemcpyAsync(b_one.get(), &one, 8, cudaMemcpyHostToDevice, st));
  if (int rc = aos_to_soa(n, m, b_aos.as<int64_t>(), b_soa.as<int64_t>(), pitch, st)) return rc;
  TK_CUDA(cudaMemsetAsync(b_soa.as<int64_t>() + (size_t)m * pitch, 0, (size_t)n * 8, st));
  std::vector<const int64_t*> cp(d);
  for (int c = 0; c < d; ++c) cp[c] = b_soa.as<int64_t>() + (size_t)c * pitch;
  // keys are arbitrary int64: declare unbounded kept dims so the sort path compares raw values
  std::vector<int64_t> shape(d, INT64_MAX);
  shape[m] = 1;
  int64_t u = 0;
  // w = weight * 1.0 is exact, so this is the reference's group-by-sum in original row order
  if (int rc = ttv_sparse_device(d, shape.data(), n, cp.data(), b_w.as<double>(), b_one.as<double>(), 1, m,
                                 b_os.as<int64_t>(), b_ov.as<double>(), &u, st, /*keep_zeros=*/true))
    return rc;
  if (int rc = d2h(out_keys, b_os.get(), (size_t)u * m * 8, st)) return rc;
  if (int rc = d2h(out_sums, b_ov.get(), (size_t)u * 8, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  *out_u = u;
  return TK_OK;
}

int tk_ttv_dense_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                            const int64_t* subs, const double* vals, int32_t keep, const double* const* vecs,
                            double* out, void* stream) {
  if (d < 2) return fail(TK_EORDER, fmt("ttv: tensor order must be at least 2, got %lld", d));
  if (keep < 0 || keep >= d) return fail(TK_EMODE, fmt("ttv: mode %lld out of range for order-%lld tensor", keep, d));
  if (d > TK_MAX_ORDER) return fail(TK_EARG, "ttv: tensor order exceeds TK_MAX_ORDER");
  if (nnz < 0 || !shape || !vecs || !out) return fail(TK_EARG, "ttv_dense: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevBuf soa;
  std::vector<const int64_t*> cp(d);
  if (cols) {
    for (int m = 0; m < d; ++m) cp[m] = cols[m];
  } else {
    const int64_t pitch = pitch_of(nnz);
    if (int rc = soa.alloc((size_t)pitch * d * 8, st)) return rc;
    if (int rc = aos_to_soa(nnz, d, subs, soa.as<int64_t>(), pitch, st)) return rc;
    for (int m = 0; m < d; ++m) cp[m] = soa.as<int64_t>() + (size_t)m * pitch;
  }
  return ttv_dense_device(d, shape, nnz, cp.data(), vals, keep, vecs, out, st);
}

int tk_ttv_dense_f64_device_peers(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                                  const double* vals, int32_t keep, const double* const* vecs,
                                  double* const* outs, int32_t nout, int64_t key_lo, int64_t key_hi,
                                  void* stream) {
  if (d < 2) return fail(TK_EORDER, fmt("ttv: tensor order must be at least 2, got %lld", d));
  if (keep < 0 || keep >= d) return fail(TK_EMODE, fmt("ttv: mode %lld out of range for order-%lld tensor", keep, d));
  if (d > TK_MAX_ORDER) return fail(TK_EARG, "ttv: tensor order exceeds TK_MAX_ORDER");
  if (nnz < 0 || !shape || !vecs || !outs || !cols || nout < 1 || nout > 8)
    return fail(TK_EARG, "ttv_dense_peers: bad arguments");
  if (key_lo < 0 || key_hi > shape[keep] || key_lo > key_hi)
    return fail(TK_EARG, "ttv_dense_peers: owned range outside the keep-mode dimension");
  for (int i = 0; i < nout; ++i)
    if (!outs[i]) return fail(TK_EARG, "ttv_dense_peers: null output");
  return ttv_dense_peers(d, shape, nnz, cols, vals, keep, vecs, outs, nout, key_lo, key_hi,
                         static_cast<cudaStream_t>(stream));
}

// ---- workspace, timed forms, one-process multi-GPU ----------------------------

int tk_ttv_workspace(int32_t d, int64_t nnz, int32_t nkeep, size_t* bytes) {
  if (!bytes || d < 2 || nnz < 0 || nkeep < 1) return fail(TK_EARG, "ttv_workspace: bad arguments");
  const size_t n = (size_t)nnz;
  const size_t tiles = n / 256 + 2;                      // smallest tile geometry
  const size_t fast = tiles * 8 + 4096;                  // status words + counters
  const size_t sort = n * 8 * 5 + n * 12 + (64u << 20);  // keys/w double buffers, 32-bit split keys, CUB temp
  const size_t lsd = n * 8 * (4 + (size_t)nkeep) + (64u << 20);  // garbage-key path: permutation + sorted columns
  *bytes = std::max(fast, std::max(sort, lsd)) + n * 8 * (size_t)d;  // + SoA transpose when subs is row-major
  return TK_OK;
}

namespace {
struct EventTimer {  // cudaEvent pair on `st` around a call
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  explicit EventTimer(cudaStream_t s) : st(s) {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  int stop(float* ms) {
    TK_CUDA(cudaEventRecord(b, st));
    TK_CUDA(cudaEventSynchronize(b));
    TK_CUDA(cudaEventElapsedTime(ms, a, b));
    return TK_OK;
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};
}  // namespace

int tk_dot_f64_device_timed(const double* x, const double* y, int64_t n, double* out, void* stream,
                            float* elapsed_ms) {
  if (!elapsed_ms) return fail(TK_EARG, "dot_timed: null elapsed_ms");
  EventTimer t(static_cast<cudaStream_t>(stream));
  if (int rc = tk_dot_f64_device(x, y, n, out, stream)) return rc;
  return t.stop(elapsed_ms);
}

int tk_matvec_f64_device_timed(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                               void* stream, float* elapsed_ms) {
  if (!elapsed_ms) return fail(TK_EARG, "matvec_timed: null elapsed_ms");
  EventTimer t(static_cast<cudaStream_t>(stream));
  if (int rc = tk_matvec_f64_device(a, rows, cols, x, y, stream)) return rc;
  return t.stop(elapsed_ms);
}

int tk_ttv_f64_device_timed(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                            const int64_t* subs, const double* vals, const double* x, int64_t nx, int32_t k,
                            int64_t* out_subs, double* out_vals, int64_t* out_nnz, void* stream,
                            float* elapsed_ms) {
  if (!elapsed_ms) return fail(TK_EARG, "ttv_timed: null elapsed_ms");
  EventTimer t(static_cast<cudaStream_t>(stream));
  if (int rc = tk_ttv_f64_device(d, shape, nnz, cols, subs, vals, x, nx, k, out_subs, out_vals, out_nnz, stream))
    return rc;
  return t.stop(elapsed_ms);
}

namespace {
std::mutex g_multi_mu;
std::vector<int> g_multi_dev;
std::vector<cudaStream_t> g_multi_st;
}  // namespace

int tk_multi_init(int32_t ndev, const int32_t* devices) {
  if (ndev < 1 || !devices) return fail(TK_EARG, "multi_init: bad arguments");
  std::lock_guard<std::mutex> lk(g_multi_mu);
  int prev = 0;
  TK_CUDA(cudaGetDevice(&prev));
  for (cudaStream_t s : g_multi_st) cudaStreamDestroy(s);
  g_multi_dev.assign(devices, devices + ndev);
  g_multi_st.assign(ndev, nullptr);
  for (int i = 0; i < ndev; ++i) {
    TK_CUDA(cudaSetDevice(devices[i]));
    TK_CUDA(cudaStreamCreateWithFlags(&g_multi_st[i], cudaStreamNonBlocking));
    for (int j = 0; j < ndev; ++j) {
      if (devices[j] == devices[i]) continue;
      int can = 0;
      TK_CUDA(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
      if (can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    }
  }
  TK_CUDA(cudaSetDevice(prev));
  return TK_OK;
}

int tk_multi_ttv_f64(int32_t d, const int64_t* shape, int32_t k, int32_t nshard, const int32_t* shard_device,
                     const int64_t* shard_nnz, const int64_t* const* const* shard_cols,
                     const double* const* shard_vals, const double* const* shard_x, int64_t nx,
                     int64_t* const* shard_out_subs, double* const* shard_out_vals, int64_t* shard_out_nnz,
                     int64_t* out_offsets) {
  if (int rc = check_ttv_args(d, shape, k, nx)) return rc;
  if (nshard < 1 || !shard_device || !shard_nnz || !shard_cols || !shard_vals || !shard_x || !shard_out_subs ||
      !shard_out_vals || !shard_out_nnz || !out_offsets)
    return fail(TK_EARG, "multi_ttv: bad arguments");
  std::vector<cudaStream_t> st(nshard);
  {
    std::lock_guard<std::mutex> lk(g_multi_mu);
    for (int s = 0; s < nshard; ++s) {
      size_t i = 0;
      while (i < g_multi_dev.size() && g_multi_dev[i] != shard_device[s]) ++i;
      if (i == g_multi_dev.size()) return fail(TK_EARG, "multi_ttv: shard device not in tk_multi_init's list");
      st[s] = g_multi_st[i];
    }
  }
  std::vector<int> rcs(nshard, TK_OK);
  std::vector<std::string> errs(nshard);
  int caller_dev = 0;
  TK_CUDA(cudaGetDevice(&caller_dev));
  // one shard per worker of the persistent host pool (no per-call threads: the workers' cached
  // pinned scratch and timing events are reused across calls)
  parallel_for(nshard, [&](int s) {
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(shard_device[s]) != cudaSuccess) {
      rcs[s] = TK_ECUDA;
      errs[s] = "cudaSetDevice failed";
      return;
    }
    rcs[s] = tk_ttv_f64_device(d, shape, shard_nnz[s], shard_cols[s], nullptr, shard_vals[s], shard_x[s], nx, k,
                               shard_out_subs[s], shard_out_vals[s], &shard_out_nnz[s], st[s]);
    if (rcs[s]) errs[s] = tk_last_error();
    cudaSetDevice(prev);
  });
  TK_CUDA(cudaSetDevice(caller_dev));
  for (int s = 0; s < nshard; ++s)
    if (rcs[s]) return fail(rcs[s], errs[s]);  // the error message is thread-local: carry it over
  out_offsets[0] = 0;
  for (int s = 0; s < nshard; ++s) out_offsets[s + 1] = out_offsets[s] + shard_out_nnz[s];
  return TK_OK;
}

int tk_multi_free(void) {
  std::lock_guard<std::mutex> lk(g_multi_mu);
  for (cudaStream_t s : g_multi_st) cudaStreamDestroy(s);
  g_multi_st.clear();
  g_multi_dev.clear();
  return TK_OK;
}

int tk_ipc_alloc(int64_t bytes, void** dev_ptr) {
  if (!dev_ptr || bytes <= 0) return fail(TK_EARG, "ipc: bad allocation request");
  TK_CUDA(cudaMalloc(dev_ptr, (size_t)bytes));
  return TK_OK;
}

int tk_ipc_free(void* dev_ptr) {
  if (!dev_ptr) return fail(TK_EARG, "ipc: null argument");
  TK_CUDA(cudaFree(dev_ptr));
  return TK_OK;
}

int tk_ipc_get_handle(const void* dev_ptr, void* handle64) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!dev_ptr || !handle64) return fail(TK_EARG, "ipc: null argument");
  cudaIpcMemHandle_t h;
  TK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  memcpy(handle64, &h, sizeof h);
  return TK_OK;
}

int tk_ipc_open(const void* handle64, void** dev_ptr) {
  if (!dev_ptr || !handle64) return fail(TK_EARG, "ipc: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof h);
  TK_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TK_OK;
}

int tk_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return fail(TK_EARG, "ipc: null argument");
  TK_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return TK_OK;
}

// ---- MTTKRP (the R-column TTV) ------------------------------------------------

static int mttkrp_check(int32_t d, const int64_t* shape, int64_t nnz, int32_t n, int64_t rank, const void* factors,
                        const void* out) {
  if (d < 2) return fail(TK_EORDER, fmt("mttkrp: tensor order must be at least 2, got %lld", d));
  if (n < 0 || n >= d) return fail(TK_EMODE, fmt("mttkrp: mode %lld out of range for order-%lld tensor", n, d));
  if (d > TK_MAX_ORDER) return fail(TK_EARG, "mttkrp: tensor order exceeds TK_MAX_ORDER");
  if (rank < 0 || rank > 128) return fail(TK_EARG, "mttkrp: rank must be in [0, 128]");
  if (nnz < 0 || !shape || !factors || !out) return fail(TK_EARG, "mttkrp: bad arguments");
  for (int m = 0; m < d; ++m)
    if (shape[m] <= 0) return fail(TK_EARG, "mttkrp: shape entries must be positive");
  return TK_OK;
}

int tk_mttkrp_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                         const int64_t* subs, const double* vals, int32_t n, int64_t rank,
                         const double* const* factors, double* out, void* stream) {
  CallClock clock_;
  if (int rc = mttkrp_check(d, shape, nnz, n, rank, factors, out)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevBuf soa;
  std::vector<const int64_t*> cp(d);
  if (cols) {
    for (int m = 0; m < d; ++m) cp[m] = cols[m];
  } else {
    const int64_t pitch = pitch_of(nnz);
    if (int rc = soa.alloc((size_t)pitch * d * 8, st)) return rc;
    if (int rc = aos_to_soa(nnz, d, subs, soa.as<int64_t>(), pitch, st)) return rc;
    for (int m = 0; m < d; ++m) cp[m] = soa.as<int64_t>() + (size_t)m * pitch;
  }
  return mttkrp_device(d, shape, nnz, cp.data(), vals, n, rank, factors, out, st);
}

int tk_mttkrp_f64_host(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* subs, const double* vals,
                       int32_t n, int64_t rank, const double* const* factors, double* out) {
  CallClock clock_;
  if (int rc = mttkrp_check(d, shape, nnz, n, rank, factors, out)) return rc;
  cudaStream_t st = lib_stream();
  const int64_t pitch = pitch_of(nnz);
  size_t fac_elems = 0;
  for (int m = 0; m < d; ++m)
    if (m != n) fac_elems += (size_t)pitch_of(shape[m] * rank);
  DevBuf b_aos, b_soa, b_vals, b_fac, b_out;
  if (int rc = b_aos.alloc((size_t)std::max<int64_t>(nnz, 1) * d * 8, st)) return rc;
  if (int rc = b_soa.alloc((size_t)pitch * d * 8 + 8, st)) return rc;
  if (int rc = b_vals.alloc((size_t)pitch * 8 + 8, st)) return rc;
  if (int rc = b_fac.alloc(fac_elems * 8 + 8, st)) return rc;
  if (int rc = b_out.alloc((size_t)shape[n] * rank * 8 + 8, st)) return rc;
  if (nnz) {
    if (int rc = h2d(b_aos.get(), subs, (size_t)nnz * d * 8, st)) return rc;
    if (int rc = h2d(b_vals.get(), vals, (size_t)nnz * 8, st)) return rc;
    if (int rc = aos_to_soa(nnz, d, b_aos.as<int64_t>(), b_soa.as<int64_t>(), pitch, st)) return rc;
  }
  std::vector<const double*> fp(d, nullptr);
  std::vector<const int64_t*> cp(d);
  size_t off = 0;
  for (int m = 0; m < d; ++m) {
    cp[m] = b_soa.as<int64_t>() + (size_t)m * pitch;
    if (m == n) continue;
    double* dst = b_fac.as<double>() + off;
    if (shape[m] > 0 && rank > 0)
      if (int rc = h2d(dst, factors[m], (size_t)shape[m] * rank * 8, st)) return rc;
    fp[m] = dst;
    off += (size_t)pitch_of(shape[m] * rank);
  }
  if (int rc = mttkrp_device(d, shape, nnz, cp.data(), b_vals.as<double>(), n, rank, fp.data(), b_out.as<double>(), st))
    return rc;
  if (int rc = d2h(out, b_out.get(), (size_t)shape[n] * rank * 8, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

// ---- generators -------------------------------------------------------------------------------

int tk_gen_coo_device(int32_t d, const int64_t* shape, int64_t nnz, double zipf_s, int32_t normal_vals,
                      uint64_t seed, int64_t* const* cols, double* vals, void* stream) {
  if (d < 1 || d > TK_MAX_ORDER || !shape || !cols || !vals || nnz < 0) return fail(TK_EARG, "gen: bad arguments");
  for (int m = 0; m < d; ++m)
    if (shape[m] <= 0) return fail(TK_EARG, "gen: shape entries must be positive");
  return gen_coo(d, shape, nnz, zipf_s, normal_vals, seed, cols, vals, static_cast<cudaStream_t>(stream));
}

int tk_gen_uniform_device(int64_t n, uint64_t seed, double* out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (int rc = gen_uniform(n, seed, out, st)) return rc;
  TK_CUDA(cudaStreamSynchronize(st));
  return TK_OK;
}

// ---- timing -----------------------------------------------------------------------------------

int tk_timer_start(void* stream) {
  const int dev = cur_dev();
  for (int i = 0; i < 2; ++i)
    if (!g_ev[dev][i]) TK_CUDA(cudaEventCreate(&g_ev[dev][i]));
  TK_CUDA(cudaEventRecord(g_ev[dev][0], static_cast<cudaStream_t>(stream)));
  return TK_OK;
}

int tk_timer_stop(void* stream, float* ms) {
  const int dev = cur_dev();
  if (!g_ev[dev][0]) return fail(TK_EARG, "timer: tk_timer_start was not called");
  TK_CUDA(cudaEventRecord(g_ev[dev][1], static_cast<cudaStream_t>(stream)));
  TK_CUDA(cudaEventSynchronize(g_ev[dev][1]));
  TK_CUDA(cudaEventElapsedTime(ms, g_ev[dev][0], g_ev[dev][1]));
  return TK_OK;
}

int tk_release(void) {
  int dev = cur_dev();
  cudaDeviceSynchronize();
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  if (g_pinned) cudaFreeHost(g_pinned);
  g_pinned = nullptr;
  g_pinned_bytes = 0;
  host_result_trim();
  return TK_OK;
}

int tk_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(TK_EARG, "host_alloc: null out");
  *out = host_result_alloc(bytes);
  return TK_OK;
}

int tk_host_free(void* p) {
  if (p && !host_result_free(p)) return fail(TK_EARG, "host_free: not a block from tk_host_alloc");
  return TK_OK;
}

}  // extern "C"
