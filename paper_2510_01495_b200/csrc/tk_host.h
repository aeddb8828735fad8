// tk_host.h -- internal host-side API shared by the translation units of libtk_b200.so.
// (The public, stable surface is include/tk_b200.h.)
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <string>

#include <cuda_runtime.h>

#include "../../include/tk_b200.h"

namespace tk {

// Thread-local last-error message, returned by tk_last_error().
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define TK_CUDA(expr)                                         \
  do {                                                        \
    cudaError_t tk_e_ = (expr);                               \
    if (tk_e_ != cudaSuccess) return cuda_fail(tk_e_, #expr); \
  } while (0)

// Stream-ordered scratch from the device's default memory pool.  The pool keeps freed
// blocks (release threshold raised at first use), so steady-state calls allocate nothing.
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_), st_(o.st_) { o.ptr_ = nullptr; o.bytes_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      ptr_ = o.ptr_; bytes_ = o.bytes_; st_ = o.st_;
      o.ptr_ = nullptr; o.bytes_ = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  int alloc(size_t bytes, cudaStream_t st);
  void reset();
  template <class T>
  T* as() const { return static_cast<T*>(ptr_); }
  void* get() const { return ptr_; }
  size_t size() const { return bytes_; }

 private:
  void* ptr_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t st_ = nullptr;
};

// Small per-thread pinned host block used to read back per-call counters.
void* pinned_scratch(size_t bytes);

int num_sms();
void prepare_pool();

// Instrumentation read by bench.py: CUDA events around the primary kernel of the last call
// (recorded on the launching stream) and a count of this library's kernel launches.
void ktimer_begin(cudaStream_t st);
void ktimer_end(cudaStream_t st);
void count_launch(int n = 1);

// sparse-result TTV on device-resident SoA data (cols[m] device pointers, m < d).
// Prefix-kept TTV (k == d-1) over device SoA columns without the sort fallback: *unsorted is set
// (and nothing written) when the kept keys are not non-decreasing.
int ttv_prefix_try(int d, int64_t nnz, const int64_t* const* cols, const double* vals, const double* x, int64_t nx,
                   int64_t* out_subs, double* out_vals, int64_t* out_nnz, bool* unsorted, cudaStream_t st);
int ttv_sparse_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                      const double* x, int64_t nx, int k, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                      cudaStream_t st, bool keep_zeros = false);

// dense-result multi-vector TTV (every mode except `keep` contracted).
// Contracted mode 1 over canonical input (the paper's middle-mode protocol): segmented counting
// by the suffix key (tk_midmode.cu).  Returns kMidDeclined when it does not apply.
constexpr int kMidDeclined = -1;
int ttv_middle_mode(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    const double* x, int64_t nx, int64_t* out_subs, double* out_vals, int64_t* out_nnz,
                    cudaStream_t st, bool keep_zeros);
// stable removal of exact-zero groups from a (groups, nk) result (tk_ttv.cu)
int compact_zeros(long long groups, int nk, long long* out_subs, double* out_vals, cudaStream_t st);

int ttv_dense_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                     int keep, const double* const* vecs, double* out, cudaStream_t st);

// The same with the result for keep-mode indices [key_lo, key_hi) stored into every one of
// outs[0..nout) (this GPU's vector and NVLink-mapped peer vectors: the sharded merge).
int ttv_dense_peers(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    int keep, const double* const* vecs, double* const* outs, int nout, long long key_lo,
                    long long key_hi, cudaStream_t st);
int ttv_dense_chain(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals,
                    int keep, const double* const* vecs, double* out, cudaStream_t st);

// row-major (nnz, d) -> SoA columns with the given pitch (elements)
int mttkrp_device(int d, const int64_t* shape, int64_t nnz, const int64_t* const* cols, const double* vals, int mode,
                  int64_t R, const double* const* factors, double* out, cudaStream_t st);
int aos_to_soa(int64_t nnz, int d, const int64_t* aos, int64_t* soa, int64_t pitch, cudaStream_t st);

// ---- host side of the host-buffer calls (tk_hostio.cu) ----
int host_threads();
void parallel_for(int n, const std::function<void(int)>& fn);  // persistent host thread pool
void pmemcpy(void* dst, const void* src, size_t bytes);          // parallel host memcpy
bool host_is_pinned(const void* p);
// cached pinned result blocks (capped at a quarter of host RAM, TK_HOST_POOL_MB overrides);
// alloc returns nullptr when the cap is reached
void* host_result_alloc(size_t bytes);
bool host_result_free(void* p);
void host_result_trim();
// H2D / D2H of caller host memory: pinned -> direct DMA; pageable -> chunked through a per-device
// pinned arena (parallel host copy of chunk i+1 overlapping the DMA of chunk i).  h2d is
// stream-ordered (the source may be reused on return); d2h returns with the data on the host.
int h2d(void* dst, const void* src, size_t bytes, cudaStream_t st);
int d2h(void* dst, const void* src, size_t bytes, cudaStream_t st);
// Packed tensor rows: coordinate m of a row in bits [shift[m], shift[m] + bits(dim[m]-1)) of one
// 64-bit word (only when the bit widths sum to <= 64 and every index is inside its dimension).
struct RowPack {
  int d;
  int shift[TK_MAX_ORDER];
  uint64_t dim[TK_MAX_ORDER];
};
bool row_pack_plan(int d, const int64_t* shape, RowPack* p);
// packs n row-major rows and copies their values (parallel); false if some index is out of range
bool pack_rows(const RowPack& p, const int64_t* subs, const double* vals, int64_t n, uint64_t* packed,
               double* vals_out);
int unpack_rows(const RowPack& p, int64_t n, const uint64_t* packed, int64_t* soa, int64_t pitch, cudaStream_t st);

int dot_device(const double* x, const double* y, int64_t n, double* out, cudaStream_t st);
int read_floor_device(const double* p, int64_t n, double* sink, cudaStream_t st);
int matvec_device(const double* a, int64_t rows, int64_t cols, const double* x, double* y, cudaStream_t st);

}  // namespace tk
