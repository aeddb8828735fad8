/*
 * tk_b200.h -- C ABI of libtk_b200.so, the B200 (sm_100a) kernel library behind the
 * drop-in kernel module paper_2510_01495_b200 (BACKEND "b200").
 *
 * It replaces the reference's native kernel module, pkg/src/tenkern/_ckernels.pyx,
 * which the reference reaches through its kernel-module protocol
 * (pkg/src/tenkern/backend.py:33-49) and its FFI wrapper BoundKernelSet
 * (pkg/hostbench/src/tenhost/bindings.py:40-79).  Each entry point below names the
 * reference function whose contract it carries.
 *
 * Conventions
 *   - every function returns a tk_status; on failure tk_last_error() holds a message
 *     (thread-local) worded like the reference's exception text;
 *   - *_device functions take DEVICE pointers and a cudaStream_t passed as void*;
 *     they return after the result (and *out_nnz) is final on the host;
 *   - *_host functions take HOST pointers (pinned or pageable) and move the data
 *     themselves: this is the call a cgo / JNI / ctypes binding of the reference's
 *     ttv_raw / dot / matvec would make;
 *   - inputs are borrowed read-only (the reference takes const memoryviews,
 *     _ckernels.pyx:40, 48, 129), outputs are caller-owned;
 *   - mode numbers are 0-based like tenkern.ttv (sparse.py:213);
 *   - subs are int64; vals / vectors float64 (the reference's boundary dtypes,
 *     bindings.py:19-37);
 *   - one call at a time per device (the reference is single-threaded).
 */
#ifndef TK_B200_H
#define TK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tk_status {
  TK_OK = 0,
  TK_EDIM = 1,     /* tenkern.DimensionError  (lengths / shapes / mode-k index)       */
  TK_EMODE = 2,    /* tenkern.ModeError       (k outside [0, d))                       */
  TK_EORDER = 3,   /* tenkern.OrderError      (d < 2)                                  */
  TK_EINDEX = 4,   /* tenkern.DimensionError  (mode-k index outside x, pyx:361-365)    */
  TK_ECUDA = 6,    /* CUDA runtime failure                                             */
  TK_ENCCL = 7,    /* NCCL failure (library missing, communicator or collective error) */
  TK_EARG = 8,     /* unsupported argument (e.g. order > TK_MAX_ORDER, null pointer)   */
  TK_ENOMEM = 9    /* device allocation failed                                         */
} tk_status;

#define TK_MAX_ORDER 16

/* Message for the last failing call on this thread ("" if none). */
const char* tk_last_error(void);
/* ABI version: major*10000 + minor*100 + patch. */
int tk_version(void);
/* Seconds spent inside the last *_host call on this thread, measured on the native side
 * with a monotonic clock (the reference's *_timed protocol, _ckernels.pyx:98-122, 377-388). */
double tk_last_call_seconds(void);
/* Number of visible CUDA devices (0 when none). */
int tk_device_count(int* n);

/* ---- dense kernels ---------------------------------------------------------------------- */

/* Sum_i x[i]*y[i] -> *out (device double).  Replaces _ckernels.dot / _dot_impl
 * (_ckernels.pyx:40-45, 76-83).  Parallel tree order: within 1e-12 relative of the
 * reference's left-to-right sum (documented deviation). */
int tk_dot_f64_device(const double* x, const double* y, int64_t n, double* out, void* stream);
/* Same with host operands and a host result; copies included. */
int tk_dot_f64_host(const double* x, const double* y, int64_t n, double* out);

/* y[i] = Sum_j A[i*cols+j]*x[j], A row-major.  Replaces _ckernels.matvec / _matvec_impl
 * (_ckernels.pyx:48-56, 86-95). */
int tk_matvec_f64_device(const double* a, int64_t rows, int64_t cols, const double* x, double* y, void* stream);
int tk_matvec_f64_host(const double* a, int64_t rows, int64_t cols, const double* x, double* y);

/* ---- sparse tensor-times-vector ---------------------------------------------------------- */

/* Mode-k TTV of a COO tensor; sparse result in canonical form.
 * Replaces _ckernels.ttv_raw / _ttv_pipeline (_ckernels.pyx:313-374).
 *
 *   d, shape[d]        tensor order and shape (host array)
 *   nnz                stored entries
 *   cols               host array of d DEVICE pointers, cols[m][r] = subs[r, m] (SoA);
 *                      or NULL, then `subs` is a DEVICE row-major (nnz, d) array
 *   vals[nnz], x[nx]   device
 *   k                  contracted mode (0-based)
 *   out_subs           device, capacity nnz*(d-1), written row-major (u, d-1)
 *   out_vals           device, capacity nnz
 *   out_nnz            HOST: number u of output entries
 * Values are bit-identical to the reference: each group is summed left to right in
 * ascending original-row order with round-to-nearest adds, exact zeros dropped. */
int tk_ttv_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                      const int64_t* subs, const double* vals, const double* x, int64_t nx, int32_t k,
                      int64_t* out_subs, double* out_vals, int64_t* out_nnz, void* stream);

/* Host-buffer form of tk_ttv_f64_device: subs row-major (nnz, d) int64, vals, x on the host;
 * out_subs (capacity nnz*(d-1)) and out_vals (capacity nnz) on the host.  This is the exact
 * argument list of the reference's ttv_raw(subs, vals, shape, x, k) (_ckernels.pyx:370-374,
 * bindings.py:68-79) flattened to pointers. */
int tk_ttv_f64_host(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* subs, const double* vals,
                    const double* x, int64_t nx, int32_t k, int64_t* out_subs, double* out_vals,
                    int64_t* out_nnz);

/* Unique rows of keys (host, row-major (n, m) int64) in lexicographic order with the sum
 * of their weights, each group summed left to right in ascending original-row order; zero
 * sums are KEPT.  Replaces tenkern.unique_rows_accumulate (sparse.py:179-197,
 * _pykernels.py:43-68), which also canonicalises SparseCooTensor input (sparse.py:90-99).
 * out_keys capacity n*m, out_sums capacity n (host). */
int tk_group_sum_f64_host(int64_t n, int32_t m, const int64_t* keys, const double* weights, int64_t* out_keys,
                          double* out_sums, int64_t* out_u);

/* Multi-vector TTV to a dense vector: every mode except `keep` is contracted with
 * vecs[m] (host array of d device pointers, vecs[keep] ignored), out[shape[keep]] dense.
 * Defined as the chained single-mode ttv in descending mode order followed by densify
 * (the reference has no multi-vector TTV).  Canonical input with
 * keep == 0 takes the fused single-pass kernel (values within 1e-12 relative of the chain);
 * anything else runs the chain on the GPU. */
int tk_ttv_dense_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                            const int64_t* subs, const double* vals, int32_t keep, const double* const* vecs,
                            double* out, void* stream);

/* Sharded form of tk_ttv_dense_f64_device (SURVEY.md 8e, config 4 on N GPUs): this GPU's
 * shard (rows split at keep-mode key changes) produces the result for keep-mode indices
 * [key_lo, key_hi) -- zeros for indices without rows -- and stores it straight into every
 * one of outs[0..nout) (host array of device pointers: this GPU's output vector and the
 * peers' output vectors mapped over NVLink with tk_ipc_open).  The N shards together write
 * every element of every copy exactly once, so after a barrier every GPU holds the full,
 * bit-identical result: this replaces the all-reduce of the reference-style merge
 * (multi.merge_dense) with the kernel's own epilogue stores.  nout <= 8. */
int tk_ttv_dense_f64_device_peers(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                                  const double* vals, int32_t keep, const double* const* vecs,
                                  double* const* outs, int32_t nout, int64_t key_lo, int64_t key_hi,
                                  void* stream);

/* CUDA IPC for the peer outputs: allocate / free an exportable device buffer (its own
 * cudaMalloc, so the handle maps to its first byte), export it (64-byte handle), map a peer's
 * exported buffer into this process (peer access enabled lazily), unmap it. */
int tk_ipc_alloc(int64_t bytes, void** dev_ptr);
int tk_ipc_free(void* dev_ptr);
int tk_ipc_get_handle(const void* dev_ptr, void* handle64);
int tk_ipc_open(const void* handle64, void** dev_ptr);
int tk_ipc_close(void* dev_ptr);

/* Sparse MTTKRP: out(i_n, r) = sum over nonzeros of val * prod_{m != n} U_m(i_m, r), r < rank
 * (rank <= 128).  factors: host array of d pointers (factors[n] ignored) to row-major
 * (shape[m] x rank) matrices; out row-major (shape[n] x rank), dense.  Column r equals the
 * multi-vector TTV of every mode but n with the vectors U_m(:, r) (the paper's named consumer
 * of TTV; the reference has no MTTKRP, so its oracle is the reference's
 * ttv_raw chained per column).  Each column is folded left to right in the kept mode's sorted
 * row order (deterministic); canonical input with n == 0 streams without a sort, other modes
 * sort row ids stably by subs[:, n] on the device.  Values within 1e-12 relative of the chain
 * for non-cancelling data.  _device: cols/subs/vals/factors/out on the device; _host: all on
 * the host (subs row-major (nnz, d)). */
int tk_mttkrp_f64_device(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                         const int64_t* subs, const double* vals, int32_t n, int64_t rank,
                         const double* const* factors, double* out, void* stream);
int tk_mttkrp_f64_host(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* subs, const double* vals,
                       int32_t n, int64_t rank, const double* const* factors, double* out);

/* ---- synthetic operands (measurement inputs, generated on the device) ------------------- */

/* Exactly nnz distinct coordinates of a d-way tensor, drawn per mode from a truncated
 * Zipf(s) law on {0..shape[m]-1} (s <= 0: uniform), seeded counter-based RNG; the set is
 * the first nnz distinct draws of the sequence.  Sorted canonical SoA output
 * cols[m] (device, capacity nnz each).  vals: uniform [0,1) (normal_vals=0) or N(0,1)
 * (normal_vals=1), exact zeros redrawn.  Mirrors the exact-nnz protocol of gen_sparse3
 * (synth.py:103-143) generalised to order d and skewed coordinates (BASELINE configs 4, 5). */
int tk_gen_coo_device(int32_t d, const int64_t* shape, int64_t nnz, double zipf_s, int32_t normal_vals,
                      uint64_t seed, int64_t* const* cols, double* vals, void* stream);
/* Uniform [0,1) vector from the same counter-based generator. */
int tk_gen_uniform_device(int64_t n, uint64_t seed, double* out, void* stream);

/* ---- workspace, timed forms, one-process multi-GPU ---------------------- */

/* Upper bound of the device scratch a tk_ttv_f64_device call with these sizes takes from the
 * stream-ordered pool (sorted fast path; the general sort path; the larger of the two).  The
 * library allocates it itself; this is for callers sizing device memory. */
int tk_ttv_workspace(int32_t d, int64_t nnz, int32_t nkeep, size_t* bytes);

/* The device entry points with the call's device time: a cudaEvent pair recorded on `stream`
 * around the whole call (elapsed_ms, host).  The reference's self-timed protocol
 * (_ckernels.pyx:98-122, 377-388: dot_timed / matvec_timed / ttv_timed). */
int tk_dot_f64_device_timed(const double* x, const double* y, int64_t n, double* out, void* stream,
                            float* elapsed_ms);
int tk_matvec_f64_device_timed(const double* a, int64_t rows, int64_t cols, const double* x, double* y,
                               void* stream, float* elapsed_ms);
int tk_ttv_f64_device_timed(int32_t d, const int64_t* shape, int64_t nnz, const int64_t* const* cols,
                            const int64_t* subs, const double* vals, const double* x, int64_t nx, int32_t k,
                            int64_t* out_subs, double* out_vals, int64_t* out_nnz, void* stream,
                            float* elapsed_ms);

/* One process driving several GPUs (the torch.distributed path runs one process per GPU
 * instead; both shard the same way).  tk_multi_init enables peer access among
 * `devices` and creates a stream per device.  tk_multi_ttv_f64 runs the sparse-result TTV of
 * every shard concurrently (one host thread per shard): shard s is a contiguous row range of
 * the canonical tensor cut at kept-key changes, resident on device shard_device[s] (SoA
 * columns shard_cols[s][0..d), shard_vals[s], the vector shard_x[s]); its result goes to
 * shard_out_subs[s] / shard_out_vals[s] on that device, its count to shard_out_nnz[s], and
 * out_offsets[0..nshard] is the exclusive prefix of the counts: the rank-order concatenation is
 * the one-GPU result, bit for bit.  The first failing shard's status is returned. */
int tk_multi_init(int32_t ndev, const int32_t* devices);
int tk_multi_ttv_f64(int32_t d, const int64_t* shape, int32_t k, int32_t nshard, const int32_t* shard_device,
                     const int64_t* shard_nnz, const int64_t* const* const* shard_cols,
                     const double* const* shard_vals, const double* const* shard_x, int64_t nx,
                     int64_t* const* shard_out_subs, double* const* shard_out_vals, int64_t* shard_out_nnz,
                     int64_t* out_offsets);
int tk_multi_free(void);

/* ---- multi-GPU data plane: NCCL inside the library ------------------------
 * One process per GPU.  The reference has no distributed code; this is the
 * exchange the sharded TTV needs: per-rank result counts (offsets), the optional gather of the
 * sparse slices to a root, the IPC-handle exchange and stream-ordered barrier of the dense
 * peer-store merge, and the all-reduce merge baseline.  NCCL is bound at run time (dlopen; the
 * copy already in the process -- PyTorch's -- is reused, or the path given to tk_nccl_load).
 * Bootstrap: rank 0 calls tk_nccl_get_unique_id and ships the 128 bytes to the other ranks by
 * any means (torch.distributed broadcast); every rank then calls tk_nccl_comm_init on its
 * current device.  Collectives are enqueued on the caller's stream unless noted. */
int tk_nccl_load(const char* path);
int tk_nccl_version(int* version);
int tk_nccl_get_unique_id(void* id128);
int tk_nccl_comm_init(const void* id128, int32_t nranks, int32_t rank, void** comm);
int tk_nccl_comm_free(void* comm);
int tk_nccl_rank(void* comm, int32_t* rank, int32_t* nranks);
/* all-gather of one host count per rank, after `stream`, on the comm's own stream (non-blocking);
 * tk_nccl_counts_wait returns the counts (rank order) of a ticket */
int tk_nccl_counts_start(void* comm, int64_t count, void* stream, int32_t* ticket);
int tk_nccl_counts_wait(void* comm, int32_t ticket, int64_t* counts);
/* the ranks' (counts[r], nk) row-major slices gathered to `root` in rank order (device buffers) */
int tk_nccl_gather_rows(void* comm, int32_t root, const int64_t* subs, const double* vals, int32_t nk,
                        const int64_t* counts, int64_t* dst_subs, double* dst_vals, void* stream);
/* every rank's nbytes of host data to every rank (host buffers; synchronous) */
int tk_nccl_allgather_bytes(void* comm, const void* host_src, void* host_dst, int64_t nbytes);
int tk_nccl_barrier(void* comm, void* stream);
int tk_nccl_allreduce_sum_f64(void* comm, double* buf, int64_t n, void* stream);

/* Measurement floor, not a reference kernel: a read-only stream of n doubles (device pointer,
 * 16-byte aligned) with dot's load pattern and launch shape; its time under an L2 flush is the
 * cold-read floor the small configs are judged against (tk_last_kernel_ms). */
int tk_read_floor_f64_device(const double* p, int64_t n, double* sink, void* stream);

/* ---- timing helper ----------------------------------------------------------------------- */
/* Device milliseconds between two points on a stream (cudaEvent pair). */
int tk_timer_start(void* stream);
int tk_timer_stop(void* stream, float* ms);

/* Device milliseconds of the primary kernel(s) of the last call on this thread (the
 * streaming TTV kernel, the dense TTV kernel, dot's two reduction kernels, matvec), from
 * cudaEvents recorded on the launching stream; -1 if none.  Used for roofline reporting. */
double tk_last_kernel_ms(void);
/* Number of kernels this library has launched in this process (instrumentation). */
long long tk_launch_count(void);

/* Release cached device memory (pool trim), pinned scratch and cached result blocks. */
int tk_release(void);

/* Pinned host blocks for results of the host-buffer calls, cached across calls: a caller that
 * allocates its output arrays here (the Python module does for results >= 64 MB) gets the D2H
 * straight into them.  *out = NULL (status TK_OK) when the cache cap (a quarter of host RAM,
 * env TK_HOST_POOL_MB) would be exceeded -- allocate ordinary memory then.  tk_host_free returns
 * the block to the cache (TK_EARG for a pointer that is not a live block). */
int tk_host_alloc(size_t bytes, void** out);
int tk_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* TK_B200_H */
