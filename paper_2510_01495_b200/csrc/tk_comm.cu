// tk_comm.cu -- the multi-GPU data plane of the sharded TTV inside the C ABI (NCCL).
//
// nonzeros are sharded across one process per GPU at kept-key changes, so every
// rank's result is a canonical slice and the only exchanges are (a) an all-gather of per-rank
// result counts (global offsets), (b) the optional gather of the sparse slices to one root, (c)
// for the dense result (config 4) the exchange of CUDA IPC handles once plus a stream-ordered
// barrier after the kernels' peer stores, or the all-reduce of zero-padded partials (baseline).
// All of it runs here over NCCL on the caller's stream; torch.distributed at most broadcasts the
// 128-byte NCCL unique id (bootstrap).
//
// NCCL is bound at run time with dlopen: the process may already hold PyTorch's NCCL
// (RTLD_NOLOAD finds it) -- two NCCL copies in one process must be avoided -- or the caller names
// the library (tk_nccl_load).  Only the handful of entry points below are used.
#include <dlfcn.h>

#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "tk_host.h"

namespace tk {
namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

std::mutex g_api_mu;
NcclApi g_api;

int bind_api(const char* path) {
  std::lock_guard<std::mutex> lk(g_api_mu);
  if (g_api.so) return TK_OK;
  void* so = nullptr;
  if (path && *path) so = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (PyTorch)
  if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!so) return fail(TK_ENCCL, std::string("NCCL: cannot load libnccl.so.2: ") + dlerror());
  NcclApi a;
  a.so = so;
  bool ok = true;
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(so, name));
    ok = ok && fn != nullptr;
  };
  sym(a.GetUniqueId, "ncclGetUniqueId");
  sym(a.CommInitRank, "ncclCommInitRank");
  sym(a.CommDestroy, "ncclCommDestroy");
  sym(a.AllGather, "ncclAllGather");
  sym(a.AllReduce, "ncclAllReduce");
  sym(a.Send, "ncclSend");
  sym(a.Recv, "ncclRecv");
  sym(a.GroupStart, "ncclGroupStart");
  sym(a.GroupEnd, "ncclGroupEnd");
  sym(a.GetErrorString, "ncclGetErrorString");
  sym(a.GetVersion, "ncclGetVersion");
  if (!ok) return fail(TK_ENCCL, "NCCL: a required entry point is missing from the loaded library");
  g_api = a;
  return TK_OK;
}

#define TK_NCCL(expr)                                                                               \
  do {                                                                                              \
    ncclResult_t tk_r_ = (expr);                                                                    \
    if (tk_r_ != ncclSuccess)                                                                       \
      return fail(TK_ENCCL, std::string("NCCL error: ") + g_api.GetErrorString(tk_r_) + " (" #expr ")"); \
  } while (0)

constexpr int kSlots = 4;  // count all-gathers in flight (the bench overlaps step i's with step i+1)

// One rank's communicator plus the small device / pinned buffers its collectives use.
struct Comm {
  ncclComm_t nc = nullptr;
  int nranks = 0, rank = 0, device = 0;
  cudaStream_t cs = nullptr;            // the comm's own stream (count gathers run beside the TTV)
  int64_t* d_cnt = nullptr;             // kSlots x (1 + nranks) int64: send slot + gathered counts
  int64_t* h_cnt = nullptr;             // pinned: kSlots x (1 + nranks)
  cudaEvent_t ev[kSlots] = {};
  unsigned int next = 0;
  int* d_flag = nullptr;                // barrier operand
};

}  // namespace
}  // namespace tk

using namespace tk;

extern "C" {

int tk_nccl_load(const char* path) { return bind_api(path); }

int tk_nccl_version(int* version) {
  if (!version) return fail(TK_EARG, "nccl_version: null argument");
  if (int rc = bind_api(nullptr)) return rc;
  TK_NCCL(g_api.GetVersion(version));
  return TK_OK;
}

int tk_nccl_get_unique_id(void* id128) {
  if (!id128) return fail(TK_EARG, "nccl_get_unique_id: null argument");
  if (int rc = bind_api(nullptr)) return rc;
  ncclUniqueId id;
  TK_NCCL(g_api.GetUniqueId(&id));
  memcpy(id128, &id, sizeof id);
  return TK_OK;
}

int tk_nccl_comm_init(const void* id128, int32_t nranks, int32_t rank, void** comm) {
  if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return fail(TK_EARG, "nccl_comm_init: bad arguments");
  if (int rc = bind_api(nullptr)) return rc;
  *comm = nullptr;
  Comm* c = new Comm();
  struct Guard {
    Comm*& c;
    ~Guard() {
      if (c) {
        if (c->nc) g_api.CommDestroy(c->nc);
        delete c;
      }
    }
  } guard{c};
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  TK_CUDA(cudaGetDevice(&c->device));
  c->nranks = nranks;
  c->rank = rank;
  TK_NCCL(g_api.CommInitRank(&c->nc, nranks, id, rank));
  TK_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  TK_CUDA(cudaMalloc(&c->d_cnt, sizeof(int64_t) * kSlots * (1 + nranks)));
  TK_CUDA(cudaMallocHost(&c->h_cnt, sizeof(int64_t) * kSlots * (1 + nranks)));
  TK_CUDA(cudaMalloc(&c->d_flag, 16));
  TK_CUDA(cudaMemset(c->d_flag, 0, 16));
  for (int i = 0; i < kSlots; ++i) TK_CUDA(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  *comm = c;
  c = nullptr;  // owned by the caller now
  return TK_OK;
}

int tk_nccl_comm_free(void* comm) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c) return fail(TK_EARG, "nccl_comm_free: null communicator");
  cudaStreamSynchronize(c->cs);
  if (c->nc) g_api.CommDestroy(c->nc);
  for (int i = 0; i < kSlots; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->cs) cudaStreamDestroy(c->cs);
  cudaFree(c->d_cnt);
  cudaFreeHost(c->h_cnt);
  cudaFree(c->d_flag);
  delete c;
  return TK_OK;
}

int tk_nccl_rank(void* comm, int32_t* rank, int32_t* nranks) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !rank || !nranks) return fail(TK_EARG, "nccl_rank: null argument");
  *rank = c->rank;
  *nranks = c->nranks;
  return TK_OK;
}

// (a) per-rank result counts -> global offsets.  Start: the host count goes up, the all-gather
// runs on the comm's own stream after `stream` (the TTV that produced the count) and the gathered
// counts come back to pinned memory -- nothing blocks; returns a ticket.  Wait: the ticket's
// counts, rank order.
int tk_nccl_counts_start(void* comm, int64_t count, void* stream, int32_t* ticket) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !ticket) return fail(TK_EARG, "nccl_counts_start: bad arguments");
  const unsigned int s = c->next++ % kSlots;
  const int w = 1 + c->nranks;
  TK_CUDA(cudaEventSynchronize(c->ev[s]));  // the slot's previous gather has been read
  c->h_cnt[s * w] = count;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TK_CUDA(cudaEventRecord(c->ev[s], st));
  TK_CUDA(cudaStreamWaitEvent(c->cs, c->ev[s], 0));
  TK_CUDA(cudaMemcpyAsync(c->d_cnt + s * w, c->h_cnt + s * w, 8, cudaMemcpyHostToDevice, c->cs));
  TK_NCCL(g_api.AllGather(c->d_cnt + s * w, c->d_cnt + s * w + 1, 1, ncclInt64, c->nc, c->cs));
  TK_CUDA(cudaMemcpyAsync(c->h_cnt + s * w + 1, c->d_cnt + s * w + 1, 8 * c->nranks, cudaMemcpyDeviceToHost, c->cs));
  TK_CUDA(cudaEventRecord(c->ev[s], c->cs));
  *ticket = (int32_t)s;
  return TK_OK;
}

int tk_nccl_counts_wait(void* comm, int32_t ticket, int64_t* counts) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !counts || ticket < 0 || ticket >= kSlots) return fail(TK_EARG, "nccl_counts_wait: bad arguments");
  TK_CUDA(cudaEventSynchronize(c->ev[ticket]));
  memcpy(counts, c->h_cnt + ticket * (1 + c->nranks) + 1, 8 * (size_t)c->nranks);
  return TK_OK;
}

// (b) gather of the ranks' sparse slices to `root` (the canonical result there, rank order): the
// root receives rank r's counts[r] rows at offset sum(counts[:r]); grouped point-to-point on the
// caller's stream.  subs row-major (u, nk) int64, vals (u); dst_* used on the root only.
int tk_nccl_gather_rows(void* comm, int32_t root, const int64_t* subs, const double* vals, int32_t nk,
                        const int64_t* counts, int64_t* dst_subs, double* dst_vals, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !counts || nk < 1 || root < 0 || root >= c->nranks) return fail(TK_EARG, "nccl_gather_rows: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t mine = counts[c->rank];
  if (c->rank == root) {
    if (!dst_subs || !dst_vals) return fail(TK_EARG, "nccl_gather_rows: root needs destination buffers");
    int64_t off = 0;
    TK_NCCL(g_api.GroupStart());
    for (int r = 0; r < c->nranks; ++r) {
      const int64_t n = counts[r];
      if (n > 0 && r != root) {
        g_api.Recv(dst_subs + off * nk, (size_t)(n * nk), ncclInt64, r, c->nc, st);
        g_api.Recv(dst_vals + off, (size_t)n, ncclFloat64, r, c->nc, st);
      }
      off += n;
    }
    TK_NCCL(g_api.GroupEnd());
    int64_t my_off = 0;
    for (int r = 0; r < root; ++r) my_off += counts[r];
    if (mine > 0 && dst_subs + my_off * nk != subs) {
      TK_CUDA(cudaMemcpyAsync(dst_subs + my_off * nk, subs, 8 * (size_t)(mine * nk), cudaMemcpyDeviceToDevice, st));
      TK_CUDA(cudaMemcpyAsync(dst_vals + my_off, vals, 8 * (size_t)mine, cudaMemcpyDeviceToDevice, st));
    }
  } else if (mine > 0) {
    TK_NCCL(g_api.GroupStart());
    g_api.Send(subs, (size_t)(mine * nk), ncclInt64, root, c->nc, st);
    g_api.Send(vals, (size_t)mine, ncclFloat64, root, c->nc, st);
    TK_NCCL(g_api.GroupEnd());
  }
  return TK_OK;
}

// (c1) every rank's `nbytes` of host data to every rank (rank order), e.g. the 64-byte CUDA IPC
// handles of the dense result's peer-store merge; synchronous, once per merge set-up.
int tk_nccl_allgather_bytes(void* comm, const void* host_src, void* host_dst, int64_t nbytes) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !host_src || !host_dst || nbytes <= 0) return fail(TK_EARG, "nccl_allgather_bytes: bad arguments");
  DevBuf b;
  if (int rc = b.alloc((size_t)nbytes * (1 + c->nranks), c->cs)) return rc;
  char* d = b.as<char>();
  TK_CUDA(cudaMemcpyAsync(d, host_src, (size_t)nbytes, cudaMemcpyHostToDevice, c->cs));
  TK_NCCL(g_api.AllGather(d, d + nbytes, (size_t)nbytes, ncclUint8, c->nc, c->cs));
  TK_CUDA(cudaMemcpyAsync(host_dst, d + nbytes, (size_t)nbytes * c->nranks, cudaMemcpyDeviceToHost, c->cs));
  TK_CUDA(cudaStreamSynchronize(c->cs));
  return TK_OK;
}

// (c2) stream-ordered barrier: a one-element all-reduce enqueued on `stream`; it completes on a
// rank only after every rank has reached it on its own stream -- i.e. after every rank's
// preceding kernels (and their NVLink peer stores) are done.
int tk_nccl_barrier(void* comm, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c) return fail(TK_EARG, "nccl_barrier: null communicator");
  TK_NCCL(g_api.AllReduce(c->d_flag, c->d_flag, 1, ncclInt32, ncclSum, c->nc, static_cast<cudaStream_t>(stream)));
  return TK_OK;
}

// (c3) the baseline dense merge: in-place sum of zero-padded partials (disjoint supports: exact).
int tk_nccl_allreduce_sum_f64(void* comm, double* buf, int64_t n, void* stream) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || (!buf && n > 0) || n < 0) return fail(TK_EARG, "nccl_allreduce: bad arguments");
  if (n == 0) return TK_OK;
  TK_NCCL(g_api.AllReduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, c->nc, static_cast<cudaStream_t>(stream)));
  return TK_OK;
}

}  // extern "C"
