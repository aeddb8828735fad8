// tk_common.cuh -- shared device helpers for the sm_100a kernels of tk-b200.
//
// Everything on the TTV/dot/matvec path is an FP64, HBM-bandwidth-bound stream
// (<= 0.125 FLOP/B), so the helpers here are about moving bytes: 1-D TMA bulk
// copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier, relaxed
// GPU-scope loads/stores for the tile prefix scan, and a streaming L2
// policy for data that is read exactly once.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tk {

constexpr int kMaxOrder = 16;              // largest tensor order the GPU path accepts
constexpr int kMaxKeep = kMaxOrder - 1;    // kept (output) modes
constexpr int kMaxPeers = 8;               // output copies of a sharded dense result (GPUs per node)

// device-side status bits, collected in Counters::flags
enum : unsigned int {
  kFlagIndex = 1u,     // contracted-mode index outside x -> DimensionError
  kFlagUnsorted = 2u,  // kept-mode keys not non-decreasing -> take the sort path
  kFlagKeptOob = 4u,   // kept-mode index outside its dimension (garbage input)
  kFlagStall = 8u,     // a cross-CTA wait gave up (watchdog): the call fails instead of hanging
};
constexpr unsigned int kSpinLimit = 1u << 25;  // polls (>= ~64 ns each) before a wait gives up

// Per-call scalars written by the kernels and read back by the host once.
struct Counters {
  unsigned long long groups;     // number of output groups (before zero elimination)
  unsigned long long zeros;      // groups whose serial sum is exactly 0.0
  unsigned int flags;            // kFlag* bits
  unsigned int tile_ticket;      // watchdog report: the tile whose wait gave up
  unsigned int grab_ticket;      // watchdog report: the wait site that gave up
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier + 1-D bulk async copy (TMA engine, no tensor map needed) ----------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "TK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TK_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---- relaxed GPU-scope accesses for the look-back status words ------------------------------
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- per-tile status words of the tile kernel's prefix scan -------------------------------------
// status word: [63:62] = 0 invalid, 1 aggregate, 2 inclusive prefix; [61:0] = count.
constexpr unsigned long long kStAgg = 1ull << 62;
constexpr unsigned long long kStPre = 2ull << 62;
constexpr unsigned long long kStVal = (1ull << 62) - 1;

}  // namespace tk
