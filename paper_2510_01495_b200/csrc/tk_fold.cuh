// tk_fold.cuh -- the serial in-group fold and the named-barrier helper shared by the tile kernel.
//
// Every output group of the sparse-result TTV is folded exactly as the reference does it
// (_ckernels.pyx:274-294): acc = w[first]; acc = acc + w[next] ... in ascending row order with
// round-to-nearest adds and no FMA contraction, so values are bit-identical to the reference.
#pragma once

#include "tk_ttv_kernels.cuh"

namespace tk {

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// acc, then s_a[j .. end) added in order (independent loads, dependent adds).
__device__ __forceinline__ double fold_run(const double* s_a, int j, int end, double acc) {
#ifdef TK_DIAG_NOFOLD  // diagnostics only: wrong values, measures the cost of the serial folds
  return acc + (end > j ? s_a[end - 1] : 0.0);
#endif
  // 16-byte shared loads: half the shared-memory wavefronts of a serial fold
  if ((j & 1) && j < end) acc = __dadd_rn(acc, s_a[j++]);
  for (; j + 4 <= end; j += 4) {
    const double2 v01 = *reinterpret_cast<const double2*>(s_a + j);
    const double2 v23 = *reinterpret_cast<const double2*>(s_a + j + 2);
    acc = __dadd_rn(acc, v01.x);
    acc = __dadd_rn(acc, v01.y);
    acc = __dadd_rn(acc, v23.x);
    acc = __dadd_rn(acc, v23.y);
  }
  if (j + 2 <= end) {
    const double2 v01 = *reinterpret_cast<const double2*>(s_a + j);
    acc = __dadd_rn(acc, v01.x);
    acc = __dadd_rn(acc, v01.y);
    j += 2;
  }
  if (j < end) acc = __dadd_rn(acc, s_a[j]);
  return acc;
}

}  // namespace tk
