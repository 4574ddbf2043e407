// sm100_common.cuh — device helpers shared by the sm_100a translation units
// (hydro_kernels.cu, field_step.cu): shared-memory addressing, mbarrier
// transaction barriers, the TMA descriptor encoder, the team-id parameter
// block, and the reference's minmod (kernels.py:58-60).  Header-only, in an
// anonymous namespace: each translation unit keeps its own copy.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <mutex>

#include "../../include/taskfuse_b200.h"

namespace {

// A team's sub-grid ids by value in the kernel parameters (<= 128 x int32
// = 512 B, __grid_constant__): a team launch needs no host->device copy.
struct TeamIds {
  int32_t id[TF_MAX_TEAM];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// kernels.py:58-60 — product test first, then strict |a|<|b|.  NaN in the
// product fails `<= 0` and NaN in |a| fails `<`, both yielding b, as numpy.
// The product is __dmul_rn: never contracted into a neighbouring FMA.
__device__ __forceinline__ double minmod(double a, double b) {
  return (__dmul_rn(a, b) <= 0.0) ? 0.0 : ((fabs(a) < fabs(b)) ? a : b);
}

// sigma = minmod(w[+e] - base, base - w[-e]) at index b along stride st
// (kernels.py:76-79)
__device__ __forceinline__ double slope(const double* __restrict__ s, int b,
                                        int st) {
  const double base = s[b];
  return minmod(__dsub_rn(s[b + st], base), __dsub_rn(base, s[b - st]));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// -lcuda link dependency); nullptr if unavailable
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault,
                                &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace
