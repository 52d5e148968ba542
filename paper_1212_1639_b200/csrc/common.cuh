// Shared device/host helpers for the parsmc-b200 engine (sm_100a).
//
// Parity-critical arithmetic follows the reference's numpy evaluation order
// with no fused multiply-add: the whole library is compiled with
// -fmad=false, and the places that *want* FMA (polynomial tables, Philox is
// integer) call fma() explicitly.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define PF_HD __host__ __device__ __forceinline__
#define PF_D __device__ __forceinline__

namespace pf {

// Status codes of the C-ABI (include/parsmc_b200.h); map 1:1 onto the
// reference's exception classes (errors.py:4-35).
enum Code : int32_t {
  OK = 0,
  ALL_WEIGHTS_ZERO = 1,   // AllWeightsZeroError(step)   filtering.py:294-296, prefix_sum.py:97-100
  NON_FINITE_WEIGHT = 2,  // NonFiniteWeightError         core.py:26-27, filtering.py:130-131
  NOT_POWER_OF_TWO = 3,   // NotPowerOfTwoError           core.py:16-18
  VALUE_ERROR = 4,        // ValueError                   filtering.py:205-208
  CUDA_ERROR = 5,
  OUT_OF_MEMORY = 6,
  NOT_IMPLEMENTED = 7,
};

PF_HD int pf_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __popc(x);
#else
  return __builtin_popcount(x);
#endif
}
PF_HD bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
PF_HD int ilog2(int64_t n) {
  int k = 0;
  while ((int64_t(1) << k) < n) ++k;
  return k;
}

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-stream-serialization attribute may start while its stream
// predecessor is still draining.  pdl_wait() blocks until every prerequisite
// grid has completed and its memory is visible -- it must precede any read
// of a predecessor's output (and any write a predecessor could still read).
// pdl_launch_dependents() lets the next kernel in the stream be scheduled
// early.  Both are no-ops for kernels launched without the attribute.
PF_D void pdl_wait() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
PF_D void pdl_launch_dependents() {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 900
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// numpy's np.max propagates NaN: keep a NaN from either side.
PF_D double nan_max(double a, double b) { return (a > b || a != a) ? a : b; }

// Monotone map of a double onto uint64 (total order for non-NaN values).
PF_HD uint64_t ordered_bits(double v) {
  union { double d; uint64_t u; } c;
  c.d = v;
  return (c.u >> 63) ? ~c.u : (c.u | 0x8000000000000000ull);
}

}  // namespace pf
