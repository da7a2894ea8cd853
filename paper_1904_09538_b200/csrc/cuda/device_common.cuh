// Device helpers shared by every kernel translation unit.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ps {

// ---------------------------------------------------------------------------
// Shared-memory accesses the compiler must not hoist, fold or drop
// (lmem_shuffle copies a loop-invariant slot, uipick.cpp:399-400; the
// overlap kernel's shuffle result is dead, uipick.cpp:457-459).
__device__ __forceinline__ float lds_volatile(const float* p) {
  float v;
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_volatile(float* p, float v) {
  unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
// 32-byte read-only global load (sm_100 LDG.E.ENL2.256); p must be 32-byte aligned.
struct f8 {
  float v[8];
};
__device__ __forceinline__ f8 ldg256(const float* p) {
  f8 r;
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
        "=f"(r.v[6]), "=f"(r.v[7])
      : "l"(p));
  return r;
}
__device__ __forceinline__ void bar_sync() { asm volatile("bar.sync 0;" ::: "memory"); }

template <typename T>
__device__ __forceinline__ T fma_t(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_t<float>(float a, float b, float c) {
  return __fmaf_rn(a, b, c);
}
template <>
__device__ __forceinline__ double fma_t<double>(double a, double b, double c) {
  return __fma_rn(a, b, c);
}
template <typename T>
__device__ __forceinline__ T add_t(T a, T b);
template <>
__device__ __forceinline__ float add_t<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_t<double>(double a, double b) { return __dadd_rn(a, b); }

}  // namespace ps
