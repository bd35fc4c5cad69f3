// common.cuh -- device helpers shared by the libwlr kernels (CUDA path only; the
// oracle shares nothing with this directory).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define WLR_DEVI __device__ __forceinline__

namespace wlr {

constexpr int kWarp = 32;

// device-side error flags (ctx->d_flags[0]); first writer wins
enum DevFlag : int {
  DF_OK = 0,
  DF_RANK = 2,       // Cholesky of G = X1^T X1 failed      -> WLR_ERANK
  DF_EIG = 3,        // eigensolver budget exhausted        -> WLR_EEIG
  DF_ROWSPD = 4,     // per-row system not SPD              -> WLR_EINTERNAL
  DF_NONFINITE = 5,  // non-finite objective                -> WLR_ENONFINITE
};

WLR_DEVI void raise_flag(int* flags, int code) { atomicCAS(flags, 0, code); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

template <typename T>
WLR_DEVI T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 4-wide vector type per scalar
template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

template <typename T>
WLR_DEVI typename Vec4<T>::type ldg4(const T* p) {
  return __ldg(reinterpret_cast<const typename Vec4<T>::type*>(p));
}
template <>
WLR_DEVI double4 ldg4<double>(const double* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

template <typename V> WLR_DEVI auto vx(const V& v) { return v.x; }

// Programmatic dependent launch (the per-iteration kernel chain): a dependent
// waits for its predecessor grid (completion + memory flush) before touching its outputs; every
// kernel of the chain waits before it exits, so the ordering stays transitive.
WLR_DEVI void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
WLR_DEVI void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

}  // namespace wlr
