// Shared device helpers for the PAQIF B200 kernels (sm_100a, fp64).
//
// Arithmetic policy.  EXACT=true reproduces the reference's rounding bit for
// bit: numba compiles paqif/_kernels.py without FMA contraction and with IEEE
// division, so every product and sum below goes through the
// explicit round-to-nearest intrinsics, which nvcc never contracts.
// EXACT=false lets products fuse into DFMA and replaces divisions by the
// level determinant with one reciprocal: same fp64 precision, <= a few ulp
// per operation, used where parity is judged at a tolerance.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define PAQIF_TINY 1e-300

namespace paqif {

template <bool EXACT>
struct Arith;

template <>
struct Arith<true> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  // a*b - c*d, reference order: (a*b) - (c*d)
  static __device__ __forceinline__ double det2(double a, double b, double c, double d) {
    return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
  }
  // acc - (w1*z1 + w2*z2)
  static __device__ __forceinline__ double rank2(double acc, double w1, double z1, double w2,
                                                 double z2) {
    return __dadd_rn(acc, -__dadd_rn(__dmul_rn(w1, z1), __dmul_rn(w2, z2)));
  }
  // acc - z*x
  static __device__ __forceinline__ double axpy_neg(double acc, double z, double x) {
    return __dsub_rn(acc, __dmul_rn(z, x));
  }
  // acc + z*x
  static __device__ __forceinline__ double axpy(double acc, double z, double x) {
    return __dadd_rn(acc, __dmul_rn(z, x));
  }
};

template <>
struct Arith<false> {
  static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double det2(double a, double b, double c, double d) {
    // keep the breakdown test's determinant unfused so marginal decisions
    // match the exact path as closely as the inputs allow
    return __dsub_rn(__dmul_rn(a, b), __dmul_rn(c, d));
  }
  static __device__ __forceinline__ double rank2(double acc, double w1, double z1, double w2,
                                                 double z2) {
    return fma(-w2, z2, fma(-w1, z1, acc));
  }
  static __device__ __forceinline__ double axpy_neg(double acc, double z, double x) {
    return fma(-z, x, acc);
  }
  static __device__ __forceinline__ double axpy(double acc, double z, double x) {
    return fma(z, x, acc);
  }
};

__device__ __forceinline__ double shfl(double v, int src, unsigned mask = 0xffffffffu) {
  return __shfl_sync(mask, v, src);
}

__device__ __forceinline__ double warp_max(double v) {
  // NaN-propagating max (numpy max semantics)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = ((v != v) | (w != w)) ? __longlong_as_double(0x7ff8000000000000ll) : (w > v ? w : v);
  }
  return v;
}

__device__ __forceinline__ int imod(int a, int m) {
  int r = a % m;
  return r < 0 ? r + m : r;
}

}  // namespace paqif
