// Device helpers shared by the EHL Newton-step kernels (line and point
// contact): limiters, guarded ratios, numpy-semantics min/max, block
// reductions and the register-tiled Toeplitz convolution.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace paqif {

constexpr double kDensA = 0.59e9;
constexpr double kDensB = 1.34;
constexpr double kRatioGuard = 1e-30;
constexpr double kSwitch = 0.6;

// ---------------------------------------------------------------- limiters
// tvdcd.limiter_psi / limiter_weight_plus (tvdcd.py:207-235)
__device__ __forceinline__ double np_maximum(double a, double b) {
  return ((a >= b) | (a != a)) ? a : b;
}
__device__ __forceinline__ double np_minimum(double a, double b) {
  return ((a <= b) | (a != a)) ? a : b;
}
static __device__ double limiter_psi(double r, int name, double kappa) {
  switch (name) {
    case 1:  // none
      return ((1.0 + kappa) * r + (1.0 - kappa)) / 2.0;
    case 2:  // van-albada
      return r > 0.0 ? (r * r + r) / (1.0 + r * r) : 0.0;
    case 3:  // minmod
      return np_maximum(0.0, np_minimum(r, 1.0));
    case 4:  // koren
      return np_maximum(0.0, np_minimum(np_minimum(2.0 * r, (1.0 + 2.0 * r) / 3.0), 2.0));
    default: {  // kappa
      const double lin = ((1.0 + kappa) * r + (1.0 - kappa)) / 2.0;
      return np_maximum(0.0, np_minimum(np_minimum(2.0 * r, lin), 2.0));
    }
  }
}
__device__ __forceinline__ double limiter_wplus(double r, int name, double kappa) {
  const double psi = limiter_psi(r, name, kappa);
  const double safe = fabs(r) > kRatioGuard ? r : (r >= 0.0 ? kRatioGuard : -kRatioGuard);
  return r > 0.0 ? psi / safe : 0.0;
}
// sweeps._guarded_ratio with a data scale (sweeps.py:47-56)
__device__ __forceinline__ double gratio(double num, double den, double floor_) {
  return fabs(den) > floor_ ? num / den : 0.0;
}

// ---------------------------------------------------------------- block helpers
static __device__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
  __syncthreads();
  return r;
}
// NaN-propagating max (numpy max)
static __device__ double block_nanmax(double v, double* red) {
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = ((v != v) | (w != w)) ? qnan : (w > v ? w : v);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    const double x = red[w];
    r = ((r != r) | (x != x)) ? qnan : (x > r ? x : r);
  }
  __syncthreads();
  return r;
}
static __device__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red[w];
  __syncthreads();
  return r;
}

// deformation: def[i] = sign * sum_j u[j] * ext[n + i - j], i = 0..n
// (np.convolve(u, ext)[n:2n+1]); 4 consecutive outputs per thread
static __device__ void toeplitz_conv(const double* su, const double* ext, int n, double sign,
                              double* out) {
  const int N = n + 1;
  for (int i0 = 4 * threadIdx.x; i0 < N; i0 += 4 * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    // e_r = ext[n + i0 + r - j]; slide as j increases
    const double* eb = ext + n + i0;
    double e0 = eb[0], e1 = eb[1], e2 = eb[2], e3 = eb[3];
    for (int j = 0; j < N; ++j) {
      const double uj = su[j];
      a0 = fma(uj, e0, a0);
      a1 = fma(uj, e1, a1);
      a2 = fma(uj, e2, a2);
      a3 = fma(uj, e3, a3);
      e3 = e2;
      e2 = e1;
      e1 = e0;
      e0 = eb[-j - 1];
    }
    out[i0] = sign * a0;
    if (i0 + 1 < N) out[i0 + 1] = sign * a1;
    if (i0 + 2 < N) out[i0 + 2] = sign * a2;
    if (i0 + 3 < N) out[i0 + 3] = sign * a3;
  }
}


}  // namespace paqif
