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

// One row of the change system of a line (assemble_line_system,
// ehl/sweeps.py:157-267): the 5 band entries e[0..4] (offsets -2..2),
// oriented for a positive diagonal, with the bad-row fallback to the
// first-order face sensitivities.  ex/ey: face mobilities as the reference
// passes them (already scaled by the transverse spacing for the point
// contact; ey = 0 for the line contact); hy: h (point) or 1 (line).
// jac: 0 scheme, 1 first-order, 2 diagonal.
__device__ __forceinline__ void line_row_entries(double rw, double rc, double re, double ex_p,
                                                 double ex_m, double ey_p, double ey_m,
                                                 double phi_p, double phi_m, double h, double hy,
                                                 bool weighted, int jac, double ks0, double ks1,
                                                 double* e) {
  if (jac != 0) {
    phi_p = 0.0;
    phi_m = 0.0;
  }
  const double a_p = 1.0 - 0.5 * phi_p, b_p = 0.5 * phi_p;
  const double a_m = 1.0 - 0.5 * phi_m, b_m = 0.5 * phi_m;
  double c_m2, c_m1, c_0, c_p1, c_p2;
  if (jac == 2) {
    c_m2 = 0.0; c_m1 = 0.0; c_p1 = 0.0; c_p2 = 0.0;
    c_0 = -hy * rc * fabs(ks0);
  } else {
    c_m2 = hy * (a_m * rw * ks1);
    c_m1 = -hy * (a_p * rc * ks1 - a_m * rw * ks0 - b_m * rc * ks1);
    c_0 = -hy * (a_p * rc * ks0 + b_p * re * ks1 - a_m * rw * ks1 - b_m * rc * ks0);
    c_p1 = -hy * (a_p * rc * ks1 + b_p * re * ks0 - b_m * rc * ks1);
    c_p2 = -hy * (b_p * re * ks1);
  }
  const double ey_sum = ey_p + ey_m;
  double p_m2, p_m1, p_0, p_p1, p_p2;
  if (weighted) {
    p_m2 = -0.25 * ex_m / h;
    p_m1 = (1.25 * ex_m + 0.25 * ex_p) / h + 0.25 * ey_sum / h;
    p_0 = -1.25 * (ex_p + ex_m + ey_sum) / h;
    p_p1 = (1.25 * ex_p + 0.25 * ex_m) / h + 0.25 * ey_sum / h;
    p_p2 = -0.25 * ex_p / h;
  } else {
    p_m2 = 0.0;
    p_m1 = ex_m / h;
    p_0 = -(ex_p + ex_m + ey_sum) / h;
    p_p1 = ex_p / h;
    p_p2 = 0.0;
  }
  e[0] = -(c_m2 + p_m2);
  e[1] = -(c_m1 + p_m1);
  e[2] = -(c_0 + p_0);
  e[3] = -(c_p1 + p_p1);
  e[4] = -(c_p2 + p_p2);
  const double off_mag = fabs(e[0]) + fabs(e[1]) + fabs(e[3]) + fabs(e[4]);
  const double floor_ = 0.05 * hy * fabs(rc) * fabs(ks0);
  if (fabs(e[2]) < np_maximum(0.2 * off_mag, floor_)) {
    const double fo_m2 = hy * rw * ks1;
    const double fo_m1 = -hy * (rc * ks1 - rw * ks0);
    const double fo_0 = -hy * (rc * ks0 - rw * ks1);
    const double fo_p1 = -hy * rc * ks1;
    e[0] = -(fo_m2 + p_m2);
    e[1] = -(fo_m1 + p_m1);
    e[2] = -(fo_0 + p_0);
    e[3] = -(fo_p1 + p_p1);
    e[4] = -p_p2;
  }
}

// The mirrored line kernel ext[k] = table[|k - n|] (k = 0..2n; zero on 8
// guard entries each side) in an 8-phase shared-memory layout,
//   ext[k] at ext4[((k + 8) & 7) * Q + ((k + 8) >> 3)],  Q = ext4_q(n),
// so that threads holding 8 consecutive outputs each read consecutive words
// at every step of the convolution (no bank conflicts).
__host__ __device__ inline int ext4_q(int n) { return (2 * n + 17 + 7) / 8; }
__host__ __device__ inline int ext4_doubles(int n) { return 8 * ext4_q(n); }
__device__ __forceinline__ void ext4_build(const double* __restrict__ table, int n, double* ext4) {
  const int Q = ext4_q(n);
  for (int idx = threadIdx.x; idx < 8 * Q; idx += blockDim.x) {
    const int ph = idx / Q, q = idx - ph * Q;
    const int k = 8 * q + ph - 8;
    ext4[idx] = (k >= 0 && k <= 2 * n) ? table[k >= n ? k - n : n - k] : 0.0;
  }
}
__device__ __forceinline__ double ext4_at(const double* ext4, int Q, int k) {
  const int kk = k + 8;
  return ext4[(kk & 7) * Q + (kk >> 3)];
}

// deformation: def[i] = sign * sum_j u[j] * ext[n + i - j], i = 0..n
// (np.convolve(u, ext)[n:2n+1]), ext in the 8-phase layout.  8 consecutive
// outputs per thread sliding along the kernel: per 8 steps of j eight
// conflict-free kernel loads, eight broadcast u loads, 64 DFMA.  The j range
// is split into S segments so that the 8-output groups fill the block; the
// segments are added in a fixed order (one barrier each).  The N mod 8
// outputs past the last full group are warp dot products.  All threads of
// the CTA call.
static __device__ void toeplitz_conv(const double* su, const double* ext4, int n, double sign,
                                     double* out) {
  const int N = n + 1, T = blockDim.x, Q = ext4_q(n);
  const int G = N / 8;
  int S = G > 0 ? T / G : 1;
  if (S < 1) S = 1;
  if (S > 8) S = 8;
  const int seg_len = (N + S - 1) / S;
  auto group = [&](int g, int j0, int j1, double* a) {
    const int i0 = 8 * g;
    // e[r] = ext[n + i0 + r - j]; the entry entering at step j is
    // ext[n - 1 - j + i0]
    double e[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      e[r] = ext4_at(ext4, Q, n + i0 + r - j0);
      a[r] = 0.0;
    }
    auto step = [&](double uj, double enew) {
#pragma unroll
      for (int r = 0; r < 8; ++r) a[r] = fma(uj, e[r], a[r]);
#pragma unroll
      for (int r = 7; r > 0; --r) e[r] = e[r - 1];
      e[0] = enew;
    };
    int j = j0;
    for (; j < j1 && ((n + 7 - j) & 7) != 7; ++j) step(su[j], ext4_at(ext4, Q, n - 1 - j + i0));
    // blocks of 8 steps: entering entries of phases 7..0 at q0, then q0 - 1 ...
    const double* p = ext4 + ((n + 7 - j) >> 3) + g;
    for (; j + 8 <= j1; j += 8, --p) {
      double f[8], uu[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        f[t] = p[(7 - t) * Q];
        uu[t] = su[j + t];
      }
#pragma unroll
      for (int t = 0; t < 8; ++t) step(uu[t], f[t]);
    }
    for (; j < j1; ++j) step(su[j], ext4_at(ext4, Q, n - 1 - j + i0));
  };
  const int t = threadIdx.x;
  const int g = G > 0 ? t % G : 0, sg = G > 0 ? t / G : S;
  double a[8];
  const bool mine = sg < S && g < G;
  if (mine) {
    const int j0 = sg * seg_len, j1 = j0 + seg_len < N ? j0 + seg_len : N;
    group(g, j0, j1, a);
  }
  for (int q = 0; q < S; ++q) {  // fixed order: segment 0, 1, ...
    if (mine && sg == q)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double v = q == 0 ? a[r] : out[8 * g + r] + a[r];
        out[8 * g + r] = q == S - 1 ? sign * v : v;
      }
    __syncthreads();
  }
  if (G > T) {  // more groups than threads (very long lines): remaining groups
    for (int g2 = T + t; g2 < G; g2 += T) {
      double b[8];
      group(g2, 0, N, b);
#pragma unroll
      for (int r = 0; r < 8; ++r) out[8 * g2 + r] = sign * b[r];
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = 8 * G + warp; i < N; i += T >> 5) {
    double acc = 0.0;
    for (int j = lane; j < N; j += 32) acc = fma(su[j], ext4_at(ext4, Q, n + i - j), acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) out[i] = sign * acc;
  }
}


}  // namespace paqif
