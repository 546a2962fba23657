// Banded line solve used by the EHL step kernels: the CTA has assembled a
// pentadiagonal system (diagonal-major, beta = 2, padded even order) and its
// right side in global scratch; warp 0 factors it with the AQIF engine (W
// solve fused) and runs the full outside-in Z solve.  All threads of the
// CTA call; returns nonzero on a breakdown (FactorizationBreakdownError).
#pragma once
#include "aqif_warp.cuh"
#include "zsolve.cuh"

namespace paqif {

constexpr int kLineBeta = 2;

struct LineSysPol {
  static constexpr bool kFuseW = true;
  static constexpr bool kResidual = false;
  static constexpr bool kFastDiv = false;  // branch-free divisions, checked repeat
  static constexpr bool kLazyBreakdown = false;  // breakdown found after the loop
  static constexpr bool kRecordW = false;
  using PL = PivotLayout<kLineBeta>;
  const double* band;
  const double* rhs;
  double* zs;
  int n;
  __device__ __forceinline__ const double* raw_ptr(int i, int d) const {
    return band + (size_t)(d + kLineBeta) * n + i;
  }
  __device__ __forceinline__ double raw(int i, int d) const { return *raw_ptr(i, d); }
  __device__ __forceinline__ const uint64_t* pin_ptr(int) const { return nullptr; }
  __device__ __forceinline__ bool pinned(int) const { return false; }
  __device__ __forceinline__ const double* frhs_ptr(int i) const { return rhs + i; }
  __device__ __forceinline__ double frhs(int i) const { return rhs[i]; }
  __device__ __forceinline__ void on_level(int k, const double* pb, int gl, int G) {
    double2* dst = reinterpret_cast<double2*>(zs + (size_t)k * PL::kSize);
    const double2* src = reinterpret_cast<const double2*>(pb);
    for (int idx = gl; idx < PL::kSize / 2; idx += G) dst[idx] = src[idx];
  }
  __device__ __forceinline__ void on_w(int, int, double, double) {}
  __device__ __forceinline__ void on_resid(int, int, double) {}
};

// scratch: band (5 x n_sys) | rhs (n_sys) | x (n_sys) | zs ((n_sys/2+1) x kSize)
__host__ __device__ inline size_t line_scratch_doubles(int n_sys) {
  return (size_t)(2 * kLineBeta + 1) * n_sys + 2 * (size_t)n_sys +
         (size_t)(n_sys / 2 + 1) * PivotLayout<kLineBeta>::kSize + 32;
}

template <bool EXACT>
__device__ int solve_line_system(double* scratch, int n_sys, EngineSmem<kLineBeta>& eng,
                                 double* ring, int* flag_smem) {
  double* band = scratch;
  double* rhs = band + (size_t)(2 * kLineBeta + 1) * n_sys;
  double* x = rhs + n_sys;
  double* zs = x + n_sys;
  __syncthreads();
  if (threadIdx.x < 32) {
    constexpr int G = Group<kLineBeta>::G;
    const int lane = threadIdx.x;
    const bool alive = lane < G;
    LineSysPol pol{band, rhs, zs, n_sys};
    int fst = aqif_factor_group<kLineBeta, EXACT>(pol, n_sys, 1e-14, eng, lane % G, alive);
    fst = __shfl_sync(0xffffffffu, fst, 0);
    int zst = 0;
    if (fst == 0) {
      zst = zsolve_group<kLineBeta, EXACT, true>(zs, n_sys, x, ring, lane % G, alive);
      zst = __shfl_sync(0xffffffffu, zst, 0);
    }
    if (lane == 0) *flag_smem = (fst || zst) ? 1 : 0;
  }
  __syncthreads();
  const int st = *flag_smem;
  __syncthreads();
  return st;
}

__device__ __forceinline__ const double* line_solution(const double* scratch, int n_sys) {
  return scratch + (size_t)(2 * kLineBeta + 1) * n_sys + n_sys;
}

}  // namespace paqif
