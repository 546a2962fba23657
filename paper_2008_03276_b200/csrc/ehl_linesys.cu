// Stand-alone line-system entry points of paqif/ehl/sweeps.py on the GPU:
//   assemble_line_system / splitting_ls4 / splitting_ls5 (sweeps.py:157-267,
//   298-313), robust_line_solve (sweeps.py:270-295: scheme, first-order and
//   diagonal Jacobians until the AQIF factorization succeeds) and
//   reynolds_residual_field (sweeps.py:106-138, line and point contact).
// The fused sweep kernels (ehl_line.cu, ehl_point.cu) use the same device
// functions (line_row_entries, limiter_wplus, gratio, the aqif2 engine);
// these entries expose them for callers that work line by line with the
// reference's arrays.  One CTA per call; [dev] pointers.
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "aqif2.cuh"
#include "capi_util.cuh"
#include "ehl_common.cuh"

extern "C" {
#include "../../include/paqif_ehl.h"
}

namespace paqif {

constexpr int kLsThreads = 256;

// frozen face weights phi+ / phi- of the interior nodes i = 1..n-1
// (sweeps._faces, sweeps.py:88-103): guarded ratios with the floor
// 1e-12 max(max|q|, guard), as the fused kernels compute them
__device__ void line_faces(const double* __restrict__ q, int n, int limiter, double kappa,
                           double* php, double* phm, double* red) {
  double qmax = 0.0;
  for (int i = threadIdx.x; i <= n; i += blockDim.x) qmax = fmax(qmax, fabs(q[i]));
  const double gfloor = 1e-12 * fmax(block_max(qmax, red), kRatioGuard);
  for (int i = 1 + threadIdx.x; i < n; i += blockDim.x) {
    const double dqi = q[i + 1] - q[i], dqm = q[i] - q[i - 1];
    php[i] = limiter_wplus(gratio(dqi, dqm, gfloor), limiter, kappa);
    phm[i] = i >= 2 ? limiter_wplus(gratio(dqm, q[i - 1] - q[i - 2], gfloor), limiter, kappa)
                    : 0.0;
  }
  __syncthreads();
}

// assemble (solve = 0: bands / rhs in the reference's BandedMatrix layout
// bands[(d + 2) * n_sys + i]) or solve with the Jacobian ladder jac0..2
// (solve = 1: sigma[0..n-2], rung = the Jacobian that factored, -1 if none)
template <bool EXACT>
__global__ void __launch_bounds__(kLsThreads, 1)
linesys_kernel(paqif_ehl_linesys a, int jac0, int solve, double* bands, double* rhs_out,
               double* sigma, int32_t* rung_out) {
  extern __shared__ __align__(16) double lsm[];
  __shared__ double red[32];
  __shared__ int flag;
  const int n = a.n, N = n + 1, n_int = n - 1;
  const int n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  double* php = lsm;
  double* phm = php + N;
  double* band = phm + N;  // 2N doubles in: 16-byte aligned
  double* rhs = band + aqif2_band_doubles(n_sys);
  double* rec = rhs + aqif2_rhs_doubles(n_sys);
  line_faces(a.q, n, a.limiter, a.kappa, php, phm, red);
  if (solve) aqif2_zero_pads(band, rhs, n_sys);
  int st = 1, jac = jac0;
  for (; jac <= 2; ++jac) {
    for (int r = threadIdx.x; r < n_sys; r += blockDim.x) {
      double e[5] = {0.0, 0.0, 1.0, 0.0, 0.0};
      double rr = 0.0;
      if (r < n_int) {
        const int i = r + 1;
        line_row_entries(a.rho[i - 1], a.rho[i], a.rho[i + 1], a.ex_p[r], a.ex_m[r], a.ey_p[r],
                         a.ey_m[r], php[i], phm[i], a.h, a.hy, a.weighted != 0, jac, a.ks0, a.ks1,
                         e);
        rr = a.resid[r];
      }
#pragma unroll
      for (int d = 0; d < 5; ++d) {
        // padded-matrix semantics (sweeps._padded_matrix): pad rows are
        // identity, entries whose column leaves the matrix are zero
        const int col = r + d - 2;
        const bool keep = r < n_int ? (col >= 0 && col < n_sys) : (d == 2);
        const double v = keep ? e[d] : 0.0;
        if (solve) band2_ref(band, n_sys, r, d - 2) = v;
        else bands[(size_t)d * n_sys + r] = v;
      }
      if (solve) rhs[kBandPad + r] = rr;
      else rhs_out[r] = rr;
    }
    if (!solve) return;
    st = aqif2_solve<EXACT>(band, rhs, n_sys, rec, band, &flag) & 1;
    if (!st) break;
  }
  for (int r = threadIdx.x; r < n_int; r += blockDim.x) sigma[r] = st ? 0.0 : band[r];
  if (threadIdx.x == 0) *rung_out = st ? -1 : jac;
}

__device__ __forceinline__ void rheo_point(double u, double film, const paqif_ehl_rheo& p,
                                           double& rho, double& eps) {
  double eta;
  if (p.compressible) {
    const double pp = u * p.p_hertz;
    rho = (kDensA + kDensB * pp) / (kDensA + pp);
    const double arg = (p.alpha * p.p0 / p.z) * (-1.0 + pow(1.0 + pp / p.p0, p.z));
    eta = exp(np_minimum(arg, 200.0));
  } else {
    rho = 1.0;
    eta = 1.0;
  }
  const double gap = np_maximum(film, 1e-8);
  eps = (rho / (eta * p.lam)) * (gap * gap * gap);
}

// residual field of one line (block = one row j of the point contact, or
// the whole line contact); boundary entries zero
__global__ void __launch_bounds__(kLsThreads)
residual_field_kernel(const double* __restrict__ u, const double* __restrict__ film, int n,
                      int point, paqif_ehl_rheo rp, double h, int limiter, double kappa,
                      double* r) {
  extern __shared__ __align__(16) double rsm[];
  __shared__ double red[32];
  const int N = n + 1;
  const int j = blockIdx.x;
  double* out = r + (size_t)j * N;
  if (point && (j == 0 || j == n)) {
    for (int i = threadIdx.x; i < N; i += blockDim.x) out[i] = 0.0;
    return;
  }
  double* q = rsm;          // rho * film of the row
  double* ec = q + N;       // eps of the row
  double* en = ec + N;      // eps of rows j+1, j-1 (point contact)
  double* es = en + N;
  double* php = es + N;
  double* phm = php + N;
  const size_t row = point ? (size_t)j * N : 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double rho, eps;
    rheo_point(u[row + i], film[row + i], rp, rho, eps);
    q[i] = rho * film[row + i];
    ec[i] = eps;
    if (point) {
      rheo_point(u[row + N + i], film[row + N + i], rp, rho, eps);
      en[i] = eps;
      rheo_point(u[row - N + i], film[row - N + i], rp, rho, eps);
      es[i] = eps;
    }
  }
  __syncthreads();
  line_faces(q, n, limiter, kappa, php, phm, red);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double v = 0.0;
    if (i >= 1 && i < n) {
      const double dqi = q[i + 1] - q[i], dqm = q[i] - q[i - 1];
      const double fd = (q[i] + 0.5 * php[i] * dqi) - (q[i - 1] + 0.5 * phm[i] * dqm);
      const double uc = u[row + i];
      if (!point) {
        const double e_p = 0.5 * (ec[i] + ec[i + 1]);
        const double e_m = 0.5 * (ec[i] + ec[i - 1]);
        v = (e_p * (u[i + 1] - uc) + e_m * (u[i - 1] - uc)) / h - fd;
      } else {
        const double exp_ = 0.5 * (ec[i] + ec[i + 1]) * h;
        const double exm = 0.5 * (ec[i] + ec[i - 1]) * h;
        const double eyp = 0.5 * (ec[i] + en[i]) * h;
        const double eym = 0.5 * (ec[i] + es[i]) * h;
        v = (exp_ * (u[row + i + 1] - uc) + exm * (u[row + i - 1] - uc)) / h +
            (eyp * (u[row + N + i] - uc) + eym * (u[row - N + i] - uc)) / h - h * fd;
      }
    }
    out[i] = v;
  }
}

size_t linesys_smem(int n) {
  const int N = n + 1, n_int = n - 1;
  const int n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  return (2 * (size_t)N + 1 + aqif2_band_doubles(n_sys) + aqif2_rhs_doubles(n_sys) +
          (size_t)(n_sys / 2 + 1) * kRec2) * 8;
}

}  // namespace paqif

using namespace paqif;

namespace {
int linesys_launch(const paqif_ehl_linesys* a, int jac0, int solve, double* bands, double* rhs,
                   double* sigma, int32_t* rung, void* stream, const char* who) {
  if (!a || a->n < 4 || a->limiter < 0 || a->limiter > 4 || !a->q || !a->rho || !a->resid)
    return set_arg_error(who);
  const size_t smem = linesys_smem(a->n);
  if (smem > 227 * 1024) return set_arg_error("ehl_linesys: line too long for one CTA");
  cudaFuncSetAttribute(linesys_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  linesys_kernel<true><<<1, kLsThreads, smem, (cudaStream_t)stream>>>(*a, jac0, solve, bands, rhs,
                                                                      sigma, rung);
  return check_launch(who);
}
}  // namespace

extern "C" int paqif_ehl_assemble_line(const paqif_ehl_linesys* a, int32_t jacobian,
                                       double* bands, double* rhs, void* stream) {
  if (jacobian < 0 || jacobian > 2 || !bands || !rhs)
    return set_arg_error("ehl_assemble_line: jacobian / outputs");
  return linesys_launch(a, jacobian, 0, bands, rhs, nullptr, nullptr, stream,
                        "paqif_ehl_assemble_line");
}

extern "C" int paqif_ehl_robust_line_solve(const paqif_ehl_linesys* a, double* sigma,
                                           int32_t* rung, void* stream) {
  if (!sigma || !rung) return set_arg_error("ehl_robust_line_solve: outputs");
  return linesys_launch(a, 0, 1, nullptr, nullptr, sigma, rung, stream,
                        "paqif_ehl_robust_line_solve");
}

extern "C" int paqif_ehl_residual_field(const double* u, const double* film, int64_t n,
                                        int32_t point, const paqif_ehl_rheo* rp, double h,
                                        int32_t limiter, double kappa, double* r, void* stream) {
  if (!u || !film || !r || !rp || n < 2 || limiter < 0 || limiter > 4)
    return set_arg_error("ehl_residual_field");
  const size_t smem = 6 * (size_t)(n + 1) * 8;
  if (smem > 227 * 1024) return set_arg_error("ehl_residual_field: line too long");
  cudaFuncSetAttribute(residual_field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  residual_field_kernel<<<point ? (unsigned)(n + 1) : 1u, kLsThreads, smem,
                          (cudaStream_t)stream>>>(u, film, (int)n, point, *rp, h, limiter, kappa,
                                                  r);
  return check_launch("paqif_ehl_residual_field");
}
