// Fused EHL line-contact Newton step (configs 1 and 3): one CTA per load
// case runs one complete outer iteration of solve_ehl for the line contact
// (paqif/ehl/solver.py:131-183 + 217-222 + 43-51):
//
//   film    = h0 + x^2/2 - (1/pi) sum_j K|i-j| u_j     deformation, film.py:67-71
//   rho, eta, eps = rheology(u, film)                  params.py:149-175
//   q = rho film; limited faces phi+, phi-; flux diff  sweeps.py:47-56, 89-103
//   resid = (e+ (u_E-u_P) + e- (u_W-u_P))/h - fdiff   solver.py:144-149
//   Ls1 / Ls4 pentadiagonal Jacobians + bad-row fix,
//   row merge by the weighted mask eps/h <= 0.6        sweeps.py:157-267, solver.py:153-162
//   AQIF solve (factor + W fused, Z outside-in); on a
//   breakdown the Ls4 ladder scheme/first-order/diag   sweeps.py:270-295, solver.py:163-168
//   clip, weighted spread, u = max(0, u + w(s - sp/4))  solver.py:169-181
//   deformation of the new pressure                    solver.py:182
//   force balance every force_every-th iteration       sweeps.py:521-535
//   complementarity residual max|min(u, -R)|/h         solver.py:43-51
//
// The Toeplitz convolution is register-tiled (4 outputs per thread, one
// shared-memory kernel value and one broadcast pressure per 4 DFMA); the
// banded solve runs on one warp through the beta=2 latency engine
// (aqif2.cuh) with the line system, right side and pivot records in shared
// memory (in the case's workspace when n is too large for that).  Elementwise formulas follow numpy's operation order; the
// convolution and the load sum use a different summation order than
// numpy's BLAS dot / pairwise sum (documented tolerance).
#include <cfloat>
#include <cstdlib>
#include "aqif2.cuh"
#include "aqif_warp.cuh"
#include "zsolve.cuh"
#include "ehl_common.cuh"
#include "capi_util.cuh"

namespace paqif {

constexpr int kEhlThreads = 256;
constexpr int kEhlBeta = 2;

struct EhlSmemLayout {
  // offsets in doubles
  // band/rhs/rec: the line system (5 x n_sys), its right side and the AQIF
  // pivot records, when they fit (sys_in_smem); else in the workspace
  int ext, su, sun, film, rho, eps, q, php, phm, res, sig, def, red, band, rhs, rec, total;
  bool sys_in_smem;
  __host__ __device__ static int nsys(int n) {
    const int n_int = n - 1;
    return (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  }
  __host__ __device__ explicit EhlSmemLayout(int n) {
    const int N = n + 1, NA = (N + 3 + 1) & ~1;  // padded for the 4-wide conv tail
    int o = 0;
    ext = o; o += ext4_doubles(n); o = (o + 1) & ~1;  // line kernel, ext4 layout
    su = o; o += NA;
    sun = o; o += NA;
    film = o; o += NA;
    rho = o; o += NA;
    eps = o; o += NA;
    q = o; o += NA;
    php = o; o += NA;
    phm = o; o += NA;
    res = o; o += NA;
    sig = o; o += NA;
    def = o; o += NA;
    red = o; o += 32;
    const int ns = nsys(n);
    const int sys = (int)(aqif2_band_doubles(ns) + aqif2_rhs_doubles(ns)) + (ns / 2 + 1) * kRec2;
    sys_in_smem = (size_t)(o + sys) * 8 <= 227 * 1024;
    band = o;
    rhs = o + (int)aqif2_band_doubles(ns);
    rec = rhs + (int)aqif2_rhs_doubles(ns);
    if (sys_in_smem) o += sys;
    total = o;
  }
};

}  // namespace paqif

// ----------------------------------------------------------------- C ABI cfg
extern "C" {
#include "../../include/paqif_ehl.h"
}

namespace paqif {

__device__ __forceinline__ void rheology(double u, double film, const paqif_ehl_line_cfg& c,
                                         double ph, double lam, double& rho, double& eps) {
  double eta;
  if (c.compressible) {
    const double p = u * ph;
    rho = (kDensA + kDensB * p) / (kDensA + p);
    const double arg = (c.alpha * c.p0 / c.z) * (-1.0 + pow(1.0 + p / c.p0, c.z));
    eta = exp(np_minimum(arg, 200.0));
  } else {
    rho = 1.0;
    eta = 1.0;
  }
  const double coeff = rho / (eta * lam);
  const double gap = np_maximum(film, 1e-8);
  eps = coeff * (gap * gap * gap);
}

// Assemble row r (interior node i = r+1) of the change system in the
// requested scheme / Jacobian mode; writes the 5 band entries.
// jac: 0 scheme, 1 first-order, 2 diagonal.  weighted: Ls4/Ls5 pattern.
__device__ void assemble_row(int i, const double* rho, const double* eps, const double* php,
                             const double* phm, double h, bool weighted, int jac, double ks0,
                             double ks1, double* e /*[5]*/) {
  const double ex_p = 0.5 * (eps[i] + eps[i + 1]);
  const double ex_m = 0.5 * (eps[i] + eps[i - 1]);
  line_row_entries(rho[i - 1], rho[i], rho[i + 1], ex_p, ex_m, 0.0, 0.0, php[i], phm[i], h, 1.0,
                   weighted, jac, ks0, ks1, e);
}

// complementarity residual max|min(u, -R(u))| of a pressure (solver.py:43-51,
// sweeps.py:106-123) with its film; returns the CTA-wide (NaN-propagating) max
__device__ double line_comp_residual(const paqif_ehl_line_cfg& c, double h0, const double* sun,
                                     const double* sdef, double ph, double lam, double* sfilm,
                                     double* seps, double* sq, double* red) {
  const int n = c.n, N = n + 1;
  const double h = c.h;
  const double sign = -1.0 / 3.141592653589793;
  double qmax = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double x = c.lo + h * (double)i;
    const double fv = (h0 + 0.5 * (x * x)) + sign * sdef[i];
    double rho, eps;
    rheology(sun[i], fv, c, ph, lam, rho, eps);
    sfilm[i] = fv;
    seps[i] = eps;
    sq[i] = rho * fv;
    qmax = fmax(qmax, fabs(rho * fv));
  }
  const double gfloor2 = 1e-12 * fmax(block_max(qmax, red), kRatioGuard);
  double comp = 0.0;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double r = 0.0;
    if (i >= 1 && i <= n - 1) {
      const double dqi = sq[i + 1] - sq[i], dqm = sq[i] - sq[i - 1];
      const double php = limiter_wplus(gratio(dqi, dqm, gfloor2), c.limiter, c.kappa);
      double phm = 0.0;
      if (i >= 2) {
        const double dqmm = sq[i - 1] - sq[i - 2];
        phm = limiter_wplus(gratio(dqm, dqmm, gfloor2), c.limiter, c.kappa);
      }
      const double fd = (sq[i] + 0.5 * php * dqi) - (sq[i - 1] + 0.5 * phm * dqm);
      const double e_p = 0.5 * (seps[i] + seps[i + 1]);
      const double e_m = 0.5 * (seps[i] + seps[i - 1]);
      r = (e_p * (sun[i + 1] - sun[i]) + e_m * (sun[i - 1] - sun[i])) / h - fd;
    }
    const double m = fabs(np_minimum(sun[i], -r));
    comp = ((comp != comp) | (m != m)) ? qnan : (m > comp ? m : comp);
  }
  return block_nanmax(comp, red);
}

// residual-only pass (EhlState.complementarity_residual for line states)
__global__ void __launch_bounds__(kEhlThreads)
ehl_line_residual_kernel(paqif_ehl_line_cfg c, int64_t B, const double* __restrict__ table,
                         const double* __restrict__ p_hertz, const double* __restrict__ lamv,
                         const double* u_in, const double* h0_in, double* film_out,
                         double* res_out, double* gscratch, size_t gstride) {
  extern __shared__ __align__(16) double dsm[];
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  // arrays in HBM (gscratch, one stride per case) when the grid is too fine
  // for one CTA's shared memory
  double* esm = gscratch ? gscratch + (size_t)b * gstride : dsm;
  const int n = c.n, N = n + 1;
  const EhlSmemLayout L(n);
  double* ext = esm + L.ext;
  double* su = esm + L.su;
  double* sdef = esm + L.def;
  for (int k = threadIdx.x; k < N; k += blockDim.x) su[k] = u_in[b * N + k];
  ext4_build(table, n, ext);
  __syncthreads();
  toeplitz_conv(su, ext, n, 1.0, sdef);
  __syncthreads();
  const double cmax = line_comp_residual(c, h0_in[b], su, sdef, p_hertz[b], lamv[b],
                                         esm + L.film, esm + L.eps, esm + L.q, esm + L.red);
  if (film_out)
    for (int i = threadIdx.x; i < N; i += blockDim.x) film_out[b * N + i] = esm[L.film + i];
  if (threadIdx.x == 0) res_out[b] = cmax / c.h;
}

// solve_ehl's per-iteration bookkeeping and stop / divergence tests
// (ehl/solver.py:219-240), same comparisons in the same order.
__device__ void line_drive_update(paqif_ehl_line_drive& d, double res, int fb, double deficit,
                                  int finite, double* hist_res, double* hist_def, int hist_cap,
                                  int64_t b) {
  const int k = d.outer;
  if (hist_res && hist_cap > 0) {
    hist_res[b * hist_cap + k % hist_cap] = res;
    hist_def[b * hist_cap + k % hist_cap] = fb ? deficit : __longlong_as_double(0x7ff8000000000000ll);
  }
  if (fb) d.deficit = fabs(deficit);
  d.outer = k + 1;
  if (!finite) {  // the host driver raises after this step
    d.done = 5;
    return;
  }
  if (res <= d.tol && fabs(d.deficit) <= d.tol_fb) {
    d.done = 1;
    return;
  }
  if (res < d.best) {
    d.best = res;
    d.grow = 0;
  } else {
    d.grow += 1;
    if (d.grow >= 20 && res > 1e3 * fmax(d.best, d.tol)) {
      d.done = 2;
      return;
    }
  }
  if (d.outer >= d.max_outer) d.done = 3;
}


// ------------------------------------------------------------------ phases
// The outer iteration of one case in three phases, shared by the fused
// kernel (one CTA per case runs all three, the solve on one warp) and the
// split path for large batches (phase A, a batched solve of every case's
// rung systems, phase C as three kernels).

// Phase A: film, rheology, limited faces and Reynolds residual of the
// current pressure su (solver.py:141-149); fills sdef, sfilm, srho, seps,
// sq, sphp, sphm, sres.  All threads call.
__device__ __forceinline__ void line_phase_a(const paqif_ehl_line_cfg& c, double h0, double ph,
                                             double lam, const double* su, const double* ext,
                                             double* sdef, double* sfilm, double* srho,
                                             double* seps, double* sq, double* sphp,
                                             double* sphm, double* sres, double* red) {
  const int n = c.n, N = n + 1;
  const double h = c.h;
  const double sign = -1.0 / 3.141592653589793;
  toeplitz_conv(su, ext, n, 1.0, sdef);
  __syncthreads();
  double qmax = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double x = c.lo + h * (double)i;
    const double fv = (h0 + 0.5 * (x * x)) + sign * sdef[i];
    double rho, eps;
    rheology(su[i], fv, c, ph, lam, rho, eps);
    if (sfilm) sfilm[i] = fv;
    srho[i] = rho;
    seps[i] = eps;
    sq[i] = rho * fv;
    qmax = fmax(qmax, fabs(rho * fv));
  }
  const double gfloor = 1e-12 * fmax(block_max(qmax, red), kRatioGuard);
  for (int i = 1 + threadIdx.x; i < n; i += blockDim.x) {
    const double dqi = sq[i + 1] - sq[i], dqm = sq[i] - sq[i - 1];
    const double php = limiter_wplus(gratio(dqi, dqm, gfloor), c.limiter, c.kappa);
    double phm = 0.0;
    if (i >= 2) {
      const double dqmm = sq[i - 1] - sq[i - 2];
      phm = limiter_wplus(gratio(dqm, dqmm, gfloor), c.limiter, c.kappa);
    }
    sphp[i] = php;
    sphm[i] = phm;
    const double fd = (sq[i] + 0.5 * php * dqi) - (sq[i - 1] + 0.5 * phm * dqm);
    const double e_p = 0.5 * (seps[i] + seps[i + 1]);
    const double e_m = 0.5 * (seps[i] + seps[i - 1]);
    sres[i] = (e_p * (su[i + 1] - su[i]) + e_m * (su[i - 1] - su[i])) / h - fd;
  }
  __syncthreads();
}

// kernel sensitivities of the plain (Newton) and weighted rows
// (film.sensitivity, sweeps.kernel_nu)
struct LineKs {
  double ks0n, ks1n, ks0w, ks1w;
  __device__ LineKs(const paqif_ehl_line_cfg& c, const double* table) {
    const double sign = -1.0 / 3.141592653589793;
    const double s0 = sign * table[0], s1 = sign * table[1], s2 = sign * table[2];
    const double nu = c.variant == 0 ? (2.0 - c.kappa) / 2.0
                                     : (2.0 - c.kappa) / 2.0 + (1.0 - c.kappa) / 4.0;
    ks0n = s0;
    ks1n = s1;
    ks0w = nu * (s0 - 0.25 * (2.0 * s1 + 0.0));
    ks1w = nu * (s1 - 0.25 * (s0 + s2 + 0.0));
  }
};

// Assemble rung `rung` of row r of the padded change system (rung -1: the
// combined per-row Ls1/Ls4 system; 0..2: Ls4 with scheme / first-order /
// diagonal Jacobian, solver.py:153-168, sweeps.py:276-295).  Writes the 5
// band entries (offsets -2..2, exact zeros outside the padded matrix) and
// returns the right side; *wrow = the row is weighted (eps/h <= 0.6).
__device__ __forceinline__ double line_row(const paqif_ehl_line_cfg& c, int rung, int r,
                                           int n_int, int n_sys, const double* srho,
                                           const double* seps, const double* sphp,
                                           const double* sphm, const double* sres,
                                           const LineKs& ks, double* e, bool* wrow) {
  const double h = c.h;
  e[0] = 0.0; e[1] = 0.0; e[2] = 1.0; e[3] = 0.0; e[4] = 0.0;
  double rr = 0.0;
  *wrow = false;
  if (r < n_int) {
    const int i = r + 1;
    *wrow = (seps[i] / h) <= kSwitch;
    const bool weighted = rung >= 0 || *wrow;
    assemble_row(i, srho, seps, sphp, sphm, h, weighted, rung < 0 ? 0 : rung,
                 weighted ? ks.ks0w : ks.ks0n, weighted ? ks.ks1w : ks.ks1n, e);
    rr = sres[i];
  }
#pragma unroll
  for (int d = 0; d < 5; ++d) {
    const int col = r + d - kEhlBeta;
    // padded-matrix semantics: rows beyond n_int are identity; entries
    // leaving the (padded) matrix are exact zeros
    const bool keep = r < n_int ? (col >= 0 && col < n_sys) : (d == kEhlBeta);
    if (!keep) e[d] = 0.0;
  }
  return rr;
}

// Phase C: clip, weighted spread and update (solver.py:169-181), deformation
// of the new pressure, force balance, complementarity residual and the
// outputs / drive bookkeeping of case b.  xsol(i) = the line solve's change
// of unknown i; seps holds phase A's eps (the weighted mask) on entry.
template <class XS>
__device__ __forceinline__ void line_phase_c(
    const paqif_ehl_line_cfg& c, int outer, double h0, double ph, double lam, XS xsol,
    const double* su, double* sun, double* ssig, const double* ext, double* sdef, double* sfilm,
    double* seps, double* sq, double* red, int rung, int weighted_rows, double* u_io,
    double* h0_io, double* film_out, double* res_out, double* deficit_out, int32_t* info_out,
    paqif_ehl_line_drive* drv, double* hist_res, double* hist_def, int hist_cap, int64_t b) {
  const int n = c.n, N = n + 1;
  const double h = c.h;
  bool finite = true;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    double sg = 0.0;
    if (i >= 1 && i <= n - 1) {
      sg = xsol(i - 1);
      finite &= isfinite(sg);
      sg = np_minimum(np_maximum(sg, -c.max_change), c.max_change);
    }
    ssig[i] = sg;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    auto wsig = [&](int k) -> double {
      if (k < 1 || k > n - 1) return 0.0;
      return (seps[k] / h) <= kSwitch ? ssig[k] : 0.0;
    };
    const double spread = (0.0 + (i >= 1 ? wsig(i - 1) : 0.0)) + (i < n ? wsig(i + 1) : 0.0);
    const double v = su[i] + c.omega * (ssig[i] - 0.25 * spread);
    sun[i] = (i == 0 || i == n) ? 0.0 : np_maximum(0.0, v);
  }
  const int fin_all = __syncthreads_and(finite);
  // ---- deformation of the new pressure, force balance, residual
  toeplitz_conv(sun, ext, n, 1.0, sdef);
  __syncthreads();
  int fb = 0;
  double deficit_v = __longlong_as_double(0x7ff8000000000000ll);
  if ((outer + 1) % c.force_every == 0) {
    double part = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) part += sun[i];
    const double total = block_sum(part, red);
    const double deficit = c.load_target - h * total;
    const double stp = np_minimum(np_maximum(c.relax_c * deficit, -c.max_h0_step), c.max_h0_step);
    h0 = h0 - stp;
    fb = 1;
    deficit_v = deficit;
  }
  const double cmax = line_comp_residual(c, h0, sun, sdef, ph, lam, sfilm, seps, sq, red);
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    u_io[b * N + i] = sun[i];
    film_out[b * N + i] = sfilm[i];
  }
  if (threadIdx.x == 0) {
    h0_io[b] = h0;
    res_out[b] = cmax / h;
    if (deficit_out) deficit_out[b] = deficit_v;
    // info: bits 0-1 rung+1 (0 combined), bit 2 force balance applied,
    // bit 3 non-finite change, bits 16.. weighted rows
    info_out[b] = (rung + 1) | (fb << 2) | ((fin_all ? 0 : 1) << 3) | (weighted_rows << 16);
    if (drv) line_drive_update(drv[b], cmax / h, fb, deficit_v, fin_all, hist_res, hist_def,
                               hist_cap, b);
  }
}

// every rung broke down: the reference re-raises (robust_line_solve)
__device__ __forceinline__ void line_all_rungs_failed(int64_t b, double* res_out,
                                                      double* deficit_out, int32_t* info_out,
                                                      paqif_ehl_line_drive* drv) {
  if (threadIdx.x == 0) {
    res_out[b] = __longlong_as_double(0x7ff8000000000000ll);
    if (deficit_out) deficit_out[b] = __longlong_as_double(0x7ff8000000000000ll);
    info_out[b] = 1 << 8;
    if (drv) drv[b].done = 4;
  }
}

// One outer iteration of case b, fused; all threads of the CTA call (esm:
// the CTA's dynamic shared memory).
template <bool EXACT, bool SMEM>
__device__ __forceinline__ void line_case(
    const paqif_ehl_line_cfg& c, int64_t B, const double* __restrict__ table,
    const double* __restrict__ p_hertz, const double* __restrict__ lamv, double* u_io,
    double* h0_io, double* film_out, double* res_out, double* deficit_out, int32_t* info_out,
    char* ws, size_t ws_per_case, paqif_ehl_line_drive* drv, double* hist_res, double* hist_def,
    int hist_cap, const int64_t b, double* esm)
{
  int outer = c.outer;
  if (drv) {  // device-driven solve_ehl: stopped cases skip
    if (drv[b].done) return;
    outer = drv[b].outer;
  }
  const int n = c.n, N = n + 1, n_int = n - 1;
  const int n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  const EhlSmemLayout L(n);
  double* ext = esm + L.ext;
  double* su = esm + L.su;
  double* red = esm + L.red;
  // line system: shared memory, or this case's workspace for large n
  double* wsd = reinterpret_cast<double*>(ws + (size_t)b * ws_per_case);
  double* band = SMEM ? esm + L.band : wsd;  // SMEM: shared address space known
  double* rhs = band + aqif2_band_doubles(n_sys);
  double* rec = rhs + aqif2_rhs_doubles(n_sys);
  aqif2_zero_pads(band, rhs, n_sys);
  double* xsol = band;  // x overwrites the band after the factor
  const double ph = p_hertz[b], lam = lamv[b];
  const double h0 = h0_io[b];

  for (int k = threadIdx.x; k < N; k += blockDim.x) su[k] = u_io[b * N + k];
  ext4_build(table, n, ext);
  __syncthreads();
  line_phase_a(c, h0, ph, lam, su, ext, esm + L.def, esm + L.film, esm + L.rho, esm + L.eps,
               esm + L.q, esm + L.php, esm + L.phm, esm + L.res, red);
  const LineKs ks(c, table);

  // rung -1: combined (per-row Ls1/Ls4); 0..2: Ls4 with scheme/first-order/diagonal
  int rung = -1;
  int st = 1;
  int weighted_rows = 0;
  for (; rung <= 2; ++rung) {
    int wcount = 0;
    for (int r = threadIdx.x; r < n_sys; r += blockDim.x) {
      double e[5];
      bool wrow;
      const double rr = line_row(c, rung, r, n_int, n_sys, esm + L.rho, esm + L.eps,
                                 esm + L.php, esm + L.phm, esm + L.res, ks, e, &wrow);
      wcount += wrow;
#pragma unroll
      for (int d = 0; d < 5; ++d) band2_ref(band, n_sys, r, d - kEhlBeta) = e[d];
      rhs[kBandPad + r] = rr;
    }
    if (rung < 0) weighted_rows = (int)block_sum((double)wcount, red);
    __syncthreads();
    // solve on warp 0 (aqif2: factor + fused W, Z outside-in)
    int* flag = reinterpret_cast<int*>(red + 30);
    st = aqif2_solve<EXACT>(band, rhs, n_sys, rec, xsol, flag) & 1;
    if (!st) break;
  }
  if (st) {
    line_all_rungs_failed(b, res_out, deficit_out, info_out, drv);
    return;
  }
  line_phase_c(c, outer, h0, ph, lam, [&](int i) { return xsol[i]; }, su, esm + L.sun,
               esm + L.sig, ext, esm + L.def, esm + L.film, esm + L.eps, esm + L.q, red, rung,
               weighted_rows, u_io, h0_io, film_out, res_out, deficit_out, info_out, drv,
               hist_res, hist_def, hist_cap, b);
}

// Grid = one CTA per SM pulling cases from a queue (`queue` non-null: the
// order kernel resets it), in `order` -- the cases that needed the Ls4
// ladder last time first, so the long ones start early and the rest fill
// in behind them; or one CTA per case (queue null).
template <bool EXACT, bool SMEM>
__global__ void __launch_bounds__(kEhlThreads, 1)
ehl_line_kernel(paqif_ehl_line_cfg c, int64_t B, const double* __restrict__ table,
                const double* __restrict__ p_hertz, const double* __restrict__ lamv, double* u_io,
                double* h0_io, double* film_out, double* res_out, double* deficit_out,
                int32_t* info_out, char* ws, size_t ws_per_case, paqif_ehl_line_drive* drv,
                double* hist_res, double* hist_def, int hist_cap, const int32_t* order,
                int* queue)
{
  extern __shared__ __align__(16) double esm[];
  if (!queue) {
    if ((int64_t)blockIdx.x >= B) return;
    line_case<EXACT, SMEM>(c, B, table, p_hertz, lamv, u_io, h0_io, film_out, res_out,
                           deficit_out, info_out, ws, ws_per_case, drv, hist_res, hist_def,
                           hist_cap, (int64_t)blockIdx.x, esm);
    return;
  }
  __shared__ int next;
#ifdef PAQIF_LINE_PROF
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long c0 = clock64();
  int ncase = 0;
#endif
  for (;;) {
    __syncthreads();  // the previous case is done with shared memory and `next`
    if (threadIdx.x == 0) next = atomicAdd(queue, 1);
    __syncthreads();
    const int idx = next;
    if (idx >= B) break;
    line_case<EXACT, SMEM>(c, B, table, p_hertz, lamv, u_io, h0_io, film_out, res_out,
                           deficit_out, info_out, ws, ws_per_case, drv, hist_res, hist_def,
                           hist_cap, (int64_t)order[idx], esm);
#ifdef PAQIF_LINE_PROF
    ++ncase;
#endif
  }
#ifdef PAQIF_LINE_PROF
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0)
    printf("[cta] %d cases %d start_ns %llu end_ns %llu cycles %lld\n", blockIdx.x, ncase, g0, g1,
           clock64() - c0);
#endif
}

// ------------------------------------------------------------- split path
// Large batches (config 3): the fused kernel runs one case per SM with the
// level chain of its line solve on one warp while seven wait.  The split
// path runs the outer iteration as three kernels:
//   A  one CTA per case: phase A and the four rung systems of the case
//      (combined, Ls4 scheme / first-order / diagonal) into its workspace
//   S  every rung system of every case solved side by side by the
//      throughput engine (aqif_warp.cuh: 4 lanes per system, 8 per warp,
//      band streamed from L2 by cp.async hooks, pivot records to a Z
//      stack, full outside-in Z solve): the reference's ladder tries the
//      rungs in order; solving them all at once costs no extra chain
//   C  one CTA per case: the first rung that did not break down, then
//      phase C.
// Same arithmetic as the fused path per phase (the general engine is
// bit-identical to aqif2 in exact mode, tools/aqif2_check.cu).
constexpr int kRungs = 4;

struct SplitSmemA {  // phase-A kernel, offsets in doubles
  int ext, su, def, rho, eps, q, php, phm, res, red, total;
  __host__ __device__ explicit SplitSmemA(int n) {
    const int NA = (n + 1 + 3 + 1) & ~1;
    int o = 0;
    ext = o; o += ext4_doubles(n); o = (o + 1) & ~1;
    su = o; o += NA; def = o; o += NA; rho = o; o += NA; eps = o; o += NA; q = o; o += NA;
    php = o; o += NA; phm = o; o += NA; res = o; o += NA; red = o; o += 32;
    total = o;
  }
};

struct SplitSmemC {  // phase-C kernel
  int ext, su, sun, sig, def, film, eps, q, red, total;
  __host__ __device__ explicit SplitSmemC(int n) {
    const int NA = (n + 1 + 3 + 1) & ~1;
    int o = 0;
    ext = o; o += ext4_doubles(n); o = (o + 1) & ~1;
    su = o; o += NA; sun = o; o += NA; sig = o; o += NA; def = o; o += NA; film = o; o += NA;
    eps = o; o += NA; q = o; o += NA; red = o; o += 32;
    total = o;
  }
};

struct SplitLayout {  // per-case workspace, offsets in doubles
  int n_sys, s;
  bool gsm;
  size_t band, rhs, x, zs, eps, ints, scratch, total;
  __host__ __device__ explicit SplitLayout(int n) {
    const int n_int = n - 1;
    n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
    s = n_sys / 2;
    size_t o = 0;
    band = o; o += (size_t)kRungs * 5 * n_sys;
    rhs = o; o += n_sys;
    x = o; o += (size_t)kRungs * n_sys;
    zs = o; o += (size_t)kRungs * (s + 1) * PivotLayout<2>::kSize;
    eps = o; o += (size_t)n + 1;
    o = (o + 1) & ~(size_t)1;
    ints = o; o += 4;  // status[kRungs] (int32), weighted rows (int32)
    // phase A / C arrays in HBM when they do not fit one CTA's shared
    // memory (very fine line grids: the reference has no size limit)
    const size_t ta = SplitSmemA(n).total, tc = SplitSmemC(n).total;
    const size_t tmax = ta > tc ? ta : tc;
    gsm = tmax * 8 > 227 * 1024;
    o = (o + 31) & ~(size_t)31;
    scratch = o;
    if (gsm) o += tmax;
    total = (o + 31) & ~(size_t)31;
  }
};

__global__ void __launch_bounds__(kEhlThreads)
line_split_a_kernel(paqif_ehl_line_cfg c, int64_t B, const double* __restrict__ table,
                    const double* __restrict__ p_hertz, const double* __restrict__ lamv,
                    const double* __restrict__ u_io, const double* __restrict__ h0_io, double* ws,
                    size_t ws_per_case, const paqif_ehl_line_drive* drv)
{
  extern __shared__ __align__(16) double dsm[];
  const int64_t b = blockIdx.x;
  if (b >= B || (drv && drv[b].done)) return;
  const int n = c.n, N = n + 1, n_int = n - 1;
  const SplitSmemA L(n);
  const SplitLayout W(n);
  const int n_sys = W.n_sys;
  double* w = ws + (size_t)b * ws_per_case;
  double* esm = W.gsm ? w + W.scratch : dsm;
  double* su = esm + L.su;
  for (int k = threadIdx.x; k < N; k += blockDim.x) su[k] = u_io[b * N + k];
  ext4_build(table, n, esm + L.ext);
  __syncthreads();
  line_phase_a(c, h0_io[b], p_hertz[b], lamv[b], su, esm + L.ext, esm + L.def, nullptr,
               esm + L.rho, esm + L.eps, esm + L.q, esm + L.php, esm + L.phm, esm + L.res,
               esm + L.red);
  const LineKs ks(c, table);
  int wcount = 0;
  for (int r = threadIdx.x; r < n_sys; r += blockDim.x) {
    double rr = 0.0;
#pragma unroll 1
    for (int rung = -1; rung <= 2; ++rung) {
      double e[5];
      bool wrow;
      rr = line_row(c, rung, r, n_int, n_sys, esm + L.rho, esm + L.eps, esm + L.php,
                    esm + L.phm, esm + L.res, ks, e, &wrow);
      if (rung < 0) wcount += wrow;
      double* band = w + W.band + (size_t)(rung + 1) * 5 * n_sys;
#pragma unroll
      for (int d = 0; d < 5; ++d) band[(size_t)d * n_sys + r] = e[d];
    }
    w[W.rhs + r] = rr;
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) w[W.eps + i] = esm[L.eps + i];
  const int wrows = (int)block_sum((double)wcount, esm + L.red);
  if (threadIdx.x == 0) reinterpret_cast<int32_t*>(w + W.ints)[kRungs] = wrows;
}

struct SplitSysPol {
  static constexpr bool kFuseW = true;
  static constexpr bool kResidual = false;
  static constexpr bool kFastDiv = true;        // branch-free divisions, checked repeat
  static constexpr bool kDivFix = true;         // subnormal midpoints fixed inline
  static constexpr bool kLazyBreakdown = true;  // breakdown found after the loop
  static constexpr bool kRecordW = false;
  using PL = PivotLayout<2>;
  const double* band;
  const double* rhs;
  double* zs;
  int n;
  __device__ __forceinline__ const double* raw_ptr(int i, int d) const {
    return band + (size_t)(d + 2) * n + i;
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
  __device__ __forceinline__ const double* record(int k) const {
    return zs + (size_t)k * PL::kSize;
  }
};

constexpr int kSplitWarps = 2;
constexpr int kSplitPerWarp = 8;  // systems per warp (measured 1/2/4/8: 1.72/1.09/0.99/0.96 ms)
struct SplitSolveSmem {
  union {
    EngineSmem<2> eng;
    double ring[ZChunk<2>::kRing];
  };
};

// Every rung system of every case side by side: system m = case m / kRungs,
// rung m % kRungs.  The reference tries the rungs in order (combined system,
// then the Ls4 ladder); solving all four at once costs no extra chain,
// while a second pass for the cases whose combined system broke down would
// add a whole level chain (measured: 1.28 vs 0.96 ms per config-3 step).
// pw systems per warp (groups g >= pw idle); a warp without a live system
// returns at once.
template <bool EXACT>
__global__ void __launch_bounds__(32 * kSplitWarps)
line_split_solve_kernel(int n, int64_t B, double* ws, size_t ws_per_case,
                        const paqif_ehl_line_drive* drv, int pw)
{
  constexpr int G = Group<2>::G, P = Group<2>::P;
  __shared__ SplitSolveSmem smem[kSplitWarps * P];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane / G, gl = lane % G;
  const int64_t m = ((int64_t)blockIdx.x * kSplitWarps + wid) * pw + g;
  const int64_t b = m / kRungs;
  const int rung = (int)(m % kRungs);
  const bool alive = g < pw && m < B * kRungs && !(drv && drv[b < B ? b : 0].done);
  if (!__any_sync(0xffffffffu, alive)) return;
  const SplitLayout W(n);
  const int n_sys = W.n_sys;
  double* w = ws + (size_t)(alive ? b : 0) * ws_per_case;
  SplitSysPol pol;
  pol.band = w + W.band + (size_t)rung * 5 * n_sys;
  pol.rhs = w + W.rhs;
  pol.zs = w + W.zs + (size_t)rung * (W.s + 1) * PivotLayout<2>::kSize;
  pol.n = n_sys;
  SplitSolveSmem& sm = smem[wid * P + g];
  int fst = aqif_factor_group<2, EXACT>(pol, n_sys, 1e-14, sm.eng, gl, alive);
  if (EXACT && __any_sync(0xffffffffu, fst < 0)) {
    // a quotient left the branch-free division's range: repeat with IEEE
    // divisions (the other systems of the warp idle)
    __syncwarp();
    const int f2 = aqif_factor_group<2, EXACT, SplitSysPol, false>(pol, n_sys, 1e-14, sm.eng, gl,
                                                                   alive && fst < 0);
    if (fst < 0) fst = f2;
  }
  __syncwarp();
  double* x = w + W.x + (size_t)rung * n_sys;
  const int zst = zsolve_group<2, EXACT, true>(pol.zs, n_sys, x, sm.ring, gl, alive && fst == 0);
  if (alive && gl == 0)
    reinterpret_cast<int32_t*>(w + W.ints)[rung] = (fst || zst) ? 1 : 0;
}

__global__ void __launch_bounds__(kEhlThreads)
line_split_c_kernel(paqif_ehl_line_cfg c, int64_t B, const double* __restrict__ table,
                    const double* __restrict__ p_hertz, const double* __restrict__ lamv,
                    double* u_io, double* h0_io, double* film_out, double* res_out,
                    double* deficit_out, int32_t* info_out, double* ws, size_t ws_per_case,
                    paqif_ehl_line_drive* drv, double* hist_res, double* hist_def, int hist_cap)
{
  extern __shared__ __align__(16) double dsm[];
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  int outer = c.outer;
  if (drv) {
    if (drv[b].done) return;
    outer = drv[b].outer;
  }
  const int n = c.n, N = n + 1;
  const SplitSmemC L(n);
  const SplitLayout W(n);
  double* w = ws + (size_t)b * ws_per_case;
  double* esm = W.gsm ? w + W.scratch : dsm;
  const int32_t* wi = reinterpret_cast<const int32_t*>(w + W.ints);
  int r = 0;
  while (r < kRungs && wi[r] != 0) ++r;
  if (r == kRungs) {
    line_all_rungs_failed(b, res_out, deficit_out, info_out, drv);
    return;
  }
  const int wrows = wi[kRungs];
  double* su = esm + L.su;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    su[k] = u_io[b * N + k];
    esm[L.eps + k] = w[W.eps + k];
  }
  ext4_build(table, n, esm + L.ext);
  __syncthreads();
  const double* xs = w + W.x + (size_t)r * W.n_sys;
  line_phase_c(c, outer, h0_io[b], p_hertz[b], lamv[b], [&](int i) { return xs[i]; }, su,
               esm + L.sun, esm + L.sig, esm + L.ext, esm + L.def, esm + L.film, esm + L.eps,
               esm + L.q, esm + L.red, r - 1, wrows, u_io, h0_io, film_out, res_out,
               deficit_out, info_out, drv, hist_res, hist_def, hist_cap, b);
}

}  // namespace paqif

using namespace paqif;

namespace {
// per-case workspace bytes: the line system when it does not fit in shared
// memory (EhlSmemLayout), else a small pad
size_t line_ws_per_case(int64_t n) {
  const int64_t n_int = n - 1;
  const int64_t n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  const int64_t s = n_sys / 2;
  if (n <= (1 << 20) && EhlSmemLayout((int)n).sys_in_smem) return 256;
  const size_t per = (aqif2_band_doubles((int)n_sys) + aqif2_rhs_doubles((int)n_sys) +
                      (size_t)(s + 1) * kRec2 + 32) * 8;
  return (per + 255) & ~(size_t)255;
}

size_t split_ws_per_case(int64_t n) {
  return (size_t)paqif::SplitLayout((int)n).total * 8;
}
}  // namespace

// B per-case areas (the larger of the fused and the split layout), then the
// case order (B int32) and the queue counter
extern "C" size_t paqif_ehl_line_workspace_bytes(int64_t B, int64_t n) {
  if (B < 0 || n < 4 || n > (1 << 20)) return 0;
  const size_t per = line_ws_per_case(n) > split_ws_per_case(n) ? line_ws_per_case(n)
                                                                 : split_ws_per_case(n);
  return (size_t)B * per + (((size_t)B * 4 + 4 + 255) & ~(size_t)255);
}

namespace paqif {
// Case order for the next launch: the cases whose last step needed the Ls4
// ladder (several line solves; info bits 0-1 or bit 8) first, so they start
// in the first wave instead of trailing the last one.  Results do not depend
// on the order (every case is independent); `info` may hold anything.
__global__ void line_order_kernel(const int32_t* __restrict__ info, int64_t B, int32_t* order,
                                  int* queue) {
  __shared__ int lo, hi;
  if (threadIdx.x == 0) {
    lo = 0;
    hi = 0;
    *queue = 0;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < B; i += blockDim.x) {
    const int32_t v = info[i];
    const bool slow = (v & 3) != 0 || (v & (1 << 8)) != 0;
    if (slow) order[atomicAdd(&hi, 1)] = (int32_t)i;
    else order[B - 1 - atomicAdd(&lo, 1)] = (int32_t)i;
  }
}
}  // namespace paqif

namespace {
int line_launch(const paqif_ehl_line_cfg* cfg, int64_t B, int32_t steps, const double* table,
                const double* p_hertz, const double* lam, double* u, double* h0, double* film,
                double* res, double* deficit, int32_t* info, paqif_ehl_line_drive* drv,
                double* hist_res, double* hist_def, int32_t hist_cap, uint32_t flags,
                void* workspace, size_t workspace_bytes, void* stream, const char* who) {
  if (!cfg || B < 0 || cfg->n < 4 || cfg->force_every < 1 || steps < 0)
    return set_arg_error("ehl_line: bad cfg");
  if (B == 0 || steps == 0) return PAQIF_OK;
  const size_t need = paqif_ehl_line_workspace_bytes(B, cfg->n);
  if (workspace_bytes < need) return set_arg_error("ehl_line: workspace too small");
  const EhlSmemLayout L(cfg->n);
  const size_t smem = (size_t)L.total * 8;
  const bool fused_fits = smem <= 227 * 1024;  // else the split path (any n)
  const size_t per = line_ws_per_case(cfg->n) > split_ws_per_case(cfg->n)
                         ? line_ws_per_case(cfg->n) : split_ws_per_case(cfg->n);
  int32_t* order = reinterpret_cast<int32_t*>((char*)workspace + (size_t)B * per);
  int* queue = reinterpret_cast<int*>(order + B);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  cudaStream_t st = (cudaStream_t)stream;
  if ((flags & PAQIF_FLAG_LINE_FUSED) && !fused_fits)
    return set_arg_error("ehl_line: grid too fine for the fused path (one CTA per case)");
  const bool split = (flags & PAQIF_FLAG_LINE_SPLIT) || !fused_fits ||
                     (!(flags & PAQIF_FLAG_LINE_FUSED) && B >= 2 * (int64_t)sms);
  if (split) {
    const bool exact = flags & PAQIF_FLAG_EXACT;
    const bool gsm = SplitLayout(cfg->n).gsm;
    const size_t sa = gsm ? 0 : (size_t)SplitSmemA(cfg->n).total * 8;
    const size_t sc = gsm ? 0 : (size_t)SplitSmemC(cfg->n).total * 8;
    if (!gsm) {
      cudaFuncSetAttribute(line_split_a_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
      cudaFuncSetAttribute(line_split_c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc);
    }
    static int pw = 0;
    if (!pw) {
      const char* e = getenv("PAQIF_SPLIT_PW");  // dev knob: systems per warp
      pw = e ? atoi(e) : kSplitPerWarp;
      if (pw < 1 || pw > Group<2>::P) pw = kSplitPerWarp;
    }
    const int64_t warps = (B * kRungs + pw - 1) / pw;
    const unsigned sgrid = (unsigned)((warps + kSplitWarps - 1) / kSplitWarps);
    double* wsd = reinterpret_cast<double*>(workspace);
    const size_t perd = per / 8;
    for (int32_t s = 0; s < steps; ++s) {
      line_split_a_kernel<<<(unsigned)B, kEhlThreads, sa, st>>>(*cfg, B, table, p_hertz, lam, u,
                                                                 h0, wsd, perd, drv);
      if (exact)
        line_split_solve_kernel<true><<<sgrid, 32 * kSplitWarps, 0, st>>>(cfg->n, B, wsd, perd,
                                                                            drv, pw);
      else
        line_split_solve_kernel<false><<<sgrid, 32 * kSplitWarps, 0, st>>>(cfg->n, B, wsd, perd,
                                                                             drv, pw);
      line_split_c_kernel<<<(unsigned)B, kEhlThreads, sc, st>>>(
          *cfg, B, table, p_hertz, lam, u, h0, film, res, deficit, info, wsd, perd, drv, hist_res,
          hist_def, hist_cap);
    }
    return check_launch(who);
  }
  const bool queued = B > sms;
  auto kern = (flags & PAQIF_FLAG_EXACT)
                  ? (L.sys_in_smem ? ehl_line_kernel<true, true> : ehl_line_kernel<true, false>)
                  : (L.sys_in_smem ? ehl_line_kernel<false, true> : ehl_line_kernel<false, false>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int32_t s = 0; s < steps; ++s) {
    if (queued) line_order_kernel<<<1, 1024, 0, st>>>(info, B, order, queue);
    kern<<<(unsigned)(queued ? sms : B), kEhlThreads, smem, st>>>(
        *cfg, B, table, p_hertz, lam, u, h0, film, res, deficit, info, (char*)workspace, per, drv,
        hist_res, hist_def, hist_cap, queued ? order : nullptr, queued ? queue : nullptr);
  }
  return check_launch(who);
}
}  // namespace

extern "C" int paqif_ehl_line_step(const paqif_ehl_line_cfg* cfg, int64_t B, const double* table,
                                   const double* p_hertz, const double* lam, double* u,
                                   double* h0, double* film, double* res, double* deficit,
                                   int32_t* info, uint32_t flags, void* workspace,
                                   size_t workspace_bytes, void* stream)
{
  return line_launch(cfg, B, 1, table, p_hertz, lam, u, h0, film, res, deficit, info, nullptr,
                     nullptr, nullptr, 0, flags, workspace, workspace_bytes, stream,
                     "paqif_ehl_line_step");
}

extern "C" int paqif_ehl_line_drive_steps(const paqif_ehl_line_cfg* cfg, int64_t B, int32_t steps,
                                          const double* table, const double* p_hertz,
                                          const double* lam, double* u, double* h0, double* film,
                                          double* res, double* deficit, int32_t* info,
                                          paqif_ehl_line_drive* drive, double* hist_res,
                                          double* hist_def, int32_t hist_cap, uint32_t flags,
                                          void* workspace, size_t workspace_bytes, void* stream)
{
  if (!drive || (hist_res && !hist_def) || (hist_res && hist_cap < 1))
    return set_arg_error("ehl_line_drive_steps: bad drive / history");
  return line_launch(cfg, B, steps, table, p_hertz, lam, u, h0, film, res, deficit, info, drive,
                     hist_res, hist_def, hist_cap, flags, workspace, workspace_bytes, stream,
                     "paqif_ehl_line_drive_steps");
}

namespace paqif {
__global__ void __launch_bounds__(kEhlThreads)
line_deformation_kernel(int n, const double* __restrict__ table, const double* __restrict__ u,
                        double* out, double* gscratch, size_t gstride)
{
  extern __shared__ __align__(16) double dsm_[];
  const int N = n + 1;
  double* dsm = gscratch ? gscratch + (size_t)blockIdx.x * gstride : dsm_;
  double* ext = dsm;
  double* su = dsm + ext4_doubles(n);
  ext4_build(table, n, ext);
  for (int k = threadIdx.x; k < N; k += blockDim.x) su[k] = u[(size_t)blockIdx.x * N + k];
  __syncthreads();
  toeplitz_conv(su, ext, n, -1.0 / 3.141592653589793, out + (size_t)blockIdx.x * N);
}
}  // namespace paqif

extern "C" int paqif_line_deformation(int64_t B, int64_t n, const double* table, const double* u,
                                      double* out, void* stream)
{
  if (B < 0 || n < 1) return set_arg_error("line_deformation: bad sizes");
  if (B == 0) return PAQIF_OK;
  const size_t smem = (size_t)(ext4_doubles((int)n) + n + 1 + 8) * 8;
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 227 * 1024) {  // too fine for shared memory: the arrays in HBM
    const size_t stride = ((smem / 8) + 31) & ~(size_t)31;
    double* g = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&g, (size_t)B * stride * 8, st);
    if (e != cudaSuccess) return set_cuda_error("line_deformation: scratch", e);
    line_deformation_kernel<<<(unsigned)B, kEhlThreads, 0, st>>>((int)n, table, u, out, g, stride);
    cudaFreeAsync(g, st);
    return check_launch("paqif_line_deformation");
  }
  cudaFuncSetAttribute(line_deformation_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  line_deformation_kernel<<<(unsigned)B, kEhlThreads, smem, st>>>((int)n, table, u, out, nullptr, 0);
  return check_launch("paqif_line_deformation");
}

extern "C" int paqif_ehl_line_residual(const paqif_ehl_line_cfg* cfg, int64_t B,
                                       const double* table, const double* p_hertz,
                                       const double* lam, const double* u, const double* h0,
                                       double* film, double* res, void* stream)
{
  if (!cfg || B < 0 || cfg->n < 4 || !res) return set_arg_error("ehl_line_residual: bad args");
  if (B == 0) return PAQIF_OK;
  const EhlSmemLayout L(cfg->n);
  const size_t smem = (size_t)L.band * 8;  // the arrays; no line system here
  cudaStream_t st = (cudaStream_t)stream;
  if (smem > 227 * 1024) {  // too fine for shared memory: the arrays in HBM
    const size_t stride = ((size_t)L.band + 31) & ~(size_t)31;
    double* g = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&g, (size_t)B * stride * 8, st);
    if (e != cudaSuccess) return set_cuda_error("ehl_line_residual: scratch", e);
    ehl_line_residual_kernel<<<(unsigned)B, kEhlThreads, 0, st>>>(*cfg, B, table, p_hertz, lam,
                                                                   u, h0, film, res, g, stride);
    cudaFreeAsync(g, st);
    return check_launch("paqif_ehl_line_residual");
  }
  cudaFuncSetAttribute(ehl_line_residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  ehl_line_residual_kernel<<<(unsigned)B, kEhlThreads, smem, st>>>(
      *cfg, B, table, p_hertz, lam, u, h0, film, res, nullptr, 0);
  return check_launch("paqif_ehl_line_residual");
}
