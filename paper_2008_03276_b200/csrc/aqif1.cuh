// Latency-first AQIF for the tridiagonal (beta = 1) column systems of the
// point contact's column_sweep (ehl/sweeps.py:421-518 builds them from the
// offsets {-1, 0, 1}, so the reference factors them with beta = 1).
//
// Same design as aqif2.cuh, one wing row per side: lane parity = side, the
// wing row (pr + dir) becomes the next level's pivot row every level and
// the lane then takes the row entering the wing (pr + 2 dir).  Rows are an
// "own" window (columns pr, pr + dir) and a "cross" window (anti-band fill,
// columns other, other - dir).  The pivot rows of a level are the level's
// record in shared memory.  Arithmetic: the reference recurrence
// (paqif/_kernels.py:62-225) at beta = 1 in the reference's operation order
// -- bit for bit in EXACT mode identical to the general warp engine
// (aqif_factor_group / zsolve_group with BETA = 1, tools/aqif1_check.cu).
//
// Record of level k (12 doubles): P_t.L[0..1], P_t.R[0..1], P_b.L[0..1],
// P_b.R[0..1], y_t, y_b, det, 1/det; after the Z solve y_t, y_b hold
// (x[p], x[n-1-p]) of that level.
#pragma once
#include "aqif2.cuh"

namespace paqif {

constexpr int kRec1 = 12;

// Band storage: diagonal-major, kBandPad zero entries before and after every
// diagonal and around the right side:
//   A(i, i + d) = band[(d + 1) * aqif1_stride(n) + kBandPad + i],  |d| <= 1
//   f(i)        = rhs[kBandPad + i]
__host__ __device__ constexpr int aqif1_stride(int n) { return n + 2 * kBandPad; }
__host__ __device__ constexpr size_t aqif1_band_doubles(int n) { return 3 * (size_t)aqif1_stride(n); }
__host__ __device__ constexpr size_t aqif1_rhs_doubles(int n) { return (size_t)aqif1_stride(n); }
__host__ __device__ constexpr size_t aqif1_rec_doubles(int n) { return (size_t)(n / 2 + 1) * kRec1; }
__device__ __forceinline__ double& band1_ref(double* band, int n, int i, int d) {
  return band[(d + 1) * aqif1_stride(n) + kBandPad + i];
}
__device__ __forceinline__ double band1_at(const double* __restrict__ band, int n, int i, int j) {
  const int d = j - i;
  const bool in = (unsigned)i < (unsigned)n && (unsigned)j < (unsigned)n && d >= -1 && d <= 1;
  return in ? band[(d + 1) * aqif1_stride(n) + kBandPad + i] : 0.0;
}
__device__ __forceinline__ double band1_pad(const double* __restrict__ band, int n, int i, int j) {
  return band[(j - i + 1) * aqif1_stride(n) + kBandPad + i];
}
__device__ __forceinline__ void aqif1_zero_pads(double* band, double* rhs, int n) {
  const int S = aqif1_stride(n);
  for (int idx = threadIdx.x; idx < 4 * 2 * kBandPad; idx += blockDim.x) {
    const int row = idx / (2 * kBandPad), q = idx % (2 * kBandPad);
    const int col = q < kBandPad ? q : kBandPad + n + (q - kBandPad);
    if (row < 3) band[row * S + col] = 0.0;
    else rhs[col] = 0.0;
  }
}

// Factor + fused W solve; all 32 lanes of one converged warp call (lanes
// >= 2 duplicate lanes 0-1).  Breakdown is tested afterwards
// (aqif1_breakdown).  CHECKED as in aqif2_factor.
template <bool EXACT, bool CHECKED>
__device__ bool aqif1_factor(const double* __restrict__ band, const double* __restrict__ rhs,
                             int n, double* rec, int lane_id) {
  using A = Arith<EXACT>;
  const int side = lane_id & 1;
  const bool writer = lane_id < 2;
  const int s = n / 2;
  const int dir = side ? 1 : -1;
  const int own_off = side ? 6 : 0, crs_off = side ? 4 : 2;
  const int oth_own = side ? 2 : 4, oth_crs = side ? 0 : 6;  // other pivot row, my orientation
  int pr = side ? s : s - 1;  // this side's pivot row at the current level
  int row = pr + dir;         // the wing row
  double wo[2], wc[2], rh;
  {
    const int other = n - 1 - pr;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      wo[e] = band1_at(band, n, row, pr + e * dir);
      wc[e] = band1_at(band, n, row, other - e * dir);
    }
    rh = (unsigned)row < (unsigned)n ? rhs[kBandPad + row] : 0.0;
    if (writer) {  // level-1 record: the two middle rows
      double* r1 = rec + kRec1;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        r1[own_off + e] = band1_at(band, n, pr, pr + e * dir);
        r1[crs_off + e] = band1_at(band, n, pr, other - e * dir);
      }
      r1[8 + side] = rhs[kBandPad + pr];
    }
  }
  __syncwarp();
  bool safe = true;
  for (int k = 1; k <= s; ++k) {
    // ---- band loads for the hand-off at the end of this level
    const int q2 = pr + 2 * dir;                       // row entering the wing
    const double ncol = band1_pad(band, n, row, q2);   // my row's new own column
    const double fresh0 = band1_pad(band, n, q2, pr + dir);
    const double fresh1 = band1_pad(band, n, q2, q2);
    const double frh = rhs[kBandPad + q2];
    // ---- this level's pivot rows (record k)
    double* rk = rec + (size_t)k * kRec1;
    const double po0 = rk[own_off], po1 = rk[own_off + 1];
    const double pc0 = rk[crs_off], pc1 = rk[crs_off + 1];
    const double oo0 = rk[oth_own], oo1 = rk[oth_own + 1];
    const double oc0 = rk[oth_crs], oc1 = rk[oth_crs + 1];
    const double ym = rk[8 + side], yo = rk[9 - side];
    // pivot block at fixed slots for both sides (uniform loads)
    const double a11 = rk[0], a12 = rk[2], a21 = rk[4], a22 = rk[6];
    const double det = A::det2(a11, a22, a21, a12);
    const double y = __drcp_rn(det);
    if (lane_id == 0) {
      rk[10] = det;
      rk[11] = y;
    }
    if (k == s) break;
    // ---- the wing row: multipliers, update, right side
    const double nm = A::det2(oc0, wo[0], oo0, wc[0]);
    const double no = A::det2(po0, wc[0], pc0, wo[0]);
    const bool ds = exp_safe(det);
    safe = safe & ds;
    const double wm = level_div<EXACT, CHECKED>(nm, det, y, ds, safe);
    const double wx = level_div<EXACT, CHECKED>(no, det, y, ds, safe);
    const bool ok = (unsigned)row < (unsigned)n;
    const bool up = ok & !(is_zero(wm) & is_zero(wx));  // bitwise: no branches
    const double u1 = A::rank2(wo[1], wm, po1, wx, oo1);
    const double v1 = A::rank2(wc[1], wm, pc1, wx, oc1);
    const double rr = A::sub(rh, A::add(A::mul(ym, wm), A::mul(yo, wx)));
    // ---- it is the next pivot row: publish as record k+1 ...
    double* rn = rk + kRec1;
    if (writer) {
      rn[own_off] = up ? u1 : wo[1];
      rn[own_off + 1] = ok ? ncol : 0.0;
      rn[crs_off] = up ? v1 : wc[1];
      rn[crs_off + 1] = 0.0;
      rn[8 + side] = ok ? rr : rh;
    }
    // ... and take the entering row
    wo[0] = fresh0;
    wo[1] = fresh1;
    wc[0] = 0.0;
    wc[1] = 0.0;
    rh = frh;
    row = q2;
    pr += dir;
    __syncwarp();
  }
  return EXACT && !CHECKED ? __all_sync(0xffffffffu, safe) : true;
}

// Outside-in Z solve from the records; all 32 lanes compute the same chain,
// lane 0 stores (x[p], x[n-1-p]) over (y_t, y_b) of the record it came from.
template <bool EXACT, bool CHECKED>
__device__ bool aqif1_zsolve(double* rec_, int n, int lane_id) {
  using A = Arith<EXACT>;
  const int s = n / 2;
  int z0;  // opaque zero: keeps the chain out of the uniform datapath
  asm volatile("mov.u32 %0, 0;" : "=r"(z0));
  double* rec = rec_ + z0;
  double xl = 0.0, xr = 0.0;  // x[p-1], x[q+1]
  bool safe = true;
  // reference term order (zsolve_group, t = 0): left term, then right term
  auto level = [&](int p, bool lead) {
    const double2* c2 = reinterpret_cast<const double2*>(rec + (size_t)(s - p) * kRec1);
    const double2 r0 = c2[0], r1 = c2[1], r2 = c2[2], r3 = c2[3], r4 = c2[4], r5 = c2[5];
    // r0 = P_t.L, r1 = P_t.R, r2 = P_b.L, r3 = P_b.R, r4 = (y_t, y_b), r5 = (det, 1/det)
    double at = r4.x, ab = r4.y;
    if (lead) {
      at = A::axpy_neg(at, r0.y, xl);
      ab = A::axpy_neg(ab, r2.y, xl);
      at = A::axpy_neg(at, r1.y, xr);
      ab = A::axpy_neg(ab, r3.y, xr);
    }
    const double a11 = r0.x, a12 = r1.x, a21 = r2.x, a22 = r3.x;
    const double det = r5.x, y = r5.y;
    const bool ds = exp_safe(det);
    safe = safe & ds;
    const double xp = level_div<EXACT, CHECKED>(A::det2(a22, at, a12, ab), det, y, ds, safe);
    const double xq = level_div<EXACT, CHECKED>(A::det2(a11, ab, a21, at), det, y, ds, safe);
    if (lane_id == 0) {
      double* c = rec + (size_t)(s - p) * kRec1;
      c[8] = xp;
      c[9] = xq;
    }
    xl = xp;
    xr = xq;
  };
  if (s >= 1) level(0, false);
#pragma unroll 2
  for (int p = 1; p < s; ++p) level(p, true);
  return EXACT && !CHECKED ? __all_sync(0xffffffffu, safe) : true;
}

__device__ __forceinline__ void aqif1_gather(const double* rec, int n, double* x, int lane_id) {
  const int s = n / 2;
  for (int p = lane_id; p < s; p += 32) {
    const double* c = rec + (size_t)(s - p) * kRec1;
    x[p] = c[8];
    x[n - 1 - p] = c[9];
  }
}

// breakdown of any level's pivot block (as aqif2_breakdown)
__device__ __forceinline__ bool aqif1_breakdown(const double* rec, int n, double tol, int lane_id) {
  const int s = n / 2;
  bool bad = false;
  for (int k = 1 + lane_id; k <= s; k += 32) {
    const double* c = rec + (size_t)k * kRec1;
    const double a11 = c[0], a12 = c[2], a21 = c[4], a22 = c[6], det = c[10];
    double scale = fabs(a11);
    if (fabs(a12) > scale) scale = fabs(a12);
    if (fabs(a21) > scale) scale = fabs(a21);
    if (fabs(a22) > scale) scale = fabs(a22);
    bad |= fabs(det) <= (k < s ? tol : 1e-14) * (scale * scale) + PAQIF_TINY;
  }
  return __any_sync(0xffffffffu, bad);
}

// Whole tridiagonal solve on warp 0 of a CTA; all threads of the CTA call.
// Returns bit 0 on a breakdown, bit 1 if the checked repeat ran.  x may
// alias band.
template <bool EXACT>
__device__ int aqif1_solve(const double* band, const double* rhs, int n, double* rec, double* x,
                           int* flag_smem) {
  __syncthreads();
  if (threadIdx.x < 32) {
    bool ok = aqif1_factor<EXACT, false>(band, rhs, n, rec, threadIdx.x);
    __syncwarp();
    bool bad = aqif1_breakdown(rec, n, 1e-14, threadIdx.x);
    // a certain breakdown (safe divisions) needs no Z solve
    if (!(ok & bad)) ok = aqif1_zsolve<EXACT, false>(rec, n, threadIdx.x) && ok;
    if (!ok) {  // a division left the Markstein range: exact slow path
      __syncwarp();
      aqif1_factor<EXACT, true>(band, rhs, n, rec, threadIdx.x);
      __syncwarp();
      bad = aqif1_breakdown(rec, n, 1e-14, threadIdx.x);
      aqif1_zsolve<EXACT, true>(rec, n, threadIdx.x);
    }
    __syncwarp();
    aqif1_gather(rec, n, x, threadIdx.x);
    if (threadIdx.x == 0) *flag_smem = (bad ? 1 : 0) | (ok ? 0 : 2);
  }
  __syncthreads();
  const int st = *flag_smem;
  __syncthreads();
  return st;
}

}  // namespace paqif
