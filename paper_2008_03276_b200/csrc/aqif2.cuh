// Latency-first AQIF for the pentadiagonal (beta = 2) EHL line systems.
//
// The EHL sweeps solve one line system at a time in Gauss-Seidel order, so a
// line solve is a pure dependency chain; the only parallelism is inside a
// level of the middle-out factorization.  Measured on B200, a single warp
// issues one fp64 instruction per ~3.5 cycles and __drcp_rn costs ~75, so a
// level's cost is its per-lane fp64 instruction count plus the
// det -> reciprocal -> multiplier -> update chain.  This engine therefore
// gives every wing row its own lane and keeps everything else off the
// level recurrence:
//
//   lane role r = lane & 3:  side = r >> 1 (0 top, 1 bottom), the two lanes
//   of a side hold the side's two wing rows (rt-1, rt-2 or rb+1, rb+2) and
//   swap "next pivot" / "far wing" roles every level.
//
// Rows are stored as an "own" window (the band side: columns rt, rt-1, rt-2
// for the top, rb, rb+1, rb+2 for the bottom) and a "cross" window
// (anti-band fill), so all lanes run one instruction stream.  The pivot
// rows of a level ARE the level's record in shared memory: the two
// next-pivot lanes write it, the warp syncs, every lane reads it.
// Breakdown (|det| <= tol*scale^2 + tiny) is tested after the factor and Z
// solve, in parallel over all records (any level breaking down fails the
// solve, exactly when the reference's factor or Z solve would raise).
//
// Arithmetic is the reference recurrence (paqif/_kernels.py:62-225) in the
// reference's operation order -- bit for bit in EXACT mode identical to
// aqif_factor_group + zsolve_group (tools/aqif2_check.cu).
//
// Record of level k (16 doubles): P_t.L[0..2], P_t.R[0..2], P_b.L[0..2],
// P_b.R[0..2], y_t, y_b, det, 1/det (RN reciprocal in EXACT mode).
#pragma once
#include "aqif_warp.cuh"

namespace paqif {

constexpr int kRec2 = 16;
// dev counters (-DPAQIF_DEV_PROF): [0..3] phase cycles, [4] solves,
// [5] factor levels, [6] levels with a numerator below the Markstein range
__device__ unsigned long long g_aqif2_prof[8];

// Band storage: diagonal-major with kBandPad zero entries before and after
// every diagonal (and around the right side), so the level loop reads rows
// up to 3 outside the matrix without a bounds test:
//   A(i, i + d) = band[(d + 2) * aqif2_stride(n) + kBandPad + i],  |d| <= 2
//   f(i)        = rhs[kBandPad + i]
// Entries whose column leaves the matrix are stored as exact zeros (the
// padded_bands semantics), so only the row needs the padding.
constexpr int kBandPad = 4;
__host__ __device__ constexpr int aqif2_stride(int n) { return n + 2 * kBandPad; }
__host__ __device__ constexpr size_t aqif2_band_doubles(int n) { return 5 * (size_t)aqif2_stride(n); }
__host__ __device__ constexpr size_t aqif2_rhs_doubles(int n) { return (size_t)aqif2_stride(n); }
__device__ __forceinline__ double& band2_ref(double* band, int n, int i, int d) {
  return band[(d + 2) * aqif2_stride(n) + kBandPad + i];
}
// checked access (setup only): zero outside the matrix and the band
__device__ __forceinline__ double band2_at(const double* __restrict__ band, int n, int i, int j) {
  const int d = j - i;
  const bool in = (unsigned)i < (unsigned)n && (unsigned)j < (unsigned)n && d >= -2 && d <= 2;
  return in ? band[(d + 2) * aqif2_stride(n) + kBandPad + i] : 0.0;
}
// unchecked access: |j - i| <= 2 and -kBandPad <= i < n + kBandPad
__device__ __forceinline__ double band2_pad(const double* __restrict__ band, int n, int i, int j) {
  return band[(j - i + 2) * aqif2_stride(n) + kBandPad + i];
}
// zero the pads of a band + right side (all threads of the CTA call)
__device__ __forceinline__ void aqif2_zero_pads(double* band, double* rhs, int n) {
  const int S = aqif2_stride(n);
  for (int idx = threadIdx.x; idx < 6 * 2 * kBandPad; idx += blockDim.x) {
    const int row = idx / (2 * kBandPad), q = idx % (2 * kBandPad);
    const int col = q < kBandPad ? q : kBandPad + n + (q - kBandPad);
    if (row < 5) band[row * S + col] = 0.0;
    else rhs[col] = 0.0;
  }
}

__device__ __forceinline__ double qdiv_rn(double a, double b, double y, bool b_safe) {
  if (b_safe && (exp_safe(a) || is_zero(a))) {
    const double q = __dmul_rn(a, y);
    const double r = fma(-q, b, a);
    return fma(r, y, q);
  }
  return __ddiv_rn(a, b);
}
template <bool EXACT, bool CHECKED>
__device__ __forceinline__ double level_div(double a, double b, double y, bool b_safe, bool& safe) {
  if (!EXACT) return a * y;
  if (CHECKED) return qdiv_rn(a, b, y, b_safe);
  return mdiv_fix(a, b, y, safe);
}

// Factor + fused W solve.  ALL 32 lanes of one converged warp call (a
// partial warp turns shuffles/syncs into divergent-collective slow paths);
// lanes >= 4 duplicate lanes 0-3 and store nothing.  rec: (n/2 + 1) * kRec2
// doubles.  Breakdown is NOT tested here (aqif2_breakdown).  CHECKED=false:
// branch-free divisions; returns false (on all lanes) if any was outside the
// Markstein range -- redo with CHECKED=true.
template <bool EXACT, bool CHECKED>
__device__ bool aqif2_factor(const double* __restrict__ band, const double* __restrict__ rhs,
                             int n, double* rec, int lane_id) {
  using A = Arith<EXACT>;
  const int r = lane_id & 3;
  const int side = r >> 1;
  const bool writer = lane_id < 4;
  const int s = n / 2;
  const int dir = side ? 1 : -1;
  const int own_off = side ? 9 : 0, crs_off = side ? 6 : 3;
  const int oth_own = side ? 3 : 6, oth_crs = side ? 0 : 9;  // other pivot row, my orientation
  int pr = side ? s : s - 1;  // this side's pivot row at the current level
  // which wing this lane holds at level 1: r&1 == 0 -> row pr+dir (next pivot)
  int row = pr + dir * (1 + (r & 1));
  double wo[3], wc[3], rh;
  {
    const int other = n - 1 - pr;
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      wo[e] = band2_at(band, n, row, pr + e * dir);
      wc[e] = band2_at(band, n, row, other - e * dir);
    }
    rh = (unsigned)row < (unsigned)n ? rhs[kBandPad + row] : 0.0;
    // level-1 record: the two middle rows (one writer lane per side)
    if (writer && (r & 1) == 0) {
      double* r1 = rec + kRec2;
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        r1[own_off + e] = band2_at(band, n, pr, pr + e * dir);
        r1[crs_off + e] = band2_at(band, n, pr, other - e * dir);
      }
      r1[12 + side] = rhs[kBandPad + pr];
    }
  }
  __syncwarp();
  bool safe = true;
  for (int k = 1; k <= s; ++k) {
    const bool nxt = ((r ^ (k - 1)) & 1) == 0;  // my row is the next pivot
    // ---- band loads for the shift at the end of this level
    const int q3 = pr + 3 * dir;                   // row entering the wing
    const double ncol = band2_pad(band, n, row, q3);  // my row's new own column
    double fresh[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) fresh[e] = band2_pad(band, n, q3, pr + dir + e * dir);
    const double frh = rhs[kBandPad + q3];
    // ---- this level's pivot rows (record k)
    double* rk = rec + (size_t)k * kRec2;
    double po[3], pc[3], oo[3], oc[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      po[e] = rk[own_off + e];
      pc[e] = rk[crs_off + e];
      oo[e] = rk[oth_own + e];
      oc[e] = rk[oth_crs + e];
    }
    const double ym = rk[12 + side], yo = rk[13 - side];
    // the pivot block sits at fixed record slots for both sides (uniform
    // loads instead of side selects)
    const double a11 = rk[0], a12 = rk[3], a21 = rk[6], a22 = rk[9];
    const double det = A::det2(a11, a22, a21, a12);
    const double y = __drcp_rn(det);  // fast mode multiplies by it
    if (lane_id == 0) {
      rk[14] = det;
      rk[15] = y;
    }
    if (k == s) break;
    // ---- my wing row: multipliers (wm for my side's pivot row, wo for the
    // other's; w1/w2 by side), updates, right side
    const double nm = A::det2(oc[0], wo[0], oo[0], wc[0]);
    const double no = A::det2(po[0], wc[0], pc[0], wo[0]);
    const bool ds = exp_safe(det);
    safe = safe & ds;
    const double wm = level_div<EXACT, CHECKED>(nm, det, y, ds, safe);
    const double wx = level_div<EXACT, CHECKED>(no, det, y, ds, safe);
#ifdef PAQIF_DEV_PROF
    {
      const unsigned em = ((unsigned)__double2hiint(nm) >> 20) & 0x7ffu;
      const unsigned ex = ((unsigned)__double2hiint(no) >> 20) & 0x7ffu;
      const bool any_tiny = __any_sync(0xffffffffu, (em < 524u) | (ex < 524u));
      if (lane_id == 0) {
        atomicAdd(&g_aqif2_prof[5], 1ull);
        if (any_tiny) atomicAdd(&g_aqif2_prof[6], 1ull);
      }
    }
#endif
    const bool ok = (unsigned)row < (unsigned)n;
    const bool up = ok & !(is_zero(wm) & is_zero(wx));  // bitwise: no branches
    const double u1 = A::rank2(wo[1], wm, po[1], wx, oo[1]);
    const double u2 = A::rank2(wo[2], wm, po[2], wx, oo[2]);
    const double v1 = A::rank2(wc[1], wm, pc[1], wx, oc[1]);
    const double v2 = A::rank2(wc[2], wm, pc[2], wx, oc[2]);
    const double rr = A::sub(rh, A::add(A::mul(ym, wm), A::mul(yo, wx)));
    // shifted row (windows of the next level)
    wo[0] = up ? u1 : wo[1];
    wo[1] = up ? u2 : wo[2];
    wo[2] = ok ? ncol : 0.0;
    wc[0] = up ? v1 : wc[1];
    wc[1] = up ? v2 : wc[2];
    wc[2] = 0.0;
    rh = ok ? rr : rh;
    // ---- next pivot: publish as record k+1, then take the entering row
    double* rn = rk + kRec2;
    if (writer & nxt) {
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        rn[own_off + e] = wo[e];
        rn[crs_off + e] = wc[e];
      }
      rn[12 + side] = rh;
    }
    if (nxt) {
#pragma unroll
      for (int e = 0; e < 3; ++e) {
        wo[e] = fresh[e];
        wc[e] = 0.0;
      }
      rh = frh;
      row = q3;
    }
    pr += dir;
    __syncwarp();
  }
  return EXACT && !CHECKED ? __all_sync(0xffffffffu, safe) : true;
}

// Outside-in Z solve from the records.  All 32 lanes of one converged warp
// call and compute the same chain; lane 0 stores the pair (x[p], x[n-1-p])
// over (y_t, y_b) of the record it came from (so x may later overwrite the
// band, which a CHECKED repeat still needs; aqif2_gather copies it out).
// CHECKED as for the factor (returns false if an unchecked division was
// outside the Markstein range).
template <bool EXACT, bool CHECKED>
__device__ bool aqif2_zsolve(double* rec_, int n, int lane_id) {
  using A = Arith<EXACT>;
  const int s = n / 2;
  // opaque zero: keeps the chain out of the uniform datapath
  int z0;
  asm volatile("mov.u32 %0, 0;" : "=r"(z0));
  double* rec = rec_ + z0;
  double xl0 = 0.0, xl1 = 0.0;  // x[p-2], x[p-1]
  double xr0 = 0.0, xr1 = 0.0;  // x[q+1], x[q+2]
  bool safe = true;
  // one level; FIRST = number of leading terms skipped for p < 2
  // (zsolve_group's term order, out-of-range columns skipped)
  auto level = [&](int p, int lead) {
    double* c = rec + (size_t)(s - p) * kRec2;
    double at = c[12], ab = c[13];
    if (lead >= 2) {
      at = A::axpy_neg(at, c[2], xl0);
      ab = A::axpy_neg(ab, c[8], xl0);
    }
    if (lead >= 1) {
      at = A::axpy_neg(at, c[4], xr0);
      ab = A::axpy_neg(ab, c[10], xr0);
      at = A::axpy_neg(at, c[1], xl1);
      ab = A::axpy_neg(ab, c[7], xl1);
    }
    if (lead >= 2) {
      at = A::axpy_neg(at, c[5], xr1);
      ab = A::axpy_neg(ab, c[11], xr1);
    }
    const double a11 = c[0], a12 = c[3], a21 = c[6], a22 = c[9];
    const double det = c[14], y = c[15];
    const bool ds = exp_safe(det);
    safe = safe & ds;
    const double xp = level_div<EXACT, CHECKED>(A::det2(a22, at, a12, ab), det, y, ds, safe);
    const double xq = level_div<EXACT, CHECKED>(A::det2(a11, ab, a21, at), det, y, ds, safe);
    if (lane_id == 0) {  // the record's y_t, y_b were read above (same warp instruction stream)
      c[12] = xp;
      c[13] = xq;
    }
    xl0 = xl1;
    xl1 = xp;
    xr1 = xr0;
    xr0 = xq;
  };
  if (s >= 1) level(0, 0);
  if (s >= 2) level(1, 1);
#pragma unroll 2
  for (int p = 2; p < s; ++p) level(p, 2);
  return EXACT && !CHECKED ? __all_sync(0xffffffffu, safe) : true;
}

// x[p] = record(s-p).y_t, x[n-1-p] = record(s-p).y_b after aqif2_zsolve.
__device__ __forceinline__ void aqif2_gather(const double* rec, int n, double* x, int lane_id) {
  const int s = n / 2;
  for (int p = lane_id; p < s; p += 32) {
    const double* c = rec + (size_t)(s - p) * kRec2;
    x[p] = c[12];
    x[n - 1 - p] = c[13];
  }
}

// Breakdown test of every level's pivot block (factor levels 1..s-1 with
// tol, Z levels 1..s with 1e-14; the line solves use tol = 1e-14).  All 32
// lanes call; returns true (on all lanes) if any level breaks down.
__device__ __forceinline__ bool aqif2_breakdown(const double* rec, int n, double tol,
                                                int lane_id) {
  const int s = n / 2;
  bool bad = false;
  for (int k = 1 + lane_id; k <= s; k += 32) {
    const double* c = rec + (size_t)k * kRec2;
    const double a11 = c[0], a12 = c[3], a21 = c[6], a22 = c[9], det = c[14];
    double scale = fabs(a11);
    if (fabs(a12) > scale) scale = fabs(a12);
    if (fabs(a21) > scale) scale = fabs(a21);
    if (fabs(a22) > scale) scale = fabs(a22);
    bad |= fabs(det) <= (k < s ? tol : 1e-14) * (scale * scale) + PAQIF_TINY;
  }
  return __any_sync(0xffffffffu, bad);
}

// Whole line solve on warp 0 of a CTA; all threads of the CTA call.
// band/rhs/x/rec in shared memory (x may alias band).  Returns bit 0 set on a
// breakdown (the reference's FactorizationBreakdownError), bit 1 if the
// checked repeat ran.
// dev phase counters (cycles: factor, breakdown, z, gather; count), per TU;
// only with -DPAQIF_DEV_PROF (PAQIF_NVCC_EXTRA), read by PAQIF_PT_PROF=1
#ifdef PAQIF_DEV_PROF
#define AQ2_T(v) const long long v = clock64()
#else
#define AQ2_T(v)
#endif

template <bool EXACT>
__device__ int aqif2_solve(const double* band, const double* rhs, int n, double* rec, double* x,
                           int* flag_smem) {
  __syncthreads();
  if (threadIdx.x < 32) {
    AQ2_T(c0);
    bool ok = aqif2_factor<EXACT, false>(band, rhs, n, rec, threadIdx.x);
    __syncwarp();
    AQ2_T(c1);
    const bool bad0 = aqif2_breakdown(rec, n, 1e-14, threadIdx.x);
    AQ2_T(c2);
    // a certain breakdown (safe divisions) needs no Z solve: the caller
    // discards the solution and tries the next rung
    if (!(ok & bad0)) ok = aqif2_zsolve<EXACT, false>(rec, n, threadIdx.x) && ok;
    AQ2_T(c3);
    bool bad = bad0;
    if (!ok) {  // a division left the Markstein range: exact slow path
      __syncwarp();
      aqif2_factor<EXACT, true>(band, rhs, n, rec, threadIdx.x);
      __syncwarp();
      bad = aqif2_breakdown(rec, n, 1e-14, threadIdx.x);
      aqif2_zsolve<EXACT, true>(rec, n, threadIdx.x);
    }
    __syncwarp();
    aqif2_gather(rec, n, x, threadIdx.x);
    if (threadIdx.x == 0) {
      *flag_smem = (bad ? 1 : 0) | (ok ? 0 : 2);
#ifdef PAQIF_DEV_PROF
      const long long c4 = clock64();
      atomicAdd(&g_aqif2_prof[0], (unsigned long long)(c1 - c0));
      atomicAdd(&g_aqif2_prof[1], (unsigned long long)(c2 - c1));
      atomicAdd(&g_aqif2_prof[2], (unsigned long long)(c3 - c2));
      atomicAdd(&g_aqif2_prof[3], (unsigned long long)(c4 - c3));
      atomicAdd(&g_aqif2_prof[4], 1ull);
#endif
    }
  }
  __syncthreads();
  const int st = *flag_smem;
  __syncthreads();
  return st;
}

}  // namespace paqif
