// Outside-in Z solve for one system per lane group, reading the per-level
// pivot records (PivotLayout, written by aqif_factor_group's policy) back
// through a double-buffered cp.async ring in shared memory.  Lane 0 of the
// group carries the top (row p) chain, lane 1 the bottom (row q) chain, in
// the reference's operation order (solve_z_batch, paqif/_kernels.py:175-225).
//
//   FULL = false: solve_z(start_level = BETA+1) -- the PAQIF middles after
//                 the corner system (parallel.py:234-258); x[0..BETA) and
//                 x[n-BETA..n) are prefilled.
//   FULL = true : solve_z(start_level = 1) -- a plain AQIF solve (the EHL
//                 line solves, ehl/sweeps.py:270-273).
#pragma once
#include <type_traits>
#include "aqif_warp.cuh"

namespace paqif {

constexpr int kZPrefetch = 4;  // record chunks prefetched into L2 ahead of the ring

template <int BETA>
struct ZChunk {
#ifndef PAQIF_ZCHUNK
#define PAQIF_ZCHUNK 8
#endif
  static constexpr int ZC = BETA * ((PAQIF_ZCHUNK + BETA - 1) / BETA);  // levels per chunk, multiple of BETA
  static constexpr int kRing = 2 * ZC * PivotLayout<BETA>::kSize;  // doubles
};

// One level of the chains; CHECK enables the boundary skips of the first
// BETA levels of a full solve.  Returns false on breakdown.
template <int BETA, bool EXACT, bool CHECK>
__device__ __forceinline__ bool zlevel(const double* rec, int sd, int p, int n, double& xp,
                                       double& xq, const double* xl, const double* xr, int ph,
                                       unsigned pair)
{
  using A = Arith<EXACT>;
  using PL = PivotLayout<BETA>;
  const int q = n - 1 - p;
  // the 2x2 pivot, its determinant, reciprocal and breakdown test depend on
  // the record only: issued first, they run under the right side's chain
  const double a11 = rec[PL::zi(0, 0, 0)], a12 = rec[PL::zi(1, 0, 0)];
  const double a21 = rec[PL::zi(0, 0, 1)], a22 = rec[PL::zi(1, 0, 1)];
  const double det = A::det2(a11, a22, a12, a21);
  double scale = fabs(a11);
  if (fabs(a12) > scale) scale = fabs(a12);
  if (fabs(a21) > scale) scale = fabs(a21);
  if (fabs(a22) > scale) scale = fabs(a22);
  const bool bad = fabs(det) <= 1e-14 * (scale * scale) + PAQIF_TINY;
  const double y = __drcp_rn(det);  // RN(1/det), either arithmetic
  double acc = rec[sd == 0 ? PL::kYT : PL::kYB];
  if (EXACT) {
    // reference order: t = 0..BETA-1, left term then right term
#pragma unroll
    for (int t = 0; t < BETA; ++t) {
      if (!CHECK || p - BETA + t >= 0)
        acc = A::axpy_neg(acc, rec[PL::zi(0, BETA - t, 0) + sd], xl[(ph + t) % BETA]);
      if (!CHECK || q + 1 + t < n)
        acc = A::axpy_neg(acc, rec[PL::zi(1, 1 + t, 0) + sd],
                          xr[(ph - 1 - t + 2 * BETA) % BETA]);
    }
  } else {
    // FMA arithmetic: the terms of the older unknowns first, in two
    // independent partial sums (left / right window), the two that the
    // previous level just produced (x[p-1], x[q+1]) last, so only two FMAs
    // wait on the previous level and the older terms' chain is half as long
    double accr = 0.0;
#pragma unroll
    for (int t = 0; t < BETA; ++t) {
      if (t != BETA - 1 && (!CHECK || p - BETA + t >= 0))
        acc = A::axpy_neg(acc, rec[PL::zi(0, BETA - t, 0) + sd], xl[(ph + t) % BETA]);
      if (t != 0 && (!CHECK || q + 1 + t < n))
        accr = A::axpy_neg(accr, rec[PL::zi(1, 1 + t, 0) + sd],
                           xr[(ph - 1 - t + 2 * BETA) % BETA]);
    }
    acc = acc + accr;
    if (!CHECK || q + 1 < n)
      acc = A::axpy_neg(acc, rec[PL::zi(1, 1, 0) + sd], xr[(ph - 1 + 2 * BETA) % BETA]);
    if (!CHECK || p - 1 >= 0)
      acc = A::axpy_neg(acc, rec[PL::zi(0, 1, 0) + sd], xl[(ph + BETA - 1) % BETA]);
  }
  const double oth = __shfl_xor_sync(pair, acc, 1);
  const double rt = sd == 0 ? acc : oth;
  const double rb = sd == 0 ? oth : acc;
  // no branch on the test: the quotients are computed either way (garbage
  // after a breakdown, which the caller discards) and the flag returned
  if (EXACT) {
    const bool ds = div_safe(det);
    xp = div_rn(A::det2(a22, rt, a12, rb), det, y, ds);
    xq = div_rn(A::det2(a11, rb, a21, rt), det, y, ds);
  } else {
    xp = (a22 * rt - a12 * rb) * y;
    xq = (a11 * rb - a21 * rt) * y;
  }
  return !bad;
}

// FMA arithmetic, both rows of a level in one lane: the two chain lanes
// compute the same pair (no shuffle on the level chain).  Per row the same
// expressions as zlevel's FMA branch; the record's (top, bottom) entries of
// one column are adjacent, so each 16-byte load serves both rows.
template <int BETA, bool CHECK>
__device__ __forceinline__ bool zlevel_fma2(const double* rec, int p, int n, double& xp,
                                            double& xq, const double* xl, const double* xr,
                                            int ph)
{
  using A = Arith<false>;
  using PL = PivotLayout<BETA>;
  const int q = n - 1 - p;
  const double2* r2 = reinterpret_cast<const double2*>(rec);
  const double2 c0 = r2[PL::zi(0, 0, 0) / 2];  // (a11, a21)
  const double2 c1 = r2[PL::zi(1, 0, 0) / 2];  // (a12, a22)
  const double a11 = c0.x, a21 = c0.y, a12 = c1.x, a22 = c1.y;
  const double det = A::det2(a11, a22, a12, a21);
  double scale = fabs(a11);
  if (fabs(a12) > scale) scale = fabs(a12);
  if (fabs(a21) > scale) scale = fabs(a21);
  if (fabs(a22) > scale) scale = fabs(a22);
  const bool bad = fabs(det) <= 1e-14 * (scale * scale) + PAQIF_TINY;
  // branch-free: a det outside the normal range fails the test above
  const double y = rcp_nobranch(det);
  const double2 yy = r2[PL::kYT / 2];
  // both partial sums run oldest unknown first (left: x[p-BETA] .. x[p-2];
  // right: x[q+BETA] .. x[q+2]), so only their last terms wait for the pair
  // solved two levels ago (the pair of the previous level enters after)
  double acc_t = yy.x, acc_b = yy.y, accr_t = 0.0, accr_b = 0.0;
#pragma unroll
  for (int t = 0; t < BETA; ++t) {
    if (t != BETA - 1 && (!CHECK || p - BETA + t >= 0)) {
      const double2 z = r2[PL::zi(0, BETA - t, 0) / 2];
      const double xv = xl[(ph + t) % BETA];
      acc_t = A::axpy_neg(acc_t, z.x, xv);
      acc_b = A::axpy_neg(acc_b, z.y, xv);
    }
    const int tr = BETA - 1 - t;  // BETA-1 .. 0 (term tr = 0 is the newest: last, below)
    if (tr != 0 && (!CHECK || q + 1 + tr < n)) {
      const double2 z = r2[PL::zi(1, 1 + tr, 0) / 2];
      const double xv = xr[(ph - 1 - tr + 2 * BETA) % BETA];
      accr_t = A::axpy_neg(accr_t, z.x, xv);
      accr_b = A::axpy_neg(accr_b, z.y, xv);
    }
  }
  acc_t = acc_t + accr_t;
  acc_b = acc_b + accr_b;
  if (!CHECK || q + 1 < n) {
    const double2 z = r2[PL::zi(1, 1, 0) / 2];
    const double xv = xr[(ph - 1 + 2 * BETA) % BETA];
    acc_t = A::axpy_neg(acc_t, z.x, xv);
    acc_b = A::axpy_neg(acc_b, z.y, xv);
  }
  if (!CHECK || p - 1 >= 0) {
    const double2 z = r2[PL::zi(0, 1, 0) / 2];
    const double xv = xl[(ph + BETA - 1) % BETA];
    acc_t = A::axpy_neg(acc_t, z.x, xv);
    acc_b = A::axpy_neg(acc_b, z.y, xv);
  }
  xp = fma_mult(a22, acc_t, a12, acc_b, y);
  xq = fma_mult(a11, acc_b, a21, acc_t, y);
  return !bad;
}

// All 32 lanes call.  Returns 0 or the 1-based breakdown level.
// SCAN: the level test is the FACTORIZATION's (policies with
// kDeferBreakdown): every level is solved (no early stop) and the return
// value is the smallest factor level k = s - p whose pivot fails the test
// (the Z solve's own test on the same record is the same test).
template <int BETA, bool EXACT, bool FULL, int G = Group<BETA>::G, bool SCAN = false>
__device__ int zsolve_group(const double* zs, int n, double* x, double* ring, int gl, bool alive)
{
  using PL = PivotLayout<BETA>;
  constexpr int ZC = ZChunk<BETA>::ZC;
  constexpr int RS = PL::kSize;
  const int s = n / 2;
  const int p0 = FULL ? 0 : BETA;  // first unknown pair solved
  const int M = s - p0;            // levels to solve
  const int sd = gl & 1;
  const unsigned pair = 0x3u << ((threadIdx.x & 31) & ~1);
  double xl[BETA], xr[BETA];
  if (alive && gl < 2) {
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      xl[j] = FULL ? 0.0 : x[j];
      xr[j] = FULL ? 0.0 : x[n - 1 - j];
    }
  }
  auto issue = [&](int c0, int buf) {
    if (alive) {
      const int k_hi = s - p0 - c0;
      const int k_lo = max(1, k_hi - ZC + 1);
      const int pieces = (k_hi - k_lo + 1) * RS / 2;
      const double* src = zs + (size_t)k_lo * RS;
      double* dst = ring + buf * ZC * RS;
      for (int q = gl; q < pieces; q += G) cp_async16(dst + 2 * q, src + 2 * q);
      // the records a few chunks further down the stack into L2 (written
      // by the factorization long ago: typically evicted to HBM)
      const int k_pf = k_lo - (kZPrefetch - 1) * ZC;
      if (gl == 0 && k_pf >= 1)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(zs + (size_t)k_pf * RS),
                     "r"((unsigned)(ZC * RS * 8))
                     : "memory");
    }
    cp_async_commit();
  };
  int status = 0;
  auto chunk = [&](const double* buf, int k_lo, int c0, auto LAST) {
#pragma unroll
    for (int ph = 0; ph < ZC; ++ph) {
      const int p = p0 + c0 + ph;
      if (decltype(LAST)::value && p >= s) break;
      const double* rec = buf + (s - p - k_lo) * RS;
      double xp, xq;
      bool ok;
      if constexpr (EXACT)
        ok = (FULL && p < BETA)
                 ? zlevel<BETA, EXACT, true>(rec, sd, p, n, xp, xq, xl, xr, ph, pair)
                 : zlevel<BETA, EXACT, false>(rec, sd, p, n, xp, xq, xl, xr, ph, pair);
      else
        ok = (FULL && p < BETA) ? zlevel_fma2<BETA, true>(rec, p, n, xp, xq, xl, xr, ph)
                                : zlevel_fma2<BETA, false>(rec, p, n, xp, xq, xl, xr, ph);
      if (SCAN)
        status = ok ? status : s - p;  // ascending p: the last one is the smallest level
      else
        status = (!ok & (status == 0)) ? p + 1 : status;  // first failing level, no branch
      x[sd == 0 ? p : n - 1 - p] = sd == 0 ? xp : xq;
      xl[ph % BETA] = xp;
      xr[ph % BETA] = xq;
    }
  };
  if (M > 0) issue(0, 0);
  for (int c0 = 0, cb = 0; c0 < M; c0 += ZC, cb ^= 1) {
    if (c0 + ZC < M) {
      issue(c0 + ZC, cb ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    if (alive && gl < 2 && (SCAN || status == 0)) {
      const int k_hi = s - p0 - c0;
      const int k_lo = max(1, k_hi - ZC + 1);
      const double* buf = ring + cb * ZC * RS;
      // a full chunk runs its ZC levels as one straight-line block (no
      // per-level exit test, so the next level's loads and older terms
      // interleave with this level's chain); the last chunk checks
      if (c0 + ZC <= M) chunk(buf, k_lo, c0, std::false_type{});
      else chunk(buf, k_lo, c0, std::true_type{});
    }
    if (!SCAN) {
      // group-uniform status (lane 0 of the group holds it)
      status = __shfl_sync(0xffffffffu, status, (threadIdx.x & 31) & ~(G - 1));
      if (__all_sync(0xffffffffu, status != 0 || !alive)) {
        cp_async_wait<0>();
        break;
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
  __syncwarp();
  if (SCAN) status = __shfl_sync(0xffffffffu, status, (threadIdx.x & 31) & ~(G - 1));
  return status;
}

}  // namespace paqif
