// TVD kappa-scheme line-splitting sweeps on the device (paqif/tvdcd.py:
// 449-489 sweep_splitting, variants Ls0 / Ls1 / Ls2; the paper's Sec. 6
// linear study).  One CTA runs a whole sweep: x-lines in lexicographic
// order (forward or backward), each line
//   r   = f[j] - L u (StencilOperator.apply_line, tvdcd.py:116-123)
//   sig = AQIF solve of the padded line matrix (tvdcd.py:424-446)
//   u[j] += omega * sig
// with the beta = 2 latency engine (aqif2.cuh; the tridiagonal Ls2 line
// stored with beta = 2 gives the same bits as beta = 1),
// then the residual field and sqrt(h^2 sum r^2) with numpy's pairwise
// summation order (ConvectionDiffusionProblem.residual_norm, tvdcd.py:
// 338-343).  Products and sums are rounded separately, as numpy's are.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "aqif2.cuh"
#include "capi_util.cuh"

extern "C" {
#include "../../include/paqif_tvd.h"
}

namespace paqif {

constexpr int kTvdThreads = 256;

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// (L u)[j, i] in StencilOperator.apply order: centre, x offsets, y offsets
__device__ __forceinline__ double apply_at(const paqif_tvd_problem& p, const double* uf, int j,
                                           int i) {
  const int W = p.nx + 4;
  const size_t k = (size_t)j * p.nx + i;
  const double* c = uf + (size_t)(2 + j) * W + 2 + i;
  const size_t plane = (size_t)p.nx * p.ny;
  double v = dmul(p.c0[k], c[0]);
  for (int t = 0; t < p.kx; ++t) v = dadd(v, dmul(p.cx[t * plane + k], c[p.ox[t]]));
  for (int t = 0; t < p.ky; ++t) v = dadd(v, dmul(p.cy[t * plane + k], c[(ptrdiff_t)p.oy[t] * W]));
  return v;
}

// (L u)[j, i] split around the term that reads row j + od (the line solved
// just before line j): the sum of the terms before it (returned) and the
// products after it (rest[], at most 3), so the line's right side can be
// finished with one product once that row is updated -- same order, same
// bits as apply_at.  dep < 0: no such term, everything summed.
__device__ __forceinline__ double apply_split(const paqif_tvd_problem& p, const double* uf, int j,
                                              int i, int dep, double* rest) {
  const int W = p.nx + 4;
  const size_t k = (size_t)j * p.nx + i;
  const double* c = uf + (size_t)(2 + j) * W + 2 + i;
  const size_t plane = (size_t)p.nx * p.ny;
  double v = dmul(p.c0[k], c[0]);
  for (int t = 0; t < p.kx; ++t) v = dadd(v, dmul(p.cx[t * plane + k], c[p.ox[t]]));
  for (int t = 0; t < p.ky; ++t) {
    const double term = dmul(p.cy[t * plane + k], c[(ptrdiff_t)p.oy[t] * W]);
    if (dep < 0 || t < dep) v = dadd(v, term);
    else if (t > dep) rest[t - dep - 1] = term;
  }
  return v;
}

// numpy's pairwise sum of a contiguous float64 array: leaves of <= 128
// summed with 8 accumulators, longer runs split at half rounded down to a
// multiple of 8 and the halves added (the recursion runs on an explicit
// stack: the call stack would overflow at study sizes).
__device__ double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = dadd(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = a[k];
  const int64_t m = n - n % 8;
  for (int64_t i = 8; i < m; i += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = dadd(r[k], a[i + k]);
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])),
                    dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (int64_t i = m; i < n; ++i) res = dadd(res, a[i]);
  return res;
}

// The pairwise recursion walked depth-first on an explicit stack; at each
// leaf, LEAF(offset, length) gives its sum.
template <typename Leaf>
__device__ double pairwise_walk(int64_t n, Leaf leaf) {
  struct Frame {
    int64_t off, n;
    double left;
    int stage;
  };
  Frame st[64];  // depth ~log2(n / 128) + 1
  int sp = 0;
  st[0] = {0, n, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = leaf(f.off, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {
      f.stage = 1;
      st[sp + 1] = {f.off, n2, 0.0, 0};
      ++sp;
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      st[sp + 1] = {f.off + n2, f.n - n2, 0.0, 0};
      ++sp;
    } else {
      ret = dadd(f.left, ret);
      --sp;
    }
  }
  return ret;
}

// numpy's pairwise sum of a (global, CTA-private) array with all threads of
// the CTA: leaf sums in parallel (thread t takes leaves t, t + blockDim,
// ... of the depth-first order and leaves each sum in its leaf's first
// slot), then thread 0 combines them in the recursion's order.  All
// threads call; the result is valid on thread 0.
__device__ double pairwise_sum_cta(double* a, int64_t n) {
  int64_t idx = 0;
  pairwise_walk(n, [&](int64_t off, int64_t len) {
    if (idx++ % blockDim.x == threadIdx.x) a[off] = pairwise_leaf(a + off, len);
    return 0.0;
  });
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) r = pairwise_walk(n, [&](int64_t off, int64_t) { return a[off]; });
  return r;
}

// solve_w + solve_z of one line on shared WZ factors (aqif.py:138-178,
// _kernels.py:152-225), reference operation order; one thread, y and x in
// shared memory.  Returns 0 or the 1-based Z breakdown level.
struct SharedFactors {
  const double *z2x2, *zl, *zr, *ww;
  const double *det, *rcp;  // per level: the 2x2 determinant, RN(1/det)
  const int* fl;            // per level: bit 0 det in the Markstein range, bit 1 breakdown
};

// The W and Z chains keep the unknowns they are about to reuse in
// registers (a window of BETA values per side that slides one row per
// level), so a level waits on its own arithmetic, not on shared memory.
template <int BETA>
__device__ int shared_line_solve(const SharedFactors& p, int n, double* __restrict__ y,
                                 double* __restrict__ x) {
  using A = Arith<true>;
  constexpr int TB = 2 * BETA, BP1 = BETA + 1;
  const int s = n / 2;
  const double* __restrict__ ww = p.ww;
  const double* __restrict__ zl = p.zl;
  const double* __restrict__ zr = p.zr;
  const double* __restrict__ z2 = p.z2x2;
  // W0 y = r, middle-out (solve_w_batch): wt[t] = y[rt - BETA + t],
  // wb[t] = y[rb + 1 + t] of the current level
  double wt[BETA], wb[BETA];
  double cur_t = y[s - 1], cur_b = y[s];
#pragma unroll
  for (int t = 0; t < BETA; ++t) {
    const int it = s - 1 - BETA + t, ib = s + 1 + t;
    wt[t] = it >= 0 ? y[it] : 0.0;
    wb[t] = ib < n ? y[ib] : 0.0;
  }
  for (int k = 1; k <= s; ++k) {
    const int rt = s - k, rb = s + k - 1;
    const double yt = cur_t, yb = cur_b;
    const double* wk = ww + (size_t)k * TB * 2;
#pragma unroll
    for (int t = 0; t < BETA; ++t) {
      if (rt - BETA + t >= 0)
        wt[t] = A::sub(wt[t], A::add(A::mul(yt, wk[t * 2]), A::mul(yb, wk[t * 2 + 1])));
      if (rb + 1 + t < n)
        wb[t] = A::sub(wb[t], A::add(A::mul(yt, wk[(BETA + t) * 2]),
                                     A::mul(yb, wk[(BETA + t) * 2 + 1])));
    }
    y[rt] = yt;  // final: no later level touches rows rt, rb
    y[rb] = yb;
    cur_t = wt[BETA - 1];
    cur_b = wb[0];
#pragma unroll
    for (int t = BETA - 1; t > 0; --t) wt[t] = wt[t - 1];
#pragma unroll
    for (int t = 0; t < BETA - 1; ++t) wb[t] = wb[t + 1];
    const int it = rt - 1 - BETA, ib = rb + 1 + BETA;
    wt[0] = it >= 0 ? y[it] : 0.0;
    wb[BETA - 1] = ib < n ? y[ib] : 0.0;
  }
  // Z0 x = y, outside-in (solve_z_batch, start level 1): xl[t] =
  // x[pp - BETA + t], xr[t] = x[q + 1 + t]
  double xl[BETA], xr[BETA];
#pragma unroll
  for (int t = 0; t < BETA; ++t) xl[t] = xr[t] = 0.0;
  for (int level = 1; level <= s; ++level) {
    const int pp = level - 1, q = n - 1 - pp, k = s - pp;
    const double* zlk = zl + (size_t)k * 2 * BP1;
    const double* zrk = zr + (size_t)k * 2 * BP1;
    double rt_rhs = y[pp], rb_rhs = y[q];
#pragma unroll
    for (int t = 0; t < BETA; ++t) {
      if (pp - BETA + t >= 0) {
        rt_rhs = A::axpy_neg(rt_rhs, zlk[t], xl[t]);
        rb_rhs = A::axpy_neg(rb_rhs, zlk[BP1 + t], xl[t]);
      }
      if (q + 1 + t < n) {
        rt_rhs = A::axpy_neg(rt_rhs, zrk[1 + t], xr[t]);
        rb_rhs = A::axpy_neg(rb_rhs, zrk[BP1 + 1 + t], xr[t]);
      }
    }
    const double* zk = z2 + (size_t)k * 4;
    const double a11 = zk[0], a12 = zk[1], a21 = zk[2], a22 = zk[3];
    const double det = p.det[k], yr = p.rcp[k];
    const int fl = p.fl[k];
    if (fl & 2) return level;
    const bool ds = fl & 1;
    // RN quotient through the reciprocal (Markstein), __ddiv_rn out of range
    const double xp = div_rn(A::det2(a22, rt_rhs, a12, rb_rhs), det, yr, ds);
    const double xq = div_rn(A::det2(a11, rb_rhs, a21, rt_rhs), det, yr, ds);
    x[pp] = xp;
    x[q] = xq;
#pragma unroll
    for (int t = 0; t < BETA - 1; ++t) xl[t] = xl[t + 1];
    xl[BETA - 1] = xp;
#pragma unroll
    for (int t = BETA - 1; t > 0; --t) xr[t] = xr[t - 1];
    xr[0] = xq;
  }
  return 0;
}

__global__ void __launch_bounds__(kTvdThreads, 1)
tvd_sweep_kernel(paqif_tvd_problem p, double* uf, int backward, int want_norm, double* resid,
                 double* norm, int32_t* status) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ int flag;
  const int nx = p.nx, ny = p.ny, W = nx + 4;
  const int n = (nx + 1) % 2 == 0 ? nx + 1 : nx + 2;  // _padded_even_order
  double* band = tsm;
  double* rhs = band + aqif2_band_doubles(n);
  double* rec = rhs + aqif2_rhs_doubles(n);
  const size_t plane = (size_t)nx * ny;
  if (!p.z2x2) aqif2_zero_pads(band, rhs, n);
  // shared factors staged in shared memory once: the line solves' chains
  // then wait on shared-memory, not L2, latency
  SharedFactors fz{};
  if (p.z2x2) {
    const int s = n / 2, bp1 = p.zf_beta + 1, tb = 2 * p.zf_beta;
    double* d = rec + (size_t)(n / 2 + 1) * kRec2;
    const size_t c4 = (size_t)(s + 1) * 4, cz = (size_t)(s + 1) * 2 * bp1,
                 cw = (size_t)(s + 1) * 2 * tb;
    for (size_t i = threadIdx.x; i < c4; i += blockDim.x) d[i] = p.z2x2[i];
    for (size_t i = threadIdx.x; i < cz; i += blockDim.x) d[c4 + i] = p.zl[i];
    for (size_t i = threadIdx.x; i < cz; i += blockDim.x) d[c4 + cz + i] = p.zr[i];
    for (size_t i = threadIdx.x; i < cw; i += blockDim.x) d[c4 + 2 * cz + i] = p.ww[i];
    double* dd = d + c4 + 2 * cz + cw;
    double* rr = dd + (s + 1);
    int* fl = reinterpret_cast<int*>(rr + (s + 1));
    __syncthreads();
    // the level's 2x2 pivot test and reciprocal depend on the factors only
    // (solve_z_batch, _kernels.py:175-225): once per sweep
    for (int k = 1 + threadIdx.x; k <= s; k += blockDim.x) {
      using A = Arith<true>;
      const double* zk = d + (size_t)k * 4;
      const double a11 = zk[0], a12 = zk[1], a21 = zk[2], a22 = zk[3];
      const double det = A::det2(a11, a22, a12, a21);
      double scale = fabs(a11);
      if (fabs(a12) > scale) scale = fabs(a12);
      if (fabs(a21) > scale) scale = fabs(a21);
      if (fabs(a22) > scale) scale = fabs(a22);
      const bool bad = fabs(det) <= 1e-14 * (scale * scale) + PAQIF_TINY;
      dd[k] = det;
      rr[k] = __drcp_rn(det);
      fl[k] = (div_safe(det) ? 1 : 0) | (bad ? 2 : 0);
    }
    fz = SharedFactors{d, d + c4, d + c4 + cz, d + c4 + 2 * cz, dd, rr, fl};
    __syncthreads();
  }
  int st = 0;
  if (p.z2x2) {
    // shared factors: warp 0 runs the line's W + Z chain while the other
    // warps form the next line's right side up to the term that reads the
    // row being solved; after the solve each thread updates its column of
    // that row and finishes the next right side with one product
    double* y = rhs;
    double* x = band;
    double* part = const_cast<double*>(fz.rcp) + (n / 2 + 1) + (n / 2 + 2) / 2;  // after the flags
    double* rest = part + nx;                              // 3 planes of nx
    const int od = backward ? 1 : -1;
    int dep = -1;
    for (int t = 0; t < p.ky; ++t)
      if (p.oy[t] == od && dep < 0) dep = t;
    const int j0 = backward ? ny - 1 : 0;
    for (int r = threadIdx.x; r < n; r += blockDim.x)
      y[r] = r < nx ? p.f[(size_t)j0 * nx + r] - apply_at(p, uf, j0, r) : 0.0;
    __syncthreads();
    for (int jj = 0; jj < ny; ++jj) {
      const int j = backward ? ny - 1 - jj : jj;
      const int jn = jj + 1 < ny ? (backward ? j - 1 : j + 1) : -1;
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) {
#ifdef PAQIF_TVD_PROF
          const long long t0 = clock64();
#endif
          flag = p.zf_beta == 1 ? shared_line_solve<1>(fz, n, y, x)
                                : shared_line_solve<2>(fz, n, y, x);
#ifdef PAQIF_TVD_PROF
          if (jj == ny / 2) printf("tvd W+Z line solve %lld cycles (n=%d)\n", clock64() - t0, n);
#endif
        }
      } else if (jn >= 0) {
        for (int i = threadIdx.x - 32; i < nx; i += blockDim.x - 32) {
          double r3[3];
          part[i] = apply_split(p, uf, jn, i, dep, r3);
          for (int t = 0; dep >= 0 && t < p.ky - dep - 1; ++t) rest[t * nx + i] = r3[t];
        }
      }
      __syncthreads();
      if (flag) {
        st = j + 1;
        break;
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        if (i >= nx) {
          y[i] = 0.0;  // pinned pad unknowns (the W sweep wrote them)
          continue;
        }
        double* c = uf + (size_t)(2 + j) * W + 2 + i;
        const double un = dadd(*c, dmul(p.omega, x[i]));
        *c = un;
        if (jn >= 0) {
          const size_t k = (size_t)jn * nx + i;
          double v = part[i];
          if (dep >= 0) {
            v = dadd(v, dmul(p.cy[dep * plane + k], un));
            for (int t = 0; t < p.ky - dep - 1; ++t) v = dadd(v, rest[t * nx + i]);
          }
          y[i] = p.f[k] - v;
        }
      }
      __syncthreads();
    }
  } else {
  for (int jj = 0; jj < ny; ++jj) {
    const int j = backward ? ny - 1 - jj : jj;
    {
      for (int r = threadIdx.x; r < n; r += blockDim.x) {
        // _line_matrix: identity diagonal, then the line's bands on rows
        // r < nx (columns may reach the pinned pad unknowns), out-of-range
        // columns zero
        double e[5] = {0.0, 0.0, 1.0, 0.0, 0.0};
        double rr = 0.0;
        if (r < nx) {
          const size_t k = (size_t)j * nx + r;
          for (int t = 0; t < 4; ++t) {
            const int o = t - 2;  // line band offsets -2, -1, 0, +1
            if (!(p.line_mask & (1 << t)) || r + o < 0) continue;
            e[o + 2] = p.lb[t * plane + k];
          }
          rr = p.f[k] - apply_at(p, uf, j, r);
        }
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int col = r + d - 2;
          band2_ref(band, n, r, d - 2) = (col >= 0 && col < n) ? e[d] : 0.0;
        }
        rhs[kBandPad + r] = rr;
      }
      // the solution goes to its own buffer: writing it over the band would
      // clobber the diagonal -2 leading pads the next line's factor reads
      double* xs = rec + (size_t)(n / 2 + 1) * kRec2;
      const int s = aqif2_solve<true>(band, rhs, n, rec, xs, &flag);
      if (s & 1) {
        st = j + 1;
        break;
      }
    }
    {
      const double* xs = rec + (size_t)(n / 2 + 1) * kRec2;
      for (int i = threadIdx.x; i < nx; i += blockDim.x) {
        double* c = uf + (size_t)(2 + j) * W + 2 + i;
        *c = dadd(*c, dmul(p.omega, xs[i]));
      }
    }
    __syncthreads();
  }
  }
  if (threadIdx.x == 0) *status = st;
  if (!want_norm || st) return;
  for (int64_t k = threadIdx.x; k < (int64_t)plane; k += blockDim.x) {
    const int j = (int)(k / nx), i = (int)(k - (int64_t)j * nx);
    const double r = p.f[k] - apply_at(p, uf, j, i);
    resid[k] = dmul(r, r);
  }
  __syncthreads();
  const double sum = pairwise_sum_cta(resid, (int64_t)plane);
  if (threadIdx.x == 0) *norm = sqrt(dmul(p.h2, sum));
}

// interior of a (ny+4) x (nx+4) field into the interior of the transposed
// (nx+4) x (ny+4) field
__global__ void tvd_transpose_kernel(const double* src, int ny, int nx, double* dst) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int j = by + r, i = bx + threadIdx.x;
    if (j < ny && i < nx) tile[r][threadIdx.x] = src[(size_t)(2 + j) * (nx + 4) + 2 + i];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + r, j = by + threadIdx.x;
    if (j < ny && i < nx) dst[(size_t)(2 + i) * (ny + 4) + 2 + j] = tile[threadIdx.x][r];
  }
}

// Ls3 line-distributive relaxation (tvdcd.py:615-656): every x-line's
// change from the current iterate -- independent lines, one CTA each:
//   rhs = resid[j] + (a/h)[j] * (k1 (u[i+1] - u[i]) - k2 (u[i-1] - u[i-2])),
//         explicit term 0 at i = 0
//   sigma[j] = AQIF solve of the padded pentadiagonal line (offsets -2..2)
__global__ void __launch_bounds__(kTvdThreads, 1)
tvd_distributive_lines_kernel(paqif_tvd_problem p, const double* uf, const double* ah,
                              const double* db, double k1, double k2, double* sigma,
                              int32_t* status) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ int flag;
  const int nx = p.nx, ny = p.ny, W = nx + 4, j = blockIdx.x;
  const int n = (nx + 1) % 2 == 0 ? nx + 1 : nx + 2;
  const size_t plane = (size_t)nx * ny;
  double* band = dsm;
  double* rhs = band + aqif2_band_doubles(n);
  double* rec = rhs + aqif2_rhs_doubles(n);
  double* x = rec + (size_t)(n / 2 + 1) * kRec2;
  aqif2_zero_pads(band, rhs, n);
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double e[5] = {0.0, 0.0, 1.0, 0.0, 0.0};
    double rr = 0.0;
    if (r < nx) {
      const size_t k = (size_t)j * nx + r;
#pragma unroll
      for (int d = 0; d < 5; ++d)
        if (r + d - 2 >= 0) e[d] = db[d * plane + k];
      const double* c = uf + (size_t)(2 + j) * W + 2 + r;
      const double res = p.f[k] - apply_at(p, uf, j, r);
      double ex = __dsub_rn(dmul(k1, __dsub_rn(c[1], c[0])), dmul(k2, __dsub_rn(c[-1], c[-2])));
      if (r == 0) ex = 0.0;
      rr = dadd(res, dmul(ah[k], ex));
    }
#pragma unroll
    for (int d = 0; d < 5; ++d) {
      const int col = r + d - 2;
      band2_ref(band, n, r, d - 2) = (col >= 0 && col < n) ? e[d] : 0.0;
    }
    rhs[kBandPad + r] = rr;
  }
  const int st = aqif2_solve<true>(band, rhs, n, rec, x, &flag);
  for (int i = threadIdx.x; i < nx; i += blockDim.x) sigma[(size_t)j * nx + i] = x[i];
  if (threadIdx.x == 0) status[j] = (st & 1) ? 1 : 0;
}

// u += omega (sigma - 0.25 spread), spread = the four neighbours' sigma
// (added left, right, below, above, as the reference's slices do), then
// the residual norm; one CTA
__global__ void __launch_bounds__(kTvdThreads, 1)
tvd_distributive_update_kernel(paqif_tvd_problem p, double* uf, const double* sigma,
                               const int32_t* lst, double* resid, double* norm,
                               int32_t* status) {
  const int nx = p.nx, ny = p.ny, W = nx + 4;
  const size_t plane = (size_t)nx * ny;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < ny; j += blockDim.x)
    if (lst[j]) atomicMax(&bad, j + 1);
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) *status = bad;  // a line broke down (the first is reported below)
    for (int j = 0; j < ny && threadIdx.x == 0; ++j)
      if (lst[j]) { *status = j + 1; break; }
    return;
  }
  for (int64_t k = threadIdx.x; k < (int64_t)plane; k += blockDim.x) {
    const int j = (int)(k / nx), i = (int)(k - (int64_t)j * nx);
    double sp = 0.0;
    if (i > 0) sp = dadd(sp, sigma[k - 1]);
    if (i < nx - 1) sp = dadd(sp, sigma[k + 1]);
    if (j > 0) sp = dadd(sp, sigma[k - nx]);
    if (j < ny - 1) sp = dadd(sp, sigma[k + nx]);
    double* c = uf + (size_t)(2 + j) * W + 2 + i;
    *c = dadd(*c, dmul(p.omega, __dsub_rn(sigma[k], dmul(0.25, sp))));
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < (int64_t)plane; k += blockDim.x) {
    const int j = (int)(k / nx), i = (int)(k - (int64_t)j * nx);
    const double r = p.f[k] - apply_at(p, uf, j, i);
    resid[k] = dmul(r, r);
  }
  __syncthreads();
  const double sum = pairwise_sum_cta(resid, (int64_t)plane);
  if (threadIdx.x == 0) {
    *norm = sqrt(dmul(p.h2, sum));
    *status = 0;
  }
}

size_t tvd_smem(int nx, int zf_beta) {
  const int n = (nx + 1) % 2 == 0 ? nx + 1 : nx + 2;
  const size_t fz =
      zf_beta ? (size_t)(n / 2 + 1) * (4 + 4 * (zf_beta + 1) + 4 * zf_beta + 3) + 4 * (size_t)nx + 8
              : (size_t)n;  // per-line factors: the solution buffer
  return (aqif2_band_doubles(n) + aqif2_rhs_doubles(n) + (size_t)(n / 2 + 1) * kRec2 + fz) * 8;
}

}  // namespace paqif

using namespace paqif;

extern "C" size_t paqif_tvd_resid_bytes(int32_t nx, int32_t ny) {
  return nx > 0 && ny > 0 ? (size_t)nx * ny * 8 : 0;
}

extern "C" int paqif_tvd_sweep(const paqif_tvd_problem* p, double* u_full, int32_t backward,
                               int32_t want_norm, double* resid, double* norm, int32_t* status,
                               void* stream) {
  if (!p || p->nx < 2 || p->ny < 1 || !p->f || !p->c0 || !p->lb || !u_full || !status ||
      p->kx < 0 || p->kx > 4 || p->ky < 0 || p->ky > 4 || (p->kx && !p->cx) ||
      (p->z2x2 && (!p->zl || !p->zr || !p->ww || p->zf_beta < 1 || p->zf_beta > 2)) ||
      (p->ky && !p->cy) || (want_norm && (!resid || !norm)))
    return set_arg_error("paqif_tvd_sweep: problem / buffers");
  for (int t = 0; t < p->kx; ++t)
    if (p->ox[t] < -2 || p->ox[t] > 2) return set_arg_error("paqif_tvd_sweep: x offset");
  for (int t = 0; t < p->ky; ++t)
    if (p->oy[t] < -2 || p->oy[t] > 2) return set_arg_error("paqif_tvd_sweep: y offset");
  const size_t smem = tvd_smem(p->nx, p->z2x2 ? p->zf_beta : 0);
  if (smem > 227 * 1024) return set_arg_error("paqif_tvd_sweep: line too long for one CTA");
  cudaFuncSetAttribute(tvd_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tvd_sweep_kernel<<<1, kTvdThreads, smem, (cudaStream_t)stream>>>(*p, u_full, backward,
                                                                    want_norm, resid, norm,
                                                                    status);
  return check_launch("paqif_tvd_sweep");
}

extern "C" int paqif_tvd_transpose(const double* src_full, int32_t ny, int32_t nx,
                                   double* dst_full, void* stream) {
  if (!src_full || !dst_full || nx < 1 || ny < 1)
    return set_arg_error("paqif_tvd_transpose");
  dim3 grid((nx + 31) / 32, (ny + 31) / 32), block(32, 8);
  tvd_transpose_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(src_full, ny, nx, dst_full);
  return check_launch("paqif_tvd_transpose");
}

extern "C" int paqif_tvd_distributive(const paqif_tvd_problem* p, double* u_full,
                                      const double* a_over_h, const double* line_bands,
                                      double k1, double k2, double* sigma, int32_t* line_status,
                                      double* resid, double* norm, int32_t* status, void* stream) {
  if (!p || p->nx < 2 || p->ny < 1 || !p->f || !p->c0 || !u_full || !a_over_h || !line_bands ||
      !sigma || !line_status || !resid || !norm || !status || p->kx < 0 || p->kx > 4 ||
      p->ky < 0 || p->ky > 4 || (p->kx && !p->cx) || (p->ky && !p->cy))
    return set_arg_error("paqif_tvd_distributive: problem / buffers");
  const int n = (p->nx + 1) % 2 == 0 ? p->nx + 1 : p->nx + 2;
  const size_t smem = (aqif2_band_doubles(n) + aqif2_rhs_doubles(n) +
                       (size_t)(n / 2 + 1) * kRec2 + n) * 8;
  if (smem > 227 * 1024) return set_arg_error("paqif_tvd_distributive: line too long");
  cudaFuncSetAttribute(tvd_distributive_lines_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  cudaStream_t st = (cudaStream_t)stream;
  tvd_distributive_lines_kernel<<<p->ny, kTvdThreads, smem, st>>>(*p, u_full, a_over_h, line_bands,
                                                                 k1, k2, sigma, line_status);
  if (int rc = check_launch("paqif_tvd_distributive")) return rc;
  tvd_distributive_update_kernel<<<1, kTvdThreads, 0, st>>>(*p, u_full, sigma, line_status, resid,
                                                            norm, status);
  return check_launch("paqif_tvd_distributive");
}
