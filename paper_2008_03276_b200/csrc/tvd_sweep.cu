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

// numpy's pairwise sum of a contiguous float64 array: leaves of <= 128
// summed with 8 accumulators, longer runs split at half rounded down to a
// multiple of 8 and the halves added.  One thread; the recursion is run on
// an explicit stack (the call stack would overflow at study sizes).
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

__device__ double pairwise_sum(const double* a, int64_t n) {
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
      ret = pairwise_leaf(a + f.off, f.n);
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
  aqif2_zero_pads(band, rhs, n);
  int st = 0;
  for (int jj = 0; jj < ny; ++jj) {
    const int j = backward ? ny - 1 - jj : jj;
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
    const int s = aqif2_solve<true>(band, rhs, n, rec, band, &flag);
    if (s & 1) {
      st = j + 1;
      break;
    }
    for (int i = threadIdx.x; i < nx; i += blockDim.x) {
      double* c = uf + (size_t)(2 + j) * W + 2 + i;
      *c = dadd(*c, dmul(p.omega, band[i]));
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = st;
  if (!want_norm || st) return;
  for (int64_t k = threadIdx.x; k < (int64_t)plane; k += blockDim.x) {
    const int j = (int)(k / nx), i = (int)(k - (int64_t)j * nx);
    const double r = p.f[k] - apply_at(p, uf, j, i);
    resid[k] = dmul(r, r);
  }
  __syncthreads();
  if (threadIdx.x == 0) *norm = sqrt(dmul(p.h2, pairwise_sum(resid, (int64_t)plane)));
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

size_t tvd_smem(int nx) {
  const int n = (nx + 1) % 2 == 0 ? nx + 1 : nx + 2;
  return (aqif2_band_doubles(n) + aqif2_rhs_doubles(n) + (size_t)(n / 2 + 1) * kRec2) * 8;
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
      (p->ky && !p->cy) || (want_norm && (!resid || !norm)))
    return set_arg_error("paqif_tvd_sweep: problem / buffers");
  for (int t = 0; t < p->kx; ++t)
    if (p->ox[t] < -2 || p->ox[t] > 2) return set_arg_error("paqif_tvd_sweep: x offset");
  for (int t = 0; t < p->ky; ++t)
    if (p->oy[t] < -2 || p->oy[t] > 2) return set_arg_error("paqif_tvd_sweep: y offset");
  const size_t smem = tvd_smem(p->nx);
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
