// Drop-in replacements for the reference's batched numba kernels
// (paqif/_kernels.py).  Same arrays, same in-place semantics, same status
// codes; with PAQIF_FLAG_EXACT the results are bit-identical to the
// reference (tests/test_dropin_gpu.py pins this against golden vectors).
//
//   factor_batch      _kernels.py:62-149   warp per system, register windows
//                                          (aqif_warp.cuh) for beta <= 8;
//                                          thread per system on the cross
//                                          layout for larger beta
//   solve_w_batch     _kernels.py:152-172  warp per system, lanes over wings
//   solve_z_batch     _kernels.py:175-225  thread per system (serial chain)
//   band_matvec_batch _kernels.py:228-241  thread per row
//   psor_sweeps       _kernels.py:244-276  single thread (sequential oracle)
#include "aqif_warp.cuh"
#include "capi_util.cuh"

namespace paqif {

// ------------------------------------------------------------------ factor
template <int BETA>
struct DropinPol {
  static constexpr bool kFuseW = false;
  static constexpr bool kResidual = true;
  static constexpr bool kFastDiv = false;  // branch-free divisions, checked repeat
  static constexpr bool kLazyBreakdown = false;  // breakdown found after the loop
  static constexpr bool kRecordW = true;
  static constexpr int BP1 = BETA + 1;
  double* band;
  double* anti;
  double* z2x2;
  double* zl;
  double* zr;
  double* ww;
  int n;

  __device__ __forceinline__ const double* raw_ptr(int i, int d) const {
    return band + (size_t)(d + BETA) * n + i;
  }
  __device__ __forceinline__ double raw(int i, int d) const { return *raw_ptr(i, d); }
  __device__ __forceinline__ const uint64_t* pin_ptr(int) const { return nullptr; }
  __device__ __forceinline__ bool pinned(int) const { return false; }
  __device__ __forceinline__ const double* frhs_ptr(int) const { return nullptr; }
  __device__ __forceinline__ double frhs(int) const { return 0.0; }
  __device__ __forceinline__ void on_level(int k, const double* pb, int gl, int G) {
    using PL = PivotLayout<BETA>;
    const int s = n / 2, rt = s - k, rb = s + k - 1;
    for (int idx = gl; idx < PL::kZ; idx += G) {
      const int side = idx & 1, e = (idx >> 1) % BP1, win = (idx >> 1) / BP1;
      const double v = pb[idx];
      if (win == 0) {
        if (rt - e >= 0) zl[((size_t)k * 2 + side) * BP1 + (BETA - e)] = v;
      } else {
        if (rb + e < n) zr[((size_t)k * 2 + side) * BP1 + e] = v;
      }
    }
    if (gl == 0) {
      double* z = z2x2 + (size_t)k * 4;
      z[0] = pb[PL::zi(0, 0, 0)];
      z[1] = pb[PL::zi(1, 0, 0)];
      z[2] = pb[PL::zi(0, 0, 1)];
      z[3] = pb[PL::zi(1, 0, 1)];
    }
  }
  __device__ __forceinline__ void on_w(int k, int t, double w1, double w2) {
    double* p = ww + ((size_t)k * 2 * BETA + t) * 2;
    p[0] = w1;
    p[1] = w2;
  }
  __device__ __forceinline__ void on_resid(int i, int j, double v) {
    const int d = j - i;
    if (d >= -BETA && d <= BETA) {
      band[(size_t)(d + BETA) * n + i] = v;
      return;
    }
    const int c = i + j - (n - 1);
    if (c >= -BETA && c <= BETA) anti[(size_t)(c + BETA) * n + i] = v;
  }
};

constexpr int kWarpsPerBlock = 4;

template <int BETA, bool EXACT>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
factor_warp_kernel(int64_t B, int n, double* band, double* anti, double* z2x2, double* zl,
                   double* zr, double* ww, double tol, int64_t* status)
{
  constexpr int G = Group<BETA>::G, P = Group<BETA>::P;
  extern __shared__ __align__(16) unsigned char dropin_dyn_smem[];
  EngineSmem<BETA>* sm = reinterpret_cast<EngineSmem<BETA>*>(dropin_dyn_smem);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane / G, gl = lane % G;
  const int64_t wb = ((int64_t)blockIdx.x * kWarpsPerBlock + wid) * P;
  if (wb >= B) return;  // whole warp past the batch
  const int64_t b = wb + g;
  const bool have = b < B;
  const int64_t bb = have ? b : wb;
  const int s = n / 2;
  const size_t nb = (size_t)(2 * BETA + 1) * n;
  DropinPol<BETA> pol;
  pol.band = band + bb * nb;
  pol.anti = anti + bb * nb;
  pol.z2x2 = z2x2 + bb * (size_t)(s + 1) * 4;
  pol.zl = zl + bb * (size_t)(s + 1) * 2 * (BETA + 1);
  pol.zr = zr + bb * (size_t)(s + 1) * 2 * (BETA + 1);
  pol.ww = ww + bb * (size_t)(s + 1) * 4 * BETA;
  pol.n = n;
  const int st = aqif_factor_group<BETA, EXACT>(pol, n, tol, sm[wid * P + g], gl, have);
  if (have && gl == 0) status[b] = st;
}

// Generic beta: direct restatement on the cross layout, one thread per system.
template <bool EXACT>
__device__ __forceinline__ double cget(const double* band, const double* anti, int beta, int n,
                                       int i, int j)
{
  const int d = j - i;
  if (d >= -beta && d <= beta) return band[(size_t)(d + beta) * n + i];
  const int c = i + j - (n - 1);
  if (c >= -beta && c <= beta) return anti[(size_t)(c + beta) * n + i];
  return 0.0;
}

template <bool EXACT>
__device__ __forceinline__ void cadd(double* band, double* anti, int beta, int n, int i, int j,
                                     double val)
{
  using A = Arith<EXACT>;
  const int d = j - i;
  if (d >= -beta && d <= beta) {
    double* p = band + (size_t)(d + beta) * n + i;
    *p = A::add(*p, val);
    return;
  }
  const int c = i + j - (n - 1);
  if (c >= -beta && c <= beta) {
    double* p = anti + (size_t)(c + beta) * n + i;
    *p = A::add(*p, val);
  }
}

template <bool EXACT>
__global__ void factor_generic_kernel(int64_t B, int n, int beta, double* band, double* anti,
                                      double* z2x2, double* zl, double* zr, double* ww,
                                      double tol, int64_t* status)
{
  using A = Arith<EXACT>;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int s = n / 2, bp1 = beta + 1, tb = 2 * beta;
  const size_t nb = (size_t)(2 * beta + 1) * n;
  double* bd = band + b * nb;
  double* an = anti + b * nb;
  double* z2 = z2x2 + b * (size_t)(s + 1) * 4;
  double* ZL = zl + b * (size_t)(s + 1) * 2 * bp1;
  double* ZR = zr + b * (size_t)(s + 1) * 2 * bp1;
  double* W = ww + b * (size_t)(s + 1) * 2 * tb;
  int st = 0;
  for (int k = 1; k <= s; ++k) {
    const int rt = s - k, rb = s + k - 1;
    double* zlk = ZL + (size_t)k * 2 * bp1;
    double* zrk = ZR + (size_t)k * 2 * bp1;
    for (int t = 0; t <= beta; ++t) {
      const int jl = rt - beta + t;
      if (jl >= 0) {
        zlk[t] = cget<EXACT>(bd, an, beta, n, rt, jl);
        zlk[bp1 + t] = cget<EXACT>(bd, an, beta, n, rb, jl);
      }
      const int jr = rb + t;
      if (jr < n) {
        zrk[t] = cget<EXACT>(bd, an, beta, n, rt, jr);
        zrk[bp1 + t] = cget<EXACT>(bd, an, beta, n, rb, jr);
      }
    }
    const double a11 = zlk[beta], a12 = zrk[0], a21 = zlk[bp1 + beta], a22 = zrk[bp1];
    double* zk = z2 + (size_t)k * 4;
    zk[0] = a11; zk[1] = a12; zk[2] = a21; zk[3] = a22;
    const int top_lo = rt - beta > 0 ? rt - beta : 0;
    const int bot_hi = rb + beta < n - 1 ? rb + beta : n - 1;
    if (!((top_lo <= rt - 1) || (rb + 1 <= bot_hi))) continue;
    const double det = A::det2(a11, a22, a21, a12);
    double scale = fabs(a11);
    if (fabs(a12) > scale) scale = fabs(a12);
    if (fabs(a21) > scale) scale = fabs(a21);
    if (fabs(a22) > scale) scale = fabs(a22);
    if (fabs(det) <= tol * (scale * scale) + PAQIF_TINY) { st = k; break; }
    double* wk = W + (size_t)k * tb * 2;
    for (int t = 0; t < tb; ++t) {
      int i;
      if (t < beta) { i = rt - beta + t; if (i < 0) continue; }
      else { i = rb + 1 + (t - beta); if (i >= n) continue; }
      const double b1 = cget<EXACT>(bd, an, beta, n, i, rt);
      const double b2 = cget<EXACT>(bd, an, beta, n, i, rb);
      const double w1 = A::div(A::det2(a22, b1, a21, b2), det);
      const double w2 = A::div(A::det2(a11, b2, a12, b1), det);
      wk[t * 2] = w1; wk[t * 2 + 1] = w2;
      if (w1 == 0.0 && w2 == 0.0) continue;
      for (int u = 0; u <= beta; ++u) {
        const int jl = rt - beta + u;
        if (jl >= 0)
          cadd<EXACT>(bd, an, beta, n, i, jl,
                      -A::add(A::mul(w1, zlk[u]), A::mul(w2, zlk[bp1 + u])));
        const int jr = rb + u;
        if (jr < n)
          cadd<EXACT>(bd, an, beta, n, i, jr,
                      -A::add(A::mul(w1, zrk[u]), A::mul(w2, zrk[bp1 + u])));
      }
    }
  }
  status[b] = st;
}

// ------------------------------------------------------------------ solve_w
template <bool EXACT>
__global__ void __launch_bounds__(32 * kWarpsPerBlock)
solve_w_kernel(int64_t B, int n, int beta, const double* ww, double* rhs)
{
  using A = Arith<EXACT>;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * kWarpsPerBlock + wid;
  if (b >= B) return;
  const int s = n / 2, tb = 2 * beta;
  const double* W = ww + b * (size_t)(s + 1) * 2 * tb;
  double* y = rhs + b * (size_t)n;
  for (int k = 1; k <= s; ++k) {
    const int rt = s - k, rb = s + k - 1;
    const double yt = y[rt], yb = y[rb];
    const double* wk = W + (size_t)k * tb * 2;
    for (int t = lane; t < tb; t += 32) {
      const int i = t < beta ? rt - beta + t : rb + 1 + (t - beta);
      if (i >= 0 && i < n)
        y[i] = A::sub(y[i], A::add(A::mul(yt, wk[t * 2]), A::mul(yb, wk[t * 2 + 1])));
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ solve_z
template <bool EXACT>
__global__ void solve_z_kernel(int64_t B, int n, int beta, const double* z2x2, const double* zl,
                               const double* zr, const double* y, double* x, int start,
                               double tol, int64_t* status, int64_t* trace)
{
  using A = Arith<EXACT>;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int s = n / 2, bp1 = beta + 1;
  const double* Z2 = z2x2 + b * (size_t)(s + 1) * 4;
  const double* ZL = zl + b * (size_t)(s + 1) * 2 * bp1;
  const double* ZR = zr + b * (size_t)(s + 1) * 2 * bp1;
  const double* Y = y + b * (size_t)n;
  double* X = x + b * (size_t)n;
  int64_t* T = trace ? trace + b * (size_t)n : nullptr;
  int st = 0, pos = 0;
  for (int level = start; level <= s; ++level) {
    const int p = level - 1, q = n - 1 - p, k = s - p;
    const double* zlk = ZL + (size_t)k * 2 * bp1;
    const double* zrk = ZR + (size_t)k * 2 * bp1;
    double rt_rhs = Y[p], rb_rhs = Y[q];
    for (int t = 0; t < beta; ++t) {
      const int j = p - beta + t;
      if (j >= 0) {
        rt_rhs = A::axpy_neg(rt_rhs, zlk[t], X[j]);
        rb_rhs = A::axpy_neg(rb_rhs, zlk[bp1 + t], X[j]);
      }
      const int j2 = q + 1 + t;
      if (j2 < n) {
        rt_rhs = A::axpy_neg(rt_rhs, zrk[1 + t], X[j2]);
        rb_rhs = A::axpy_neg(rb_rhs, zrk[bp1 + 1 + t], X[j2]);
      }
    }
    const double* zk = Z2 + (size_t)k * 4;
    const double a11 = zk[0], a12 = zk[1], a21 = zk[2], a22 = zk[3];
    const double det = A::det2(a11, a22, a12, a21);
    double scale = fabs(a11);
    if (fabs(a12) > scale) scale = fabs(a12);
    if (fabs(a21) > scale) scale = fabs(a21);
    if (fabs(a22) > scale) scale = fabs(a22);
    if (fabs(det) <= tol * (scale * scale) + PAQIF_TINY) { st = level; break; }
    X[p] = A::div(A::det2(a22, rt_rhs, a12, rb_rhs), det);
    X[q] = A::div(A::det2(a11, rb_rhs, a21, rt_rhs), det);
    if (T) { T[pos] = p; T[pos + 1] = q; }
    pos += 2;
  }
  status[b] = st;
}

// ------------------------------------------------------------------ matvec
template <bool EXACT>
__global__ void matvec_kernel(int64_t B, int n, int beta, const double* bands, const double* x,
                              double* out)
{
  using A = Arith<EXACT>;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= B * (int64_t)n) return;
  const int64_t b = g / n;
  const int i = (int)(g % n);
  const double* bd = bands + b * (size_t)(2 * beta + 1) * n;
  const double* xb = x + b * (size_t)n;
  double acc = 0.0;
  const int lo = i - beta > 0 ? i - beta : 0;
  const int hi = i + beta + 1 < n ? i + beta + 1 : n;
  for (int j = lo; j < hi; ++j) acc = A::axpy(acc, bd[(size_t)(j - i + beta) * n + i], xb[j]);
  out[g] = acc;
}

// ------------------------------------------------------------------ psor
__global__ void psor_kernel(int n, int beta, const double* bands, const double* f, double* u,
                            double omega, double tol, int64_t max_sweeps, int64_t* sweeps_out,
                            double* change_out)
{
  using A = Arith<true>;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t sweeps = 0;
  double change = 0.0;
  for (int64_t sweep = 0; sweep < max_sweeps; ++sweep) {
    change = 0.0;
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      const int lo = i - beta > 0 ? i - beta : 0;
      const int hi = i + beta + 1 < n ? i + beta + 1 : n;
      for (int j = lo; j < hi; ++j)
        if (j != i) acc = A::axpy(acc, bands[(size_t)(j - i + beta) * n + i], u[j]);
      const double diag = bands[(size_t)beta * n + i];
      double unew = A::add(A::mul(A::sub(1.0, omega), u[i]),
                           A::div(A::mul(omega, A::sub(f[i], acc)), diag));
      if (unew < 0.0) unew = 0.0;
      const double d = fabs(A::sub(unew, u[i]));
      if (d > change) change = d;
      u[i] = unew;
    }
    sweeps = sweep + 1;
    if (change <= tol) break;
  }
  *sweeps_out = sweeps;
  *change_out = change;
}

}  // namespace paqif

// ====================================================================== C ABI
using namespace paqif;

template <bool EXACT>
static void launch_factor(int64_t B, int n, int beta, double* band, double* anti, double* z2x2,
                          double* zl, double* zr, double* ww, double tol, int64_t* status,
                          cudaStream_t st)
{
  const unsigned blk = 32 * kWarpsPerBlock;
#define PAQIF_FACTOR_CASE(BB)                                                                 \
  case BB: {                                                                                  \
    const int64_t per_block = (int64_t)kWarpsPerBlock * Group<BB>::P;                          \
    const unsigned grid = (unsigned)((B + per_block - 1) / per_block);                         \
    const size_t smem = sizeof(EngineSmem<BB>) * per_block;                                    \
    cudaFuncSetAttribute(factor_warp_kernel<BB, EXACT>,                                        \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
    factor_warp_kernel<BB, EXACT><<<grid, blk, smem, st>>>(B, n, band, anti, z2x2, zl, zr, ww, \
                                                           tol, status);                      \
    break;                                                                                    \
  }
  switch (beta) {
    PAQIF_FACTOR_CASE(1)
    PAQIF_FACTOR_CASE(2)
    PAQIF_FACTOR_CASE(3)
    PAQIF_FACTOR_CASE(4)
    PAQIF_FACTOR_CASE(5)
    PAQIF_FACTOR_CASE(6)
    PAQIF_FACTOR_CASE(7)
    PAQIF_FACTOR_CASE(8)
    default:
      factor_generic_kernel<EXACT><<<(unsigned)((B + 63) / 64), 64, 0, st>>>(
          B, n, beta, band, anti, z2x2, zl, zr, ww, tol, status);
  }
#undef PAQIF_FACTOR_CASE
}

extern "C" int paqif_factor_batch(int64_t B, int64_t n, int64_t beta, double* band, double* anti,
                                  double* z2x2, double* zl, double* zr, double* ww, double tol,
                                  int64_t* status, uint32_t flags, void* stream)
{
  if (B < 0 || n < 2 || (n & 1) || beta < 1 || n > (1 << 28)) return set_arg_error("factor: bad sizes");
  if (B == 0) return PAQIF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (flags & PAQIF_FLAG_EXACT)
    launch_factor<true>(B, (int)n, (int)beta, band, anti, z2x2, zl, zr, ww, tol, status, st);
  else
    launch_factor<false>(B, (int)n, (int)beta, band, anti, z2x2, zl, zr, ww, tol, status, st);
  return check_launch("paqif_factor_batch");
}

extern "C" int paqif_solve_w_batch(int64_t B, int64_t n, int64_t beta, const double* ww,
                                   double* rhs, uint32_t flags, void* stream)
{
  if (B < 0 || n < 2 || (n & 1) || beta < 1) return set_arg_error("solve_w: bad sizes");
  if (B == 0) return PAQIF_OK;
  const unsigned grid = (unsigned)((B + kWarpsPerBlock - 1) / kWarpsPerBlock);
  if (flags & PAQIF_FLAG_EXACT)
    solve_w_kernel<true><<<grid, 32 * kWarpsPerBlock, 0, (cudaStream_t)stream>>>(B, (int)n, (int)beta, ww, rhs);
  else
    solve_w_kernel<false><<<grid, 32 * kWarpsPerBlock, 0, (cudaStream_t)stream>>>(B, (int)n, (int)beta, ww, rhs);
  return check_launch("paqif_solve_w_batch");
}

extern "C" int paqif_solve_z_batch(int64_t B, int64_t n, int64_t beta, const double* z2x2,
                                   const double* zl, const double* zr, const double* y, double* x,
                                   int64_t start, double tol, int64_t* status, int64_t* trace,
                                   uint32_t flags, void* stream)
{
  if (B < 0 || n < 2 || (n & 1) || beta < 1 || start < 1) return set_arg_error("solve_z: bad sizes");
  if (B == 0) return PAQIF_OK;
  const unsigned grid = (unsigned)((B + 63) / 64);
  if (flags & PAQIF_FLAG_EXACT)
    solve_z_kernel<true><<<grid, 64, 0, (cudaStream_t)stream>>>(B, (int)n, (int)beta, z2x2, zl, zr, y, x,
                                                              (int)start, tol, status, trace);
  else
    solve_z_kernel<false><<<grid, 64, 0, (cudaStream_t)stream>>>(B, (int)n, (int)beta, z2x2, zl, zr, y, x,
                                                               (int)start, tol, status, trace);
  return check_launch("paqif_solve_z_batch");
}

extern "C" int paqif_band_matvec_batch(int64_t B, int64_t n, int64_t beta, const double* bands,
                                       const double* x, double* out, void* stream)
{
  if (B < 0 || n < 1 || beta < 0) return set_arg_error("matvec: bad sizes");
  const int64_t total = B * n;
  if (total == 0) return PAQIF_OK;
  matvec_kernel<true><<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      B, (int)n, (int)beta, bands, x, out);
  return check_launch("paqif_band_matvec_batch");
}

extern "C" int paqif_psor_sweeps(int64_t n, int64_t beta, const double* bands, const double* f,
                                 double* u, double omega, double tol, int64_t max_sweeps,
                                 int64_t* sweeps, double* change, void* stream)
{
  if (n < 1 || beta < 0) return set_arg_error("psor: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf<int64_t> ds(1);
  DevBuf<double> dc(1);
  if (!ds.ok() || !dc.ok()) return set_cuda_error("psor: alloc", cudaErrorMemoryAllocation);
  psor_kernel<<<1, 32, 0, st>>>((int)n, (int)beta, bands, f, u, omega, tol, max_sweeps, ds.p, dc.p);
  int rc = check_launch("paqif_psor_sweeps");
  if (rc) return rc;
  cudaError_t e1 = cudaMemcpyAsync(sweeps, ds.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaError_t e2 = cudaMemcpyAsync(change, dc.p, sizeof(double), cudaMemcpyDeviceToHost, st);
  cudaError_t e3 = cudaStreamSynchronize(st);
  if (e1 != cudaSuccess) return set_cuda_error("psor: copy", e1);
  if (e2 != cudaSuccess) return set_cuda_error("psor: copy", e2);
  if (e3 != cudaSuccess) return set_cuda_error("psor: sync", e3);
  return PAQIF_OK;
}
