// r-block partitioned PAQIF on the device: the reference's seven-step block
// method (paqif/parallel.py:106-295) for a batch of B systems, every step a
// kernel -- no host arithmetic:
//
//   1. partition into r blocks of even size t > 2 beta, couplings L-/L+   parallel.py:106-147
//   2-3. factor + W solve of all B*r blocks (batched AQIF kernels)        parallel.py:159-164
//   4. per system: W corner inverses, Z corner blocks, reduced system
//      R_d (2 beta r, semibandwidth 3 beta - 1), normal equations,
//      banded Cholesky, optional projection                             parallel.py:184-231
//   5. middles: Z solve from start level beta+1 with the corners known   parallel.py:234-258
//
// Step 4 runs one CTA per system with R_d and R_d^T R_d in banded storage
// (global workspace, L2 resident), so the order 2 beta r is unbounded.  The
// reduced system uses its own summation order (the reference calls
// numpy / LAPACK there): results agree to rounding, not bit for bit.
#include <cmath>
#include "capi_util.cuh"

extern "C" {
#include "../../include/paqif_b200.h"
}

namespace paqif {

struct RbDims {
  int64_t B;
  int n, beta, r, t, st, md, w, w2;  // t block size, st = t/2, md = 2 beta r, w = 3 beta - 1, w2 = 2w
  __host__ __device__ RbDims(int64_t B_, int n_, int beta_, int r_) : B(B_), n(n_), beta(beta_), r(r_) {
    t = n / r;
    st = t / 2;
    md = 2 * beta * r;
    w = 3 * beta - 1;
    w2 = 2 * w;
  }
  __host__ __device__ int64_t nb() const { return B * r; }
};

// workspace layout (doubles unless noted), all counts per batch
struct RbLayout {
  size_t band, anti, z2x2, zl, zr, ww, y, lm, lp, rd, nn, fd, g, ud, bst, zst, total;
  __host__ __device__ explicit RbLayout(const RbDims& d) {
    const size_t NB = (size_t)d.nb();
    const size_t nd = (size_t)(2 * d.beta + 1);
    size_t o = 0;
    auto take = [&](size_t c) { size_t at = o; o += (c + 31) & ~(size_t)31; return at; };
    band = take(NB * nd * d.t);
    anti = take(NB * nd * d.t);
    z2x2 = take(NB * (d.st + 1) * 4);
    zl = take(NB * (d.st + 1) * 2 * (d.beta + 1));
    zr = take(NB * (d.st + 1) * 2 * (d.beta + 1));
    ww = take(NB * (d.st + 1) * 2 * d.beta * 2);
    y = take(NB * d.t);
    lm = take(NB * d.beta * d.beta);
    lp = take(NB * d.beta * d.beta);
    rd = take((size_t)d.B * d.md * (2 * d.w + 1));
    nn = take((size_t)d.B * d.md * (d.w2 + 1));
    fd = take((size_t)d.B * d.md);
    g = take((size_t)d.B * d.md);
    ud = take((size_t)d.B * d.md);
    bst = take(NB);  // int64 stored in double slots
    zst = take(NB);
    total = o;
  }
};

// step 1: blocks, couplings, block right sides (parallel.py:106-147)
__global__ void rb_partition_kernel(RbDims d, const double* __restrict__ bands,
                                    const double* __restrict__ f, double* band, double* anti,
                                    double* y, double* lm, double* lp) {
  const int64_t bm = blockIdx.x;  // system * r + block
  const int64_t b = bm / d.r;
  const int m = (int)(bm % d.r);
  const int be = d.beta, t = d.t, n = d.n, nd = 2 * be + 1;
  const int base = m * t;
  const double* src = bands + (size_t)b * nd * n;
  double* dst = band + (size_t)bm * nd * t;
  double* an = anti + (size_t)bm * nd * t;
  for (int idx = threadIdx.x; idx < nd * t; idx += blockDim.x) {
    const int oo = idx / t, i = idx % t, o = oo - be;
    const bool in = i + o >= 0 && i + o < t;
    dst[idx] = in ? src[(size_t)oo * n + base + i] : 0.0;
    an[idx] = 0.0;
  }
  for (int i = threadIdx.x; i < t; i += blockDim.x) y[(size_t)bm * t + i] = f[(size_t)b * n + base + i];
  for (int idx = threadIdx.x; idx < be * be; idx += blockDim.x) {
    const int a = idx / be, c = idx % be;
    double vm = 0.0, vp = 0.0;
    if (m > 0) {
      const int o = (base - be + c) - (base + a);
      if (o >= -be && o <= be) vm = src[(size_t)(be + o) * n + base + a];
    }
    if (m < d.r - 1) {
      const int i = base + t - be + a, j = base + t + c, o = j - i;
      if (o >= -be && o <= be) vp = src[(size_t)(be + o) * n + i];
    }
    lm[(size_t)bm * be * be + idx] = vm;
    lp[(size_t)bm * be * be + idx] = vp;
  }
}

// step 4 (one CTA per system): reduced system, normal equations, banded
// Cholesky, corners of x.  Shared: W corner (2b x 2b) and its inverse.
constexpr int kRbThreads = 256;
constexpr int kRbMaxBeta = 16;

__global__ void __launch_bounds__(kRbThreads) rb_reduced_kernel(RbDims d, double* ws_d,
                                                                const RbLayout L, double* x,
                                                                int project, int64_t* status) {
  __shared__ double wc[2 * kRbMaxBeta][4 * kRbMaxBeta];  // [W | I] for Gauss-Jordan
  __shared__ double wi[2 * kRbMaxBeta][2 * kRbMaxBeta];
  __shared__ int flag;
  const int64_t b = blockIdx.x;
  const int be = d.beta, t = d.t, st = d.st, r = d.r, md = d.md, w = d.w, w2 = d.w2;
  const int m2 = 2 * be;
  const int64_t* bst = reinterpret_cast<const int64_t*>(ws_d + L.bst);
  if (threadIdx.x == 0) {
    int bad = 0;
    for (int m = 0; m < r; ++m) bad |= bst[b * r + m] != 0;
    flag = bad;
  }
  __syncthreads();
  if (flag) {
    if (threadIdx.x == 0) status[b] = PAQIF_LCP_FACTOR_BREAKDOWN;
    return;
  }
  const int RW = 2 * w + 1;  // R_d row width (banded, column j at [j - i + w])
  double* rd = ws_d + L.rd + (size_t)b * md * RW;
  double* nn = ws_d + L.nn + (size_t)b * md * (w2 + 1);  // lower band: N(i, i-k) at [k]
  double* fd = ws_d + L.fd + (size_t)b * md;
  double* g = ws_d + L.g + (size_t)b * md;
  double* ud = ws_d + L.ud + (size_t)b * md;
  for (int idx = threadIdx.x; idx < md * RW; idx += blockDim.x) rd[idx] = 0.0;
  __syncthreads();
  auto RD = [&](int i, int j) -> double& { return rd[(size_t)i * RW + (j - i + w)]; };
  for (int m = 0; m < r; ++m) {
    const int64_t bm = b * r + m;
    const double* ww = ws_d + L.ww + (size_t)bm * (st + 1) * m2 * 2;
    const double* zl = ws_d + L.zl + (size_t)bm * (st + 1) * 2 * (be + 1);
    const double* zr = ws_d + L.zr + (size_t)bm * (st + 1) * 2 * (be + 1);
    const double* yb = ws_d + L.y + (size_t)bm * t;
    const double* lmm = ws_d + L.lm + (size_t)bm * be * be;
    const double* lpm = ws_d + L.lp + (size_t)bm * be * be;
    auto cidx = [&](int i) { return i < be ? i : (i >= t - be ? be + (i - (t - be)) : -1); };
    // W corner (WZFactors.w_dense restricted to rows/cols 0..b-1, t-b..t-1)
    for (int idx = threadIdx.x; idx < m2 * 2 * m2; idx += blockDim.x) {
      const int i = idx / (2 * m2), j = idx % (2 * m2);
      wc[i][j] = (j < m2) ? (i == j ? 1.0 : 0.0) : (j - m2 == i ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k <= st; ++k) {
        const int rt = st - k, rb = st + k - 1;
        const int ct = cidx(rt), cb = cidx(rb);
        for (int tt = 0; tt < m2; ++tt) {
          const int i = tt < be ? rt - be + tt : rb + 1 + (tt - be);
          if (i < 0 || i >= t) continue;
          const int ci = cidx(i);
          if (ci < 0) continue;
          if (ct >= 0) wc[ci][ct] = ww[((size_t)k * m2 + tt) * 2 + 0];
          if (cb >= 0) wc[ci][cb] = ww[((size_t)k * m2 + tt) * 2 + 1];
        }
      }
    }
    __syncthreads();
    // Gauss-Jordan with partial pivoting on [W | I] (np.linalg.inv)
    for (int c = 0; c < m2; ++c) {
      if (threadIdx.x == 0) {
        int p = c;
        for (int i = c + 1; i < m2; ++i)
          if (fabs(wc[i][c]) > fabs(wc[p][c])) p = i;
        if (p != c)
          for (int j = 0; j < 2 * m2; ++j) {
            const double tmp = wc[c][j];
            wc[c][j] = wc[p][j];
            wc[p][j] = tmp;
          }
        const double inv = 1.0 / wc[c][c];
        for (int j = 0; j < 2 * m2; ++j) wc[c][j] *= inv;
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < m2 * 2 * m2; idx += blockDim.x) {
        const int i = idx / (2 * m2), j = idx % (2 * m2);
        if (i != c) {
          const double fct = wc[i][c];
          if (j != c) wc[i][j] -= fct * wc[c][j];
        }
      }
      __syncthreads();
      if (threadIdx.x < m2 && threadIdx.x != c) wc[threadIdx.x][c] = 0.0;
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < m2 * m2; idx += blockDim.x)
      wi[idx / m2][idx % m2] = wc[idx / m2][m2 + idx % m2];
    __syncthreads();
    // Z corner blocks (z_corner_blocks) straight into R_d's diagonal block
    const int r0 = 2 * be * m;
    for (int idx = threadIdx.x; idx < be * 2 * (be + 1) * 2; idx += blockDim.x) {
      // corner rows are the pivot rows of the outermost levels k = st - kk
      // (rt = kk, rb = t-1-kk); enumerate (kk, side, window, entry)
      const int tt = idx % (be + 1);
      const int win = (idx / (be + 1)) % 2;
      const int side = (idx / (2 * (be + 1))) % 2;
      const int kk = idx / (4 * (be + 1));
      const int k = st - kk;
      if (k < 1) continue;
      const int rt = st - k, rb = st + k - 1;
      const int row = side == 0 ? rt : rb;
      const int col = win == 0 ? rt - be + tt : rb + tt;
      if (col < 0 || col >= t) continue;
      const int cr = cidx(row), cc = cidx(col);
      if (cr < 0 || cc < 0) continue;
      const double* src = win == 0 ? zl : zr;
      RD(r0 + cr, r0 + cc) = src[((size_t)k * 2 + side) * (be + 1) + tt];
    }
    // couplings: wi[:, :b] @ L-[m] into block m-1's U_L columns, wi[:, b:] @ L+[m]
    // into block m+1's U_F columns
    for (int idx = threadIdx.x; idx < m2 * be; idx += blockDim.x) {
      const int i = idx / be, c = idx % be;
      if (m > 0) {
        double s = 0.0;
        for (int q = 0; q < be; ++q) s = fma(wi[i][q], lmm[q * be + c], s);
        RD(r0 + i, 2 * be * (m - 1) + be + c) = s;
      }
      if (m < r - 1) {
        double s = 0.0;
        for (int q = 0; q < be; ++q) s = fma(wi[i][be + q], lpm[q * be + c], s);
        RD(r0 + i, 2 * be * (m + 1) + c) = s;
      }
    }
    for (int a = threadIdx.x; a < be; a += blockDim.x) {
      fd[r0 + a] = yb[a];
      fd[r0 + be + a] = yb[t - be + a];
    }
    __syncthreads();
  }
  // normal equations N = R^T R (semibandwidth 2w), g = R^T fd
  for (int idx = threadIdx.x; idx < md * (w2 + 1); idx += blockDim.x) {
    const int i = idx / (w2 + 1), kq = idx % (w2 + 1), j = i - kq;
    double s = 0.0;
    if (j >= 0) {
      const int lo = max(0, i - w), hi = min(md - 1, j + w);
      for (int q = lo; q <= hi; ++q) s = fma(rd[(size_t)q * RW + (i - q + w)], rd[(size_t)q * RW + (j - q + w)], s);
    }
    nn[idx] = s;
  }
  for (int i = threadIdx.x; i < md; i += blockDim.x) {
    double s = 0.0;
    const int lo = max(0, i - w), hi = min(md - 1, i + w);
    for (int q = lo; q <= hi; ++q) s = fma(rd[(size_t)q * RW + (i - q + w)], fd[q], s);
    g[i] = s;
  }
  __syncthreads();
  // banded Cholesky N = C C^T in place (lower band), then C C^T u = g
  auto NN = [&](int i, int j) -> double& { return nn[(size_t)i * (w2 + 1) + (i - j)]; };
  for (int j = 0; j < md; ++j) {
    if (threadIdx.x == 0) {
      const double dj = NN(j, j);
      if (!(dj > 0.0)) flag = 1;
      NN(j, j) = sqrt(dj);
    }
    __syncthreads();
    if (flag) break;
    const int hi = min(md - 1, j + w2);
    const double cjj = NN(j, j);
    for (int i = j + 1 + threadIdx.x; i <= hi; i += blockDim.x) NN(i, j) /= cjj;
    __syncthreads();
    const int span = hi - j;
    for (int idx = threadIdx.x; idx < span * span; idx += blockDim.x) {
      const int i = j + 1 + idx / span, k = j + 1 + idx % span;
      if (k <= i) NN(i, k) -= NN(i, j) * NN(k, j);
    }
    __syncthreads();
  }
  if (flag) {
    if (threadIdx.x == 0) status[b] = PAQIF_LCP_NOT_PD;
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < md; ++i) {  // C v = g
      double s = g[i];
      for (int j = max(0, i - w2); j < i; ++j) s -= NN(i, j) * ud[j];
      ud[i] = s / NN(i, i);
    }
    for (int i = md - 1; i >= 0; --i) {  // C^T u = v
      double s = ud[i];
      for (int k = i + 1; k <= min(md - 1, i + w2); ++k) s -= NN(k, i) * ud[k];
      ud[i] = s / NN(i, i);
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < md; idx += blockDim.x) {
    const int m = idx / (2 * be), a = idx % (2 * be);
    double v = ud[idx];
    if (project) v = v >= 0.0 || v != v ? v : 0.0;
    const int col = a < be ? m * t + a : m * t + t - be + (a - be);
    x[(size_t)b * d.n + col] = v;
  }
  if (threadIdx.x == 0) status[b] = 0;
}

__global__ void rb_finish_kernel(RbDims d, const double* ws_d, const RbLayout L, double* x,
                                 int project, int64_t* status) {
  const int64_t b = blockIdx.x;
  const int64_t* zst = reinterpret_cast<const int64_t*>(ws_d + L.zst);
  if (threadIdx.x == 0) {
    int z = 0;
    for (int m = 0; m < d.r; ++m) z |= zst[b * d.r + m] != 0;
    if (z && status[b] == 0) status[b] = PAQIF_LCP_ZSOLVE_BREAKDOWN;
  }
  __syncthreads();
  if (!project || status[b] != 0) return;
  for (int i = threadIdx.x; i < d.n; i += blockDim.x) {
    const int j = i % d.t;
    if (j >= d.beta && j < d.t - d.beta) {
      const double v = x[(size_t)b * d.n + i];
      x[(size_t)b * d.n + i] = (v >= 0.0 || v != v) ? v : 0.0;
    }
  }
}

}  // namespace paqif

using namespace paqif;

static int rb_check(int64_t B, int64_t n, int64_t beta, int64_t r) {
  if (B < 0 || n < 2 || beta < 1 || beta > kRbMaxBeta || r < 1 || n % r != 0)
    return set_arg_error("paqif_solve_rblock: bad sizes");
  const int64_t t = n / r;
  if (t % 2 != 0 || t <= 2 * beta) return set_arg_error("paqif_solve_rblock: block size");
  return PAQIF_OK;
}

extern "C" size_t paqif_solve_rblock_workspace_bytes(int64_t B, int64_t n, int64_t beta,
                                                     int64_t r) {
  if (rb_check(B, n, beta, r) != PAQIF_OK) return 0;
  const RbDims d(B, (int)n, (int)beta, (int)r);
  return RbLayout(d).total * sizeof(double);
}

extern "C" int paqif_solve_rblock_batch(int64_t B, int64_t n, int64_t beta, int64_t r,
                                        const double* bands, const double* f, double* x,
                                        int32_t project, int64_t* status, uint32_t flags,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  const int ck = rb_check(B, n, beta, r);
  if (ck != PAQIF_OK) return ck;
  if (B == 0) return PAQIF_OK;
  const RbDims d(B, (int)n, (int)beta, (int)r);
  const RbLayout L(d);
  if (workspace_bytes < L.total * sizeof(double) || !workspace)
    return set_arg_error("paqif_solve_rblock: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double* ws = reinterpret_cast<double*>(workspace);
  const int64_t NB = d.nb();
  rb_partition_kernel<<<(unsigned)NB, 128, 0, st>>>(d, bands, f, ws + L.band, ws + L.anti,
                                                    ws + L.y, ws + L.lm, ws + L.lp);
  int rc = check_launch("rb_partition");
  if (rc) return rc;
  int64_t* bst = reinterpret_cast<int64_t*>(ws + L.bst);
  int64_t* zst = reinterpret_cast<int64_t*>(ws + L.zst);
  rc = paqif_factor_batch(NB, d.t, beta, ws + L.band, ws + L.anti, ws + L.z2x2, ws + L.zl,
                          ws + L.zr, ws + L.ww, 1e-14, bst, flags, stream);
  if (rc) return rc;
  rc = paqif_solve_w_batch(NB, d.t, beta, ws + L.ww, ws + L.y, flags, stream);
  if (rc) return rc;
  rb_reduced_kernel<<<(unsigned)B, kRbThreads, 0, st>>>(d, ws, L, x, project, status);
  rc = check_launch("rb_reduced");
  if (rc) return rc;
  // middles: Z solve from level beta+1 with the corners prefilled (x viewed
  // as (B*r, t) blocks)
  rc = paqif_solve_z_batch(NB, d.t, beta, ws + L.z2x2, ws + L.zl, ws + L.zr, ws + L.y, x,
                           beta + 1, 1e-14, zst, nullptr, flags, stream);
  if (rc) return rc;
  rb_finish_kernel<<<(unsigned)B, 128, 0, st>>>(d, ws, L, x, project, status);
  return check_launch("rb_finish");
}

// ---------------------------------------------------------------------------
// The projected active-set pass for r > 1 (paqif_solve_lcp, parallel.py:
// 298-347), batched: pin the active rows, then after the block solve the
// multiplier / projection / residual / next active set of every system.
namespace paqif {

// lmod: active rows keep only their diagonal (1 if it is zero); fmod = 0 there
__global__ void lcp_pin_kernel(int n, int beta, const double* __restrict__ bands,
                               const double* __restrict__ f, const uint8_t* __restrict__ act,
                               double* lmod, double* fmod) {
  const int64_t b = blockIdx.y;
  const int nd = 2 * beta + 1;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nd * n; idx += gridDim.x * blockDim.x) {
    const int oo = idx / n, i = idx % n;
    const double v = bands[(size_t)b * nd * n + idx];
    double out = v;
    if (act[(size_t)b * n + i]) out = oo == beta ? (fabs(v) > 0.0 ? v : 1.0) : 0.0;
    lmod[(size_t)b * nd * n + idx] = out;
    if (oo == 0) fmod[(size_t)b * n + i] = act[(size_t)b * n + i] ? 0.0 : f[(size_t)b * n + i];
  }
}

// one CTA per system: lam = L u_eval - f, u = max(u_eval, 0),
// res = max|min(u, L u - f)| (NaN propagating), new_active = u_eval < lam,
// changed = any(new_active != active)
__global__ void lcp_pass_kernel(int n, int beta, const double* __restrict__ bands,
                                const double* __restrict__ f, const double* __restrict__ ue,
                                const uint8_t* __restrict__ act, double* u, uint8_t* nact,
                                double* res, int32_t* changed) {
  __shared__ double red[32];
  __shared__ int chg;
  const int64_t b = blockIdx.x;
  const int nd = 2 * beta + 1;
  const double* L = bands + (size_t)b * nd * n;
  const double* xe = ue + (size_t)b * n;
  double* xu = u + (size_t)b * n;
  if (threadIdx.x == 0) chg = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = xe[i];
    xu[i] = (v >= 0.0 || v != v) ? v : 0.0;
  }
  __syncthreads();
  double m = 0.0;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  int c = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double le = 0.0, lu = 0.0;
    for (int o = -beta; o <= beta; ++o) {
      const int j = i + o;
      if (j < 0 || j >= n) continue;
      const double a = L[(size_t)(beta + o) * n + i];
      le = fma(a, xe[j], le);
      lu = fma(a, xu[j], lu);
    }
    const double lam = le - f[(size_t)b * n + i];
    const double r = lu - f[(size_t)b * n + i];
    const double mn = fabs((xu[i] <= r || xu[i] != xu[i]) ? xu[i] : r);
    m = ((m != m) | (mn != mn)) ? qnan : (mn > m ? mn : m);
    const uint8_t na = xe[i] < lam ? 1 : 0;
    c |= na != act[(size_t)b * n + i];
    nact[(size_t)b * n + i] = na;
  }
  if (c) chg = 1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w2 = __shfl_xor_sync(0xffffffffu, m, o);
    m = ((m != m) | (w2 != w2)) ? qnan : (w2 > m ? w2 : m);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = red[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      const double x2 = red[k];
      r = ((r != r) | (x2 != x2)) ? qnan : (x2 > r ? x2 : r);
    }
    res[b] = r;
    changed[b] = chg;
  }
}

}  // namespace paqif

extern "C" int paqif_lcp_pin_batch(int64_t B, int64_t n, int64_t beta, const double* bands,
                                   const double* f, const uint8_t* active, double* lmod,
                                   double* fmod, void* stream) {
  if (B < 0 || n < 1 || beta < 0) return set_arg_error("paqif_lcp_pin_batch");
  if (B == 0) return PAQIF_OK;
  const int nd = 2 * (int)beta + 1;
  const unsigned gx = (unsigned)((nd * n + 255) / 256 < 1024 ? (nd * n + 255) / 256 : 1024);
  lcp_pin_kernel<<<dim3(gx, (unsigned)B), 256, 0, (cudaStream_t)stream>>>((int)n, (int)beta, bands,
                                                                         f, active, lmod, fmod);
  return check_launch("paqif_lcp_pin_batch");
}

extern "C" int paqif_lcp_pass_batch(int64_t B, int64_t n, int64_t beta, const double* bands,
                                    const double* f, const double* u_eval,
                                    const uint8_t* active, double* u, uint8_t* new_active,
                                    double* res, int32_t* changed, void* stream) {
  if (B < 0 || n < 1 || beta < 0) return set_arg_error("paqif_lcp_pass_batch");
  if (B == 0) return PAQIF_OK;
  lcp_pass_kernel<<<(unsigned)B, 256, 0, (cudaStream_t)stream>>>((int)n, (int)beta, bands, f,
                                                                u_eval, active, u, new_active, res,
                                                                changed);
  return check_launch("paqif_lcp_pass_batch");
}
