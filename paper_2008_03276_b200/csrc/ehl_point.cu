// EHL point contact (configs 4/5): one outer iteration of solve_ehl in the
// reference's Gauss-Seidel order (paqif/ehl/solver.py:76-128 then
// ehl/sweeps.py:421-518), driven by a native host loop over the grid lines.
//
// Device state mirrors FilmModel's bookkeeping (ehl/film.py:83-155): the
// deformation base of the last full evaluation plus up to 9 pending line
// updates whose exact contribution is added to the few film rows/columns a
// line needs; a fold (full FFT deformation, fft_deform.cuh) runs as soon as
// more than 8 are pending, decided on the device (gated kernels).
//
// Per line: pt_films (multi-CTA: base + pending corrections for the 3
// rows / <=4 columns the line reads) -> pt_xline / pt_yline (one CTA:
// rheology, limited faces, residual, assembly with the bad-row fix, AQIF
// line solve on warp 0 with the reference's fallback ladder, clip, immediate
// update or deferred weighted change, pending note) -> gated fold.
#include <cfloat>
#include <cstdlib>
#include <vector>
#include "ehl_common.cuh"
#include "aqif2.cuh"
#include "aqif1.cuh"
#include "fft_deform.cuh"
#include "fft_shard.cuh"
#include "capi_util.cuh"

extern "C" {
#include "../../include/paqif_ehl.h"
}

namespace paqif {

constexpr int kPtThreads = 256;
constexpr int kLineBeta = 2;
// line system (5 x n_sys band, right side, AQIF pivot records), doubles
__host__ __device__ inline size_t pt_sys_doubles(int n_sys) {
  return aqif2_band_doubles(n_sys) + aqif2_rhs_doubles(n_sys) + (size_t)(n_sys / 2 + 1) * kRec2;
}
constexpr int kMaxPending = 9;
enum { kMCount = 0, kMGate = 1, kMAnyW = 2, kMAxis = 3, kMIdx = 12, kMErr = 21, kMStop = 22,
       kMSize = 24 };
// meta[kMStop] != 0: a device-driven loop (paqif_ehl_point_drive_steps) has
// stopped -- every kernel of the later enqueued iterations returns at once
#define PT_LIVE(meta) \
  if ((meta)[kMStop]) return

// per-sweep controls (the public sweep variants of sweeps.py / solver.py)
struct SweepCtl {
  int sel;         // assembly: -1 by min(eps)/h (hybrid), 0 Newton (Ls0/Ls1), 1 weighted (Ls4/Ls5)
  int defer;       // update: -1 deferred iff weighted (_hybrid_x_sweep), 0 immediate, 1 deferred
  int nu_variant;  // 0 Ls1/Ls4 kernel strength, 1 Ls0/Ls5 (kernel_nu)
  double omega;
};

struct PointDev {
  int n, N, n_sys;
  double* u;
  double* geom;
  double* table;
  double* dbase;
  double* films;    // 4 x N
  double* sigma;    // N x N
  double* pend;     // kMaxPending x N
  int* meta;        // kMSize ints
  double* scal;     // [0] h0, [1] res, [2] deficit, [3] comp max bits, [4] worst |resid| bits
  double* scratch;  // line system when it does not fit in shared memory
  int sys_in_smem;
  unsigned long long* prof;  // dev phase timing (PAQIF_PT_PROF=1), else null
  int32_t* xinfo;   // n-1: newton tag | rung << 4
  int32_t* yinfo;   // n-1: rung
  double* film_out; // N x N
  double* rcache;   // 8 x N: rheology (eps, rho) of the points a line reads
  // batched runs of deferred x-lines (see enqueue_x_sweep)
  double* run_films;  // N x N: films of rows a-1 .. b of a run [a, b)
  double* run_rc;     // 2 x N x N: their eps (first N x N) and rho
  int32_t* run_flag;  // N: line a+l is deferred (by its own decision)
  int32_t* done;      // N: line j was solved inside a batched run
  double* run_scratch;  // kRunCtas line systems when they do not fit in shared memory
  double* fpart;        // films: per-k-segment partial corrections (kFilmSegMax x 4 x N)
};
constexpr int kRunCtas = 148;

__device__ __forceinline__ double rheo_eps(double u, double film, const paqif_ehl_point_cfg& c,
                                           double& rho) {
  double eta;
  if (c.compressible) {
    const double p = u * c.p_hertz;
    rho = (kDensA + kDensB * p) / (kDensA + p);
    const double arg = (c.alpha * c.p0 / c.z) * (-1.0 + pow(1.0 + p / c.p0, c.z));
    eta = exp(np_minimum(arg, 200.0));
  } else {
    rho = 1.0;
    eta = 1.0;
  }
  const double coeff = rho / (eta * c.lam);
  const double gap = np_maximum(film, 1e-8);
  return coeff * (gap * gap * gap);
}

// Pending-line corrections of the films of L <= 4 lines when every pending
// update lies along the sweep axis (the common case): per pending p and
// output line l a Toeplitz product  sum_k t_{|line - ell_p|}[|idx - k|]
// delta_p[k].  One warp per (128 outputs, k segment of 128, p):
// register-tiled, 4 consecutive outputs per lane, one shared load of the
// kernel window and one broadcast delta per 4 FMAs, so a single line's
// films fill the GPU.  Writes part[((p * nseg + seg) * 4 + l) * N + idx];
// pt_films_kernel sums the parts in a fixed order.  Does nothing when any
// pending update is cross-axis (pt_films_kernel then does it all).
constexpr int kFilmKS = 128;     // k per segment
constexpr int kFilmChunk = 128;  // outputs per warp: 32 lanes x 4
constexpr int kFilmSegMax = 32;  // N <= 4096
__global__ void __launch_bounds__(32) pt_films_part_kernel(PointDev d, int mode, int first, int L,
                                                           const int32_t* skip) {
  PT_LIVE(d.meta);
  if (skip && *skip) return;
  const int count = d.meta[kMCount];
  const int p = blockIdx.z;
  if (p >= count) return;
  for (int q = 0; q < count; ++q)
    if (d.meta[kMAxis + q] != mode) return;
  const int N = d.N;
  const int nch = (N + kFilmChunk - 1) / kFilmChunk, nseg = gridDim.y;
  const int l = blockIdx.x / nch, ch = blockIdx.x % nch, seg = blockIdx.y;
  if (l >= L) return;
  const int line = first + l;
  const int idx0 = ch * kFilmChunk, k0 = seg * kFilmKS;
  const int k1 = k0 + kFilmKS < N ? k0 + kFilmKS : N;
  const int nk = k1 - k0;
  __shared__ double sd[kFilmKS];
  __shared__ double se[kFilmChunk + kFilmKS + 4];  // se[1 + q] = t[|mlo + q|], se[0] = 0
  const int mlo = idx0 - (k1 - 1);
  const int nw = kFilmChunk + nk - 1;
  const double* __restrict__ delta = d.pend + (size_t)p * N;
  const double* __restrict__ tr = d.table + (size_t)abs(line - d.meta[kMIdx + p]) * N;
  const int lane = threadIdx.x;
  if (lane == 0) se[0] = 0.0;
  for (int q = lane; q < nk; q += 32) sd[q] = delta[k0 + q];
  for (int q = lane; q < nw; q += 32) {
    const int m = abs(mlo + q);
    se[1 + q] = m < N ? tr[m] : 0.0;
  }
  __syncwarp();
  // output idx0 + 4 lane + i at k0 + kk reads se[4 lane + i + nk - kk]
  int e = 4 * lane + nk;
  double w0 = se[e], w1 = se[e + 1], w2 = se[e + 2], w3 = se[e + 3];
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  for (int k = 0; k < nk; ++k) {
    const double dk = sd[k];
    acc0 = fma(w0, dk, acc0);
    acc1 = fma(w1, dk, acc1);
    acc2 = fma(w2, dk, acc2);
    acc3 = fma(w3, dk, acc3);
    --e;
    w3 = w2;
    w2 = w1;
    w1 = w0;
    w0 = se[e];
  }
  double* out = d.fpart + ((size_t)(p * nseg + seg) * 4 + l) * N;
  const int i0 = idx0 + 4 * lane;
  if (i0 < N) out[i0] = acc0;
  if (i0 + 1 < N) out[i0 + 1] = acc1;
  if (i0 + 2 < N) out[i0 + 2] = acc2;
  if (i0 + 3 < N) out[i0 + 3] = acc3;
}

// films of `L` consecutive rows (mode 0) or columns (mode 1) starting at
// `first` (FilmModel.film_rows / film_cols, film.py:98-146).  With pending
// line updates every output is a length-N dot product per update: one warp
// per output, lanes striding the sum (coalesced table/delta reads), four
// independent accumulators, shuffle reduction.  Without pending updates a
// thread per output.  Launch: kPtFilmWarps warps per block, enough blocks
// for L*N warps.
constexpr int kPtFilmWarps = 8;
__global__ void __launch_bounds__(32 * kPtFilmWarps) pt_films_kernel(PointDev d,
                                                                     paqif_ehl_point_cfg c,
                                                                     int mode, int first, int L,
                                                                     double* films_out,
                                                                     double* rc_out,
                                                                     size_t rho_off,
                                                                     const int32_t* skip,
                                                                     int nseg) {
  PT_LIVE(d.meta);
  if (skip && *skip) return;  // the line was solved in a batched run
  const int N = d.N;
  const int count = d.meta[kMCount];
  const double h0 = d.scal[0];
  auto gidx = [&](int line, int idx) {
    return mode == 0 ? (size_t)line * N + idx : (size_t)idx * N + line;
  };
  auto base = [&](int line, int idx) {
    const size_t g = gidx(line, idx);
    return (h0 + d.geom[g]) + d.dbase[g];
  };
  // film value o plus its rheology (eps, rho) for the line kernel: the
  // pointwise work of a line spread over the whole GPU
  auto emit = [&](int o, int line, int idx, double v) {
    films_out[o] = v;
    double rho;
    rc_out[o] = rheo_eps(d.u[gidx(line, idx)], v, c, rho);
    rc_out[rho_off + o] = rho;
  };
  if (count == 0) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < L * N) emit(o, first + o / N, o % N, base(first + o / N, o % N));
    return;
  }
  bool cross = false;
  for (int p = 0; p < count; ++p) cross |= d.meta[kMAxis + p] != mode;
  if (nseg > 0 && !cross) {
    // the parts of pt_films_part_kernel: one thread per output sums them in a
    // fixed order (coalesced reads) and evaluates the rheology
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= L * N) return;
    const int l = o / N, idx = o % N;
    const double* src = d.fpart + (size_t)l * N + idx;
    double v = 0.0;
    for (int q = 0; q < count * nseg; ++q) v += src[(size_t)q * 4 * N];
    emit(o, first + l, idx, base(first + l, idx) + v);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int o = blockIdx.x * kPtFilmWarps + (threadIdx.x >> 5);
  if (o >= L * N) return;
  const int l = o / N, idx = o % N;
  const int line = first + l;
  double corr = 0.0;
  for (int p = 0; p < count; ++p) {
    const int axis = d.meta[kMAxis + p], ell = d.meta[kMIdx + p];
    const double* __restrict__ delta = d.pend + (size_t)p * N;
    // same axis: Toeplitz row |line-ell| at |idx-k|; cross axis: kernel row
    // |idx-ell| at |line-k| (film.py:114-117, 131-134; symmetric table)
    const bool same = axis == mode;
    const double* __restrict__ tr = d.table + (size_t)abs(same ? line - ell : idx - ell) * N;
    const int c = same ? idx : line;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int k = lane;
    for (; k + 96 < N; k += 128) {
      a0 = fma(tr[abs(c - k)], delta[k], a0);
      a1 = fma(tr[abs(c - k - 32)], delta[k + 32], a1);
      a2 = fma(tr[abs(c - k - 64)], delta[k + 64], a2);
      a3 = fma(tr[abs(c - k - 96)], delta[k + 96], a3);
    }
    for (; k < N; k += 32) a0 = fma(tr[abs(c - k)], delta[k], a0);
    double sp = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, off);
    corr += sp;
  }
  if (lane == 0) emit(o, line, idx, base(line, idx) + corr);
}

__device__ __forceinline__ double block_min(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) r = fmin(r, red[w]);
  __syncthreads();
  return r;
}

// assemble_line_system row for an x-line of the point contact (hy = h,
// ey terms, bad-row fix; sweeps.py:157-267).  jac: 0 scheme, 1 first-order,
// 2 diagonal.  ex/ey already carry the factor h (sweeps.py:329-334).
__device__ __forceinline__ void point_row(double rw, double rc, double re, double ex_p,
                                          double ex_m, double ey_p, double ey_m, double phi_p,
                                          double phi_m, double h, bool weighted, int jac,
                                          double ks0, double ks1, double* e) {
  line_row_entries(rw, rc, re, ex_p, ex_m, ey_p, ey_m, phi_p, phi_m, h, h, weighted, jac, ks0,
                   ks1, e);
}

// worst |resid| of the sweep (python max over lines ignores NaN lines)
__device__ __forceinline__ void note_worst(PointDev& d, double v, double* red) {
  const double m = block_max(v, red);
  if (threadIdx.x == 0 && m > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(&d.scal[4]),
              (unsigned long long)__double_as_longlong(m));
}

struct PtShared {
  double red[32];
  int flag;
  int any;
  int pad[2];
};

// write one assembled row (padded-matrix semantics) of the line system
__device__ __forceinline__ void put_row(double* band, double* rhs, int n_sys, int n_int, int r,
                                        const double* e, double rr) {
#pragma unroll
  for (int dd = 0; dd < 5; ++dd) {
    const int col = r + dd - kLineBeta;
    const bool keep = r < n_int ? (col >= 0 && col < n_sys) : (dd == kLineBeta);
    band2_ref(band, n_sys, r, dd - kLineBeta) = keep ? e[dd] : 0.0;
  }
  rhs[kBandPad + r] = rr;
}

// the same for the tridiagonal column systems (aqif1 layout, offsets -1..1
// from e[1..3])
__device__ __forceinline__ void put_row1(double* band, double* rhs, int n_sys, int n_int, int r,
                                         const double* e, double rr) {
#pragma unroll
  for (int dd = 1; dd < 4; ++dd) {
    const int col = r + dd - kLineBeta;
    const bool keep = r < n_int ? (col >= 0 && col < n_sys) : (dd == kLineBeta);
    band1_ref(band, n_sys, r, dd - kLineBeta) = keep ? e[dd] : 0.0;
  }
  rhs[kBandPad + r] = rr;
}

// x-line j of _hybrid_x_sweep (solver.py:91-114) with _line_quantities
// (sweeps.py:318-341) and assemble_line_system's point terms (sweeps.py:157-267)
// where an x-line reads its films and rheology: rows j-1, j, j+1 at
// films[0..3N), eps at rc[0..3N), rho at rc[rho_off ..)
struct XSrc {
  const double* films;
  const double* rc;
  size_t rho_off;
};

// One x-line of the point contact (see pt_xline_kernel); all threads of
// the CTA call.  sysb: the line system's storage.
template <bool EXACT, bool SMEM>
__device__ void xline_body(PointDev& d, const paqif_ehl_point_cfg& c, const SweepCtl& ctl, int j,
                           const XSrc src, double* sysb, PtShared& S) {
  const int n = d.n, N = d.N, n_int = n - 1, n_sys = d.n_sys;
  const double h = c.h;
  const double* u = d.u;
  const double* F = src.films;  // rows j-1, j, j+1
  long long tp0 = clock64(), tp1 = 0, tp2 = 0, tp3 = 0;
  auto film = [&](int r, int i) { return F[(size_t)(r - (j - 1)) * N + i]; };
  auto eps_at = [&](int r, int i, double& rho) {
    return rheo_eps(u[(size_t)r * N + i], film(r, i), c, rho);
  };
  // pass 1: the rheology of rows j-1, j, j+1 came with the films
  // (pt_films_kernel); min(eps_line)/h and max|q_line|
  const double* E0 = src.rc;
  const double* E1 = E0 + N;
  const double* E2 = E1 + N;
  const double* R1 = src.rc + src.rho_off + N;
  double emin = INFINITY, qmax = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    emin = fmin(emin, E1[i]);
    qmax = fmax(qmax, fabs(R1[i] * film(j, i)));
  }
  const double ratio = block_min(emin, S.red) / h;
  const double gfloor = 1e-12 * fmax(block_max(qmax, S.red), kRatioGuard);
  tp1 = clock64();
  const bool weighted = ctl.sel < 0 ? !(ratio > kSwitch) : ctl.sel == 1;
  const bool deferred = ctl.defer < 0 ? weighted : ctl.defer == 1;
  const bool newton = !deferred;  // immediate update (and pending note)
  // kernel sensitivities (film.sensitivity, point: table[|d|][|off|])
  const double* t = d.table;
  const double s00 = t[0], s10 = t[N], s20 = t[2 * N], s01 = t[1], s11 = t[N + 1];
  const double nu = ctl.nu_variant == 0 ? (2.0 - c.kappa) / 2.0
                                   : (2.0 - c.kappa) / 2.0 + (1.0 - c.kappa) / 4.0;
  double ks0, ks1;
  if (weighted) {
    ks0 = nu * (s00 - 0.25 * (2.0 * s10 + 2.0 * s01));
    ks1 = nu * (s10 - 0.25 * (s00 + s20 + 2.0 * s11));
  } else {
    ks0 = s00;
    ks1 = s10;
  }
  double* band = sysb;
  double* rhs = band + aqif2_band_doubles(n_sys);
  double* rec = rhs + aqif2_rhs_doubles(n_sys);
  aqif2_zero_pads(band, rhs, n_sys);
  int rung = 0;
  int st = 1;
  double worst = 0.0;
  for (; rung < 3; ++rung) {
    for (int r = threadIdx.x; r < n_sys; r += blockDim.x) {
      double e[5] = {0.0, 0.0, 1.0, 0.0, 0.0};
      double rr = 0.0;
      if (r < n_int) {
        const int i = r + 1;
        const double rw = R1[i - 1], rc = R1[i], re = R1[i + 1];
        const double ew = E1[i - 1], ec = E1[i], ee = E1[i + 1];
        const double es = E0[i], en = E2[i];
        const double qw = rw * film(j, i - 1), qc = rc * film(j, i), qe = re * film(j, i + 1);
        double qww = 0.0;
        if (i >= 2) qww = R1[i - 2] * film(j, i - 2);
        const double dqi = qe - qc, dqm = qc - qw;
        const double php = limiter_wplus(gratio(dqi, dqm, gfloor), c.limiter, c.kappa);
        const double phm = i >= 2 ? limiter_wplus(gratio(dqm, qw - qww, gfloor), c.limiter, c.kappa)
                                  : 0.0;
        const double fd = (qc + 0.5 * php * dqi) - (qw + 0.5 * phm * dqm);
        const double ex_p = 0.5 * (ec + ee) * h, ex_m = 0.5 * (ec + ew) * h;
        const double ey_p = 0.5 * (ec + en) * h, ey_m = 0.5 * (ec + es) * h;
        const double uc = u[(size_t)j * N + i];
        rr = (ex_p * (u[(size_t)j * N + i + 1] - uc) + ex_m * (u[(size_t)j * N + i - 1] - uc)) / h +
             (ey_p * (u[(size_t)(j + 1) * N + i] - uc) + ey_m * (u[(size_t)(j - 1) * N + i] - uc)) / h -
             h * fd;
        point_row(rw, rc, re, ex_p, ex_m, ey_p, ey_m, php, phm, h, weighted, rung, ks0, ks1, e);
        worst = fmax(worst, fabs(rr));
      }
      put_row(band, rhs, n_sys, n_int, r, e, rr);
    }
    if (rung == 0) note_worst(d, worst, S.red);
    if (rung == 0) tp2 = clock64();
    st = aqif2_solve<EXACT>(band, rhs, n_sys, rec, band, &S.flag);
    if (rung == 0) tp3 = clock64();
    if (d.prof && threadIdx.x == 0 && (st & 2)) atomicAdd(&d.prof[5], 1ull);
    st &= 1;
    if (!st) break;
  }
  if (d.prof && threadIdx.x == 0) {
    atomicAdd(&d.prof[0], (unsigned long long)(tp1 - tp0));
    atomicAdd(&d.prof[1], (unsigned long long)(tp2 - tp1));
    atomicAdd(&d.prof[2], (unsigned long long)(tp3 - tp2));
    atomicAdd(&d.prof[4], 1ull);
  }
  if (st) {
    if (threadIdx.x == 0) {
      atomicOr(&d.meta[kMErr], 1);
      d.xinfo[j - 1] = (weighted ? 0 : 1) | (deferred ? 2 : 0) | (3 << 4);
    }
    return;
  }
  const double* x = band;  // aqif2_solve wrote x over the band
  int nz = 0, fin = 1;
  double* delta = d.pend + (size_t)d.meta[kMCount] * N;  // next pending slot (used if newton)
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    if (i >= 1 && i <= n - 1) {
      double sg = x[i - 1];
      fin &= isfinite(sg);
      sg = np_minimum(np_maximum(sg, -c.max_change), c.max_change);
      if (newton) {
        const double old = u[(size_t)j * N + i];
        const double nv = np_maximum(0.0, old + ctl.omega * sg);
        const double dl = nv - old;
        nz |= (dl != 0.0) || (dl != dl);
        delta[i] = dl;
        d.u[(size_t)j * N + i] = nv;
      } else {
        d.sigma[(size_t)j * N + i] = sg;
      }
    } else if (newton) {
      delta[i] = 0.0;
    }
  }
  nz = __syncthreads_or(nz);
  fin = __syncthreads_and(fin);
  if (threadIdx.x == 0) {
    if (!fin) atomicOr(&d.meta[kMErr], 2);
    d.xinfo[j - 1] = (weighted ? 0 : 1) | (deferred ? 2 : 0) | (rung << 4);
    if (newton && nz) {  // note_line_update("row", j, delta, u)
      const int p = d.meta[kMCount];
      d.meta[kMAxis + p] = 0;
      d.meta[kMIdx + p] = j;
      d.meta[kMCount] = p + 1;
      if (p + 1 > 8) d.meta[kMGate] = 1;
    }
    if (deferred) d.meta[kMAnyW] = 1;
    if (d.prof) atomicAdd(&d.prof[3], (unsigned long long)(clock64() - tp3));
  }
}

template <bool EXACT, bool SMEM>
__global__ void __launch_bounds__(kPtThreads, 1) pt_xline_kernel(PointDev d, paqif_ehl_point_cfg c,
                                                              SweepCtl ctl, int j) {
  PT_LIVE(d.meta);
  if (d.done[j]) return;  // solved inside a batched run of deferred lines
  extern __shared__ __align__(16) double xsm[];
  PtShared& S = *reinterpret_cast<PtShared*>(xsm);
  // SMEM: the line system in shared memory (address space known to the
  // compiler -> LDS/STS in the solver's level loops)
  double* sysb = SMEM ? xsm + sizeof(PtShared) / 8 : d.scratch;
  xline_body<EXACT, SMEM>(d, c, ctl, j, XSrc{d.films, d.rcache, 4 * (size_t)d.N}, sysb, S);
}

// Deferred decision of every line of a candidate run [a, a+L): the same
// min(eps)/h test as the line kernel's pass 1, on the run's rheology rows
// (one block per line).
__global__ void pt_run_flags_kernel(PointDev d, paqif_ehl_point_cfg c, SweepCtl ctl, int L) {
  PT_LIVE(d.meta);
  __shared__ double red[32];
  const int l = blockIdx.x;
  if (l >= L) return;
  const int N = d.N;
  const double* E = d.run_rc + (size_t)(l + 1) * N;
  double emin = INFINITY;
  for (int i = threadIdx.x; i < N; i += blockDim.x) emin = fmin(emin, E[i]);
  const double ratio = block_min(emin, red) / c.h;
  const bool weighted = ctl.sel < 0 ? !(ratio > kSwitch) : ctl.sel == 1;
  const bool deferred = ctl.defer < 0 ? weighted : ctl.defer == 1;
  if (threadIdx.x == 0) d.run_flag[l] = deferred ? 1 : 0;
}

// A run of deferred x-lines [a, a+L) solved side by side: deferred lines
// leave u, the pending list and the films untouched, so in the reference's
// Gauss-Seidel order each of them sees the same state as the run's first
// line -- identical results, any order.  CTA-strided lines; line a+l is
// solved only if lines a..a+l are all deferred (run_flag), else it is left
// to the per-line launches that follow (done[] stays 0).
template <bool EXACT, bool SMEM>
__global__ void __launch_bounds__(kPtThreads, 1) pt_xrun_kernel(PointDev d, paqif_ehl_point_cfg c,
                                                             SweepCtl ctl, int a, int L) {
  PT_LIVE(d.meta);
  extern __shared__ __align__(16) double xsm[];
  PtShared& S = *reinterpret_cast<PtShared*>(xsm);
  double* sysb = SMEM ? xsm + sizeof(PtShared) / 8
                      : d.run_scratch + (size_t)blockIdx.x * pt_sys_doubles(d.n_sys);
  const int N = d.N;
  for (int l = blockIdx.x; l < L; l += gridDim.x) {
    int ok = 1;
    for (int q = threadIdx.x; q <= l; q += blockDim.x) ok &= d.run_flag[q];
    if (!__syncthreads_and(ok)) return;  // later lines of this CTA fail the prefix too
    const XSrc src{d.run_films + (size_t)l * N, d.run_rc + (size_t)l * N, (size_t)N * N};
    xline_body<EXACT, SMEM>(d, c, ctl, a + l, src, sysb, S);
    __syncthreads();
    if (threadIdx.x == 0) d.done[a + l] = 1;
  }
}

// deferred weighted changes of the x-sweep (solver.py:115-127)
__global__ void pt_weighted_kernel(PointDev d, double omega) {
  PT_LIVE(d.meta);
  if (d.meta[kMAnyW] == 0) return;
  const int N = d.N, n = d.n;
  const size_t total = (size_t)N * N;
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(g / N), i = (int)(g % N);
    const double* s = d.sigma;
    double sp = 0.0;
    if (i >= 1) sp += s[g - 1];
    if (i < n) sp += s[g + 1];
    if (j >= 1) sp += s[g - N];
    if (j < n) sp += s[g + N];
    double v = np_maximum(0.0, d.u[g] + omega * (s[g] - 0.25 * sp));
    if (i == 0 || i == n || j == 0 || j == n) v = 0.0;
    d.film_out[g] = v;  // staged: u must not change while neighbours are read
  }
}
__global__ void pt_copy_kernel(double* dst, const double* src, size_t count, const int* flag,
                               const int* meta) {
  PT_LIVE(meta);
  if (flag && *flag == 0) return;
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < count;
       g += (size_t)gridDim.x * blockDim.x)
    dst[g] = src[g];
}
__global__ void pt_set_gate_kernel(int* meta, int from_anyw) {
  PT_LIVE(meta);
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (!from_anyw || meta[kMAnyW]) meta[kMGate] = 1;
  }
}

// column i of column_sweep (sweeps.py:437-517)
template <bool EXACT, bool SMEM>
__global__ void __launch_bounds__(kPtThreads, 1) pt_yline_kernel(PointDev d, paqif_ehl_point_cfg c,
                                                              SweepCtl ctl, int i) {
  PT_LIVE(d.meta);
  extern __shared__ __align__(16) double ysm[];
  PtShared& S = *reinterpret_cast<PtShared*>(ysm);
  double* sysb = SMEM ? ysm + sizeof(PtShared) / 8 : d.scratch;
  const int n = d.n, N = d.N, n_int = n - 1, n_sys = d.n_sys;
  const double h = c.h;
  const int lo = i - 2 > 0 ? i - 2 : 0;
  const int L = i + 2 - lo, pos = i - lo;
  const double* u = d.u;
  const double* F = d.films;  // columns lo..i+1, indexed [l][m]
  auto film = [&](int l, int m) { return F[(size_t)l * N + m]; };
  auto eps_at = [&](int l, int m, double& rho) {
    return rheo_eps(u[(size_t)m * N + (lo + l)], film(l, m), c, rho);
  };
  // the rheology of the bundle's L columns came with the films
  const double* EC = d.rcache;          // [l][m] eps
  const double* RC = d.rcache + 4 * N;  // [l][m] rho
#ifdef PAQIF_DEV_PROF
  const long long y0 = clock64();
  long long y1 = 0, y2 = 0, y3 = 0;
#endif
  double qmax = 0.0;
  for (int k = threadIdx.x; k < L * N; k += blockDim.x) {
    const int l = k / N, m = k % N;
    qmax = fmax(qmax, fabs(RC[k] * film(l, m)));
  }
  const double gfloor = 1e-12 * fmax(block_max(qmax, S.red), kRatioGuard);
#ifdef PAQIF_DEV_PROF
  y1 = clock64();
#endif
  const double* t = d.table;
  const double s00 = t[0], s10 = t[N], s01 = t[1], s11 = t[N + 1];
  double* band = sysb;
  // tridiagonal: the reference factors these with beta = 1 (aqif1.cuh)
  double* rhs = band + aqif1_band_doubles(n_sys);
  double* rec = rhs + aqif1_rhs_doubles(n_sys);
  aqif1_zero_pads(band, rhs, n_sys);
  int st = 1, rung = 0;
  double worst = 0.0;
  for (; rung < 2; ++rung) {  // 0: tridiagonal system, 1: diagonal fallback
    for (int r = threadIdx.x; r < n_sys; r += blockDim.x) {
      double e[5] = {0.0, 0.0, 1.0, 0.0, 0.0};
      double rr = 0.0;
      if (r < n_int) {
        const int jj = r + 1;
        auto ce = [&](int l, int m) { return EC[(size_t)l * N + m]; };
        auto cr = [&](int l, int m) { return RC[(size_t)l * N + m]; };
        const double rc = cr(pos, jj), rw = cr(pos - 1, jj), re = cr(pos + 1, jj);
        const double ec = ce(pos, jj), ew = ce(pos - 1, jj), ee = ce(pos + 1, jj);
        const double es = ce(pos, jj - 1), en = ce(pos, jj + 1);
        const double ey_p = 0.5 * (ec + en) * h, ey_m = 0.5 * (ec + es) * h;
        const double ex_p = 0.5 * (ec + ee) * h, ex_m = 0.5 * (ec + ew) * h;
        const double qc = rc * film(pos, jj), qw = rw * film(pos - 1, jj), qe = re * film(pos + 1, jj);
        const double dq_p = qe - qc, dq_m = qc - qw;
        const double php = limiter_wplus(gratio(dq_p, dq_m, gfloor), c.limiter, c.kappa);
        double phm = 0.0;
        if (pos >= 2) {
          const double qww = cr(pos - 2, jj) * film(pos - 2, jj);
          phm = limiter_wplus(gratio(dq_m, qw - qww, gfloor), c.limiter, c.kappa);
        }
        const double flux_p = qc + 0.5 * php * dq_p;
        const double flux_m = qw + 0.5 * phm * dq_m;
        const double uc = u[(size_t)jj * N + i];
        rr = (ex_p * (u[(size_t)jj * N + i + 1] - uc) + ex_m * (u[(size_t)jj * N + i - 1] - uc)) / h +
             (ey_p * (u[(size_t)(jj + 1) * N + i] - uc) + ey_m * (u[(size_t)(jj - 1) * N + i] - uc)) / h -
             h * (flux_p - flux_m);
        worst = fmax(worst, fabs(rr));
        if (rung == 0) {
          const double a_p = 1.0 - 0.5 * php, b_p = 0.5 * php;
          const double a_m = 1.0 - 0.5 * phm, b_m = 0.5 * phm;
          double c_diag = -h * ((a_p - b_m) * rc * s00 + (b_p * re - a_m * rw) * s10);
          double c_off = -h * ((a_p - b_m) * rc * s01 + (b_p * re - a_m * rw) * s11);
          double diag_full = -(ey_p + ey_m + ex_p + ex_m) / h + c_diag;
          const double floor_ = 0.05 * h * fabs(rc) * s00;
          if (fabs(diag_full) < floor_) {
            c_diag = -h * (rc * s00 - rw * s10);
            c_off = -h * (rc * s01 - rw * s11);
            diag_full = -(ey_p + ey_m + ex_p + ex_m) / h + c_diag;
          }
          e[0] = 0.0;
          e[1] = -(ey_m / h + c_off);
          e[2] = -diag_full;
          e[3] = -(ey_p / h + c_off);
          e[4] = 0.0;
        } else {
          e[0] = 0.0; e[1] = 0.0; e[3] = 0.0; e[4] = 0.0;
          e[2] = (ey_p + ey_m + ex_p + ex_m) / h + h * fabs(rc) * s00;
        }
      }
      put_row1(band, rhs, n_sys, n_int, r, e, rr);
    }
    if (rung == 0) note_worst(d, worst, S.red);
#ifdef PAQIF_DEV_PROF
    if (rung == 0) y2 = clock64();
#endif
    st = aqif1_solve<EXACT>(band, rhs, n_sys, rec, band, &S.flag) & 1;
#ifdef PAQIF_DEV_PROF
    if (rung == 0) y3 = clock64();
#endif
    if (!st) break;
  }
  if (st) {
    if (threadIdx.x == 0) {
      atomicOr(&d.meta[kMErr], 4);
      d.yinfo[i - 1] = 3;
    }
    return;
  }
  const double* x = band;  // aqif1_solve wrote x over the band
  int nz = 0, fin = 1;
  double* delta = d.pend + (size_t)d.meta[kMCount] * N;
  for (int m = threadIdx.x; m < N; m += blockDim.x) {
    if (m >= 1 && m <= n - 1) {
      double sg = x[m - 1];
      fin &= isfinite(sg);
      sg = np_minimum(np_maximum(sg, -c.max_change), c.max_change);
      const double old = u[(size_t)m * N + i];
      const double nv = np_maximum(0.0, old + ctl.omega * sg);
      const double dl = nv - old;
      nz |= (dl != 0.0) || (dl != dl);
      delta[m] = dl;
      d.u[(size_t)m * N + i] = nv;
    } else {
      delta[m] = 0.0;
    }
  }
  nz = __syncthreads_or(nz);
  fin = __syncthreads_and(fin);
  if (threadIdx.x == 0) {
    if (!fin) atomicOr(&d.meta[kMErr], 8);
    d.yinfo[i - 1] = rung;
    if (nz) {  // note_line_update("col", i, delta, u)
      const int p = d.meta[kMCount];
      d.meta[kMAxis + p] = 1;
      d.meta[kMIdx + p] = i;
      d.meta[kMCount] = p + 1;
      if (p + 1 > 8) d.meta[kMGate] = 1;
    }
  }
#ifdef PAQIF_DEV_PROF
  if (threadIdx.x == 0 && i == d.n / 2)
    printf("[y_prof] n=%d pass1 %lld assemble %lld solve %lld update %lld\n", d.n, y1 - y0,
           y2 - y1, y3 - y2, clock64() - y3);
#endif
}

// force balance (sweeps.py:521-535, weight h^2)
// drv (device-driven loop): balance only on the reference's schedule,
// (outer + 1) % force_every == 0 with outer from the drive record
__global__ void pt_force_kernel(PointDev d, paqif_ehl_point_cfg c,
                                const paqif_ehl_line_drive* drv) {
  PT_LIVE(d.meta);
  if (drv && (drv->outer + 1) % c.force_every != 0) return;
  __shared__ double red[32];
  const size_t total = (size_t)d.N * d.N;
  double part = 0.0;
  for (size_t g = threadIdx.x; g < total; g += blockDim.x) part += d.u[g];
  const double sum = block_sum(part, red);
  if (threadIdx.x == 0) {
    const double deficit = c.load_target - (c.h * c.h) * sum;
    const double stp = np_minimum(np_maximum(c.relax_c * deficit, -c.max_h0_step), c.max_h0_step);
    d.scal[0] = d.scal[0] - stp;
    d.scal[2] = deficit;
  }
}

// reynolds_residual_field (2-D, sweeps.py:124-140) and the complementarity
// residual; one CTA per row; film_out = h0 + geometry + deformation
__global__ void pt_residual_kernel(PointDev d, paqif_ehl_point_cfg c) {
  PT_LIVE(d.meta);
  __shared__ double red[32];
  const int n = d.n, N = d.N;
  const int j = blockIdx.x;
  const double h = c.h, h0 = d.scal[0];
  auto film = [&](int r, int i) { return (h0 + d.geom[(size_t)r * N + i]) + d.dbase[(size_t)r * N + i]; };
  auto eps_at = [&](int r, int i, double& rho) {
    return rheo_eps(d.u[(size_t)r * N + i], film(r, i), c, rho);
  };
  for (int i = threadIdx.x; i < N; i += blockDim.x) d.film_out[(size_t)j * N + i] = film(j, i);
  double comp = 0.0;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  if (j >= 1 && j <= n - 1) {
    double qmax = 0.0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      double rho;
      eps_at(j, i, rho);
      qmax = fmax(qmax, fabs(rho * film(j, i)));
    }
    const double gfloor = 1e-12 * fmax(block_max(qmax, red), kRatioGuard);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      double r = 0.0;
      if (i >= 1 && i <= n - 1) {
        double rw, rc, re, rdum, rww = 0.0;
        const double ew = eps_at(j, i - 1, rw);
        const double ec = eps_at(j, i, rc);
        const double ee = eps_at(j, i + 1, re);
        const double es = eps_at(j - 1, i, rdum);
        const double en = eps_at(j + 1, i, rdum);
        const double qw = rw * film(j, i - 1), qc = rc * film(j, i), qe = re * film(j, i + 1);
        const double dqi = qe - qc, dqm = qc - qw;
        const double php = limiter_wplus(gratio(dqi, dqm, gfloor), c.limiter, c.kappa);
        double phm = 0.0;
        if (i >= 2) {
          eps_at(j, i - 2, rww);
          phm = limiter_wplus(gratio(dqm, qw - rww * film(j, i - 2), gfloor), c.limiter, c.kappa);
        }
        const double fd = (qc + 0.5 * php * dqi) - (qw + 0.5 * phm * dqm);
        const double exp_ = 0.5 * (ec + ee) * h, exm = 0.5 * (ec + ew) * h;
        const double eyp = 0.5 * (ec + en) * h, eym = 0.5 * (ec + es) * h;
        const double uc = d.u[(size_t)j * N + i];
        r = (exp_ * (d.u[(size_t)j * N + i + 1] - uc) + exm * (d.u[(size_t)j * N + i - 1] - uc)) / h +
            (eyp * (d.u[(size_t)(j + 1) * N + i] - uc) + eym * (d.u[(size_t)(j - 1) * N + i] - uc)) / h -
            h * fd;
      }
      const double m = fabs(np_minimum(d.u[(size_t)j * N + i], -r));
      comp = ((comp != comp) | (m != m)) ? qnan : (m > comp ? m : comp);
    }
  } else {
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double m = fabs(np_minimum(d.u[(size_t)j * N + i], -0.0));
      comp = ((comp != comp) | (m != m)) ? qnan : (m > comp ? m : comp);
    }
  }
  const double cm = block_nanmax(comp, red);
  if (threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&d.scal[3]),
              (unsigned long long)__double_as_longlong(cm));
}

__global__ void pt_finish_kernel(PointDev d, paqif_ehl_point_cfg c) {
  PT_LIVE(d.meta);
  if (threadIdx.x == 0 && blockIdx.x == 0) d.scal[1] = d.scal[3] / (c.h * c.h);
}

// zero `words` 4-byte words (the per-sweep resets), unless stopped
__global__ void pt_zero_kernel(uint32_t* p, size_t words, const int* meta) {
  PT_LIVE(meta);
  for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < words;
       g += (size_t)gridDim.x * blockDim.x)
    p[g] = 0u;
}

// solve_ehl's per-iteration bookkeeping and stop / divergence tests
// (ehl/solver.py:219-240, same comparisons in the same order) on the drive
// record, after the iteration's residual; a stop sets meta[kMStop].
// A line solve with every rung broken (err bits 0/2) or a non-finite change
// (bits 1/3) stops before the residual is recorded (the reference raises
// inside the sweep).
__global__ void pt_drive_kernel(PointDev d, paqif_ehl_point_cfg c, paqif_ehl_line_drive* drv,
                                double* hist_res, double* hist_def, int hist_cap) {
  PT_LIVE(d.meta);
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  paqif_ehl_line_drive& r = *drv;
  const int err = d.meta[kMErr];
  if (err & 5) {
    r.done = 4;
    d.meta[kMStop] = 1;
    return;
  }
  if (err & (10 | 64)) {  // non-finite change, or a sharded fold lost a peer
    r.done = 5;
    d.meta[kMStop] = 1;
    return;
  }
  const int k = r.outer;
  const int fb = (k + 1) % c.force_every == 0;
  const double res = d.scal[1], deficit = d.scal[2];
  if (hist_res && hist_cap > 0) {
    hist_res[k % hist_cap] = res;
    hist_def[k % hist_cap] = fb ? deficit : __longlong_as_double(0x7ff8000000000000ll);
  }
  if (fb) r.deficit = fabs(deficit);
  r.outer = k + 1;
  if (res <= r.tol && fabs(r.deficit) <= r.tol_fb) r.done = 1;
  else if (res < r.best) {
    r.best = res;
    r.grow = 0;
  } else {
    r.grow += 1;
    if (r.grow >= 20 && res > 1e3 * fmax(r.best, r.tol)) r.done = 2;
  }
  if (!r.done && r.outer >= r.max_outer) r.done = 3;
  if (r.done) d.meta[kMStop] = 1;
}

__global__ void pt_drive_begin_kernel(int* meta, const paqif_ehl_line_drive* drv) {
  if (threadIdx.x == 0 && blockIdx.x == 0) meta[kMStop] = drv->done != 0 ? 1 : 0;
}

}  // namespace paqif

using namespace paqif;

// ============================================================== native driver
struct paqif_ehl_point {
  paqif_ehl_point_cfg cfg;
  PointDev d;
  // FFT period: the next power of two >= 2n (exact on the central window for
  // any pressure, fft_deform.cuh)
  FftPlan plan;
  cudaStream_t st;
  std::vector<void*> allocs;
  size_t line_smem;
  // previous x-sweep's per-line tags (pinned), for predicting the runs of
  // deferred lines of the next one; valid once `xinfo_ev` completed
  int32_t* xinfo_prev = nullptr;
  cudaEvent_t xinfo_ev = nullptr;
  bool xinfo_valid = false;
  bool runs = true;  // PAQIF_PT_RUNS=0 solves every x-line on its own (A/B checks)
  std::vector<int32_t> pred;  // run-prediction tags for a device-driven chunk
  // sharded folds across ranks (fft_shard.cuh), after attach_peers
  unsigned* bar = nullptr;    // this rank's barrier words
  bool sharded = false;
  FoldPeers peers{};
  std::vector<void*> ipc_opened;
};

namespace {

template <class T>
T* dalloc(paqif_ehl_point* h, size_t count) {
  void* p = nullptr;
  if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
  h->allocs.push_back(p);
  cudaMemsetAsync(p, 0, count * sizeof(T), h->st);
  return (T*)p;
}

void fold(paqif_ehl_point* h) {
  if (h->sharded) {  // split over the ranks (fft_shard.cuh)
    fold_sharded(h->plan, h->d.u, h->peers, &h->d.meta[kMGate], &h->d.meta[kMCount],
                 &h->d.meta[kMErr], h->st);
    return;
  }
  // one cooperative launch; a no-op (gate == 0) costs one empty kernel
  fft_fold(h->plan, h->d.u, h->d.dbase, &h->d.meta[kMGate], &h->d.meta[kMCount], h->st);
}

int next_pow2(int v) {
  int P = 32;
  while (P < v) P <<= 1;
  return P;
}

bool alloc_plan(paqif_ehl_point* h, FftPlan& p, int P) {
  p.n = h->d.n;
  p.P = P;
  p.logP = 0;
  while ((1 << p.logP) < p.P) ++p.logP;
  p.W = dalloc<double2>(h, fft_w_elems(p.P));
  p.KT = dalloc<double2>(h, fft_kt_elems(p.P));
  p.tw = dalloc<double2>(h, p.P / 2 + 1);
  if (!p.W || !p.KT || !p.tw) return false;
  return fft_plan_kernel(p, h->d.table, h->st) == cudaSuccess;
}

}  // namespace

extern "C" paqif_ehl_point* paqif_ehl_point_create(const paqif_ehl_point_cfg* cfg,
                                                   const double* table, const double* geometry) {
  if (!cfg || cfg->n < 8 || cfg->n > 8192) {
    set_arg_error("ehl_point: bad cfg");
    return nullptr;
  }
  auto* h = new paqif_ehl_point();
  h->cfg = *cfg;
  if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return nullptr;
  }
  const int n = cfg->n, N = n + 1, n_int = n - 1;
  const int n_sys = (n_int + 1) % 2 == 0 ? n_int + 1 : n_int + 2;
  PointDev& d = h->d;
  d.n = n;
  d.N = N;
  d.n_sys = n_sys;
  const size_t NN = (size_t)N * N;
  d.u = dalloc<double>(h, NN);
  d.geom = dalloc<double>(h, NN);
  d.table = dalloc<double>(h, NN);
  d.dbase = dalloc<double>(h, NN);
  d.films = dalloc<double>(h, 4 * (size_t)N);
  d.sigma = dalloc<double>(h, NN);
  d.pend = dalloc<double>(h, (size_t)kMaxPending * N);
  d.meta = dalloc<int>(h, kMSize);
  d.scal = dalloc<double>(h, 8);
  const size_t sys_bytes = pt_sys_doubles(n_sys) * sizeof(double);
  d.sys_in_smem = sizeof(PtShared) + sys_bytes <= 227 * 1024;
  d.scratch = dalloc<double>(h, d.sys_in_smem ? 32 : pt_sys_doubles(n_sys));
  d.xinfo = dalloc<int32_t>(h, N);
  d.yinfo = dalloc<int32_t>(h, N);
  d.film_out = dalloc<double>(h, NN);
  d.rcache = dalloc<double>(h, 8 * (size_t)N);
  d.run_films = dalloc<double>(h, NN);
  d.run_rc = dalloc<double>(h, 2 * NN);
  d.run_flag = dalloc<int32_t>(h, N);
  d.done = dalloc<int32_t>(h, N);
  d.run_scratch = dalloc<double>(h, d.sys_in_smem ? 32 : (size_t)kRunCtas * pt_sys_doubles(n_sys));
  d.fpart = dalloc<double>(h, (size_t)kMaxPending * kFilmSegMax * 4 * N);
  h->bar = dalloc<unsigned>(h, 64);
  if (const char* e = getenv("PAQIF_PT_RUNS")) h->runs = e[0] != '0';
  d.prof = nullptr;
  if (const char* e = getenv("PAQIF_PT_PROF"))
    if (e[0] == '1') d.prof = dalloc<unsigned long long>(h, 8);
  for (void* a : h->allocs)
    if (!a) {
      paqif_ehl_point_destroy(h);
      set_cuda_error("ehl_point: alloc", cudaErrorMemoryAllocation);
      return nullptr;
    }
  if (h->allocs.size() != (d.prof ? 22u : 21u) ||
      cudaMallocHost((void**)&h->xinfo_prev, (size_t)N * sizeof(int32_t)) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->xinfo_ev, cudaEventDisableTiming) != cudaSuccess) {
    paqif_ehl_point_destroy(h);
    set_cuda_error("ehl_point: alloc", cudaErrorMemoryAllocation);
    return nullptr;
  }
  cudaMemcpyAsync(d.table, table, NN * 8, cudaMemcpyHostToDevice, h->st);
  cudaMemcpyAsync(d.geom, geometry, NN * 8, cudaMemcpyHostToDevice, h->st);
  if (!alloc_plan(h, h->plan, next_pow2(2 * n))) {
    paqif_ehl_point_destroy(h);
    set_cuda_error("ehl_point: FFT plan", cudaErrorMemoryAllocation);
    return nullptr;
  }
  h->line_smem = sizeof(PtShared) + (d.sys_in_smem ? sys_bytes : 0);
  if (cudaStreamSynchronize(h->st) != cudaSuccess || check_launch("ehl_point_create")) {
    paqif_ehl_point_destroy(h);
    return nullptr;
  }
  return h;
}

extern "C" void paqif_ehl_point_destroy(paqif_ehl_point* h) {
  if (!h) return;
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->d.prof) {
    unsigned long long pr[8] = {0};
    cudaMemcpy(pr, h->d.prof, sizeof(pr), cudaMemcpyDeviceToHost);
    const double nl = pr[4] ? (double)pr[4] : 1.0;
    fprintf(stderr, "[pt_prof] x-lines %llu (checked repeats %llu): cycles/line pass1 %.0f assemble %.0f solve %.0f update %.0f\n",
            pr[4], pr[5], pr[0] / nl, pr[1] / nl, pr[2] / nl, pr[3] / nl);
    unsigned long long ap[8];
    cudaMemcpyFromSymbol(ap, g_aqif2_prof, sizeof(ap));
    const double na = ap[4] ? (double)ap[4] : 1.0;
    fprintf(stderr, "[pt_prof] aqif2 solves %llu: factor %.0f breakdown %.0f z %.0f gather %.0f cycles"
            "; levels %llu, with a tiny numerator %llu\n",
            ap[4], ap[0] / na, ap[1] / na, ap[2] / na, ap[3] / na, ap[5], ap[6]);
  }
  for (void* a : h->ipc_opened) cudaIpcCloseMemHandle(a);
  for (void* a : h->allocs)
    if (a) cudaFree(a);
  if (h->xinfo_prev) cudaFreeHost(h->xinfo_prev);
  if (h->xinfo_ev) cudaEventDestroy(h->xinfo_ev);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

extern "C" int paqif_ehl_point_set_state(paqif_ehl_point* h, const double* u, double h0) {
  if (!h || !u) return set_arg_error("ehl_point_set_state");
  const size_t NN = (size_t)h->d.N * h->d.N;
  cudaMemcpyAsync(h->d.u, u, NN * 8, cudaMemcpyHostToDevice, h->st);
  double s[8] = {h0, 0, 0, 0, 0, 0, 0, 0};
  cudaMemcpyAsync(h->d.scal, s, sizeof(s), cudaMemcpyHostToDevice, h->st);
  cudaMemsetAsync(h->d.meta, 0, kMSize * sizeof(int), h->st);
  pt_set_gate_kernel<<<1, 32, 0, h->st>>>(h->d.meta, 0);
  fold(h);  // deformation_full(u): fresh base, no pending updates
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? check_launch("ehl_point_set_state") : set_cuda_error("set_state", e);
}

namespace {

unsigned film_blocks(int N, int L) {
  return (unsigned)((L * N + kPtFilmWarps - 1) / kPtFilmWarps);
}

// films + rheology of L consecutive lines into (films_out, rc_out, rho at
// rc_out + rho_off): tiled partial corrections and the per-output sum, four
// lines at a time (the same arithmetic for every line, whatever L)
void films(paqif_ehl_point* h, int mode, int first, int L, const int32_t* skip,
           double* films_out, double* rc_out, size_t rho_off) {
  PointDev& d = h->d;
  const int N = d.N;
  const int nseg = (N + kFilmKS - 1) / kFilmKS;
  const bool tiled = nseg <= kFilmSegMax;
  for (int l0 = 0; l0 < L; l0 += 4) {
    const int Lc = L - l0 < 4 ? L - l0 : 4;
    if (tiled) {
      const dim3 grid((unsigned)(((N + kFilmChunk - 1) / kFilmChunk) * Lc), (unsigned)nseg,
                      (unsigned)kMaxPending);
      pt_films_part_kernel<<<grid, 32, 0, h->st>>>(d, mode, first + l0, Lc, skip);
    }
    pt_films_kernel<<<film_blocks(N, Lc), 32 * kPtFilmWarps, 0, h->st>>>(
        d, h->cfg, mode, first + l0, Lc, films_out + (size_t)l0 * N, rc_out + (size_t)l0 * N,
        rho_off, skip, tiled ? nseg : 0);
  }
}

void prepare_attrs(paqif_ehl_point* h) {
  static bool done = false;  // per process; attributes are per function
  if (done) return;
  (void)h;
  const int smem = 227 * 1024;  // the largest any handle asks for
  cudaFuncSetAttribute(pt_xline_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pt_xline_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pt_yline_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pt_yline_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pt_xrun_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pt_xrun_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  done = true;
}

// Runs [a, b) of deferred lines for this x-sweep: every line when all
// updates are deferred (weighted_change_sweep); for the hybrid sweep the
// previous x-sweep's deferred runs (the weighted block in the contact is
// stable from one outer iteration to the next) -- a prediction only: the
// run kernel checks every line's own decision and leaves the rest to the
// per-line launches.
std::vector<std::pair<int, int>> x_runs(paqif_ehl_point* h, const SweepCtl& ctl) {
  std::vector<std::pair<int, int>> runs;
  const int n = h->d.n;
  if (!h->runs) return runs;
  // tags: the last completed x-sweep's (or, inside a device-driven chunk,
  // the snapshot taken when the chunk was enqueued)
  const int32_t* tags = nullptr;
  if (!h->pred.empty()) tags = h->pred.data();
  else if (h->xinfo_valid && cudaEventQuery(h->xinfo_ev) == cudaSuccess) tags = h->xinfo_prev;
  if (ctl.defer == 1) {
    runs.emplace_back(1, n);
  } else if (ctl.defer < 0 && ctl.sel != 0 && tags) {
    constexpr int kMinRun = 4;
    int a = -1;
    for (int j = 1; j <= n; ++j) {
      const bool dfr = j < n && (tags[j - 1] & 2) != 0;
      if (dfr && a < 0) a = j;
      if (!dfr && a >= 0) {
        if (j - a >= kMinRun) runs.emplace_back(a, j);
        a = -1;
      }
    }
  }
  return runs;
}

// x-direction sweep: lines j = 1..n-1 in order, each followed by the gated
// fold; deferred changes applied (and folded) at the end.  Runs of deferred
// lines are solved side by side first (pt_xrun_kernel); the per-line
// launches of a line the run solved return at once (done[j]).
void enqueue_x_sweep(paqif_ehl_point* h, const SweepCtl& ctl, bool exact) {
  PointDev& d = h->d;
  const int n = d.n, N = d.N;
  cudaStream_t st = h->st;
  const size_t NN = (size_t)N * N;
  pt_zero_kernel<<<296, 256, 0, st>>>(reinterpret_cast<uint32_t*>(d.sigma), NN * 2, d.meta);
  pt_zero_kernel<<<1, 32, 0, st>>>(reinterpret_cast<uint32_t*>(&d.meta[kMAnyW]), 1, d.meta);
  pt_zero_kernel<<<(N + 255) / 256, 256, 0, st>>>(reinterpret_cast<uint32_t*>(d.done), N, d.meta);
  const auto runs = x_runs(h, ctl);
  size_t next_run = 0;
  const bool certain = ctl.defer == 1;  // every line deferred: no per-line launches needed
  for (int j = 1; j < n; ++j) {
    if (next_run < runs.size() && runs[next_run].first == j) {
      const int a = runs[next_run].first, L = runs[next_run].second - a;
      ++next_run;
      // films + rheology of rows a-1 .. a+L, the deferred flags, the run
      films(h, 0, a - 1, L + 2, nullptr, d.run_films, d.run_rc, NN);
      pt_run_flags_kernel<<<L, 256, 0, st>>>(d, h->cfg, ctl, L);
      const unsigned g = (unsigned)(L < kRunCtas ? L : kRunCtas);
      if (d.sys_in_smem) {
        if (exact) pt_xrun_kernel<true, true><<<g, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, a, L);
        else pt_xrun_kernel<false, true><<<g, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, a, L);
      } else {
        if (exact) pt_xrun_kernel<true, false><<<g, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, a, L);
        else pt_xrun_kernel<false, false><<<g, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, a, L);
      }
      if (certain) {
        j = a + L - 1;
        continue;
      }
    }
    films(h, 0, j - 1, 3, &d.done[j], d.films, d.rcache, 4 * (size_t)N);
    if (d.sys_in_smem) {
      if (exact) pt_xline_kernel<true, true><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, j);
      else pt_xline_kernel<false, true><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, j);
    } else {
      if (exact) pt_xline_kernel<true, false><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, j);
      else pt_xline_kernel<false, false><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, j);
    }
    fold(h);
  }
  if (ctl.defer != 0) {
    pt_weighted_kernel<<<296, 256, 0, st>>>(d, ctl.omega);
    pt_copy_kernel<<<296, 256, 0, st>>>(d.u, d.film_out, NN, &d.meta[kMAnyW], d.meta);
    pt_set_gate_kernel<<<1, 32, 0, st>>>(d.meta, 1);
    fold(h);
  }
  // this sweep's tags: the next hybrid sweep's run prediction
  if (ctl.defer < 0 && ctl.sel < 0) {
    cudaMemcpyAsync(h->xinfo_prev, d.xinfo, (size_t)(n - 1) * sizeof(int32_t),
                    cudaMemcpyDeviceToHost, st);
    cudaEventRecord(h->xinfo_ev, st);
    h->xinfo_valid = true;
  }
}

void enqueue_y_sweep(paqif_ehl_point* h, const SweepCtl& ctl, bool exact) {
  PointDev& d = h->d;
  const int n = d.n, N = d.N;
  cudaStream_t st = h->st;
  for (int i = 1; i < n; ++i) {
    const int lo = i - 2 > 0 ? i - 2 : 0;
    const int L = i + 2 - lo;
    films(h, 1, lo, L, nullptr, d.films, d.rcache, 4 * (size_t)N);
    if (d.sys_in_smem) {
      if (exact) pt_yline_kernel<true, true><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, i);
      else pt_yline_kernel<false, true><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, i);
    } else {
      if (exact) pt_yline_kernel<true, false><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, i);
      else pt_yline_kernel<false, false><<<1, kPtThreads, h->line_smem, st>>>(d, h->cfg, ctl, i);
    }
    fold(h);
  }
}

void enqueue_residual(paqif_ehl_point* h) {
  PointDev& d = h->d;
  cudaStream_t st = h->st;
  pt_set_gate_kernel<<<1, 32, 0, st>>>(d.meta, 0);
  fold(h);  // film_full: fresh deformation, pending list cleared
  pt_zero_kernel<<<1, 32, 0, st>>>(reinterpret_cast<uint32_t*>(&d.scal[3]), 2, d.meta);
  pt_residual_kernel<<<d.N, 256, 0, st>>>(d, h->cfg);
  pt_finish_kernel<<<1, 32, 0, st>>>(d, h->cfg);
}

}  // namespace

extern "C" int paqif_ehl_point_sweep(paqif_ehl_point* h, int32_t kind, int32_t sel,
                                     int32_t nu_variant, double omega, uint32_t flags) {
  if (!h) return set_arg_error("ehl_point_sweep");
  if (kind < 0 || kind > 3 || sel < -1 || sel > 1 || nu_variant < 0 || nu_variant > 1)
    return set_arg_error("ehl_point_sweep: kind/sel/nu_variant");
  prepare_attrs(h);
  const bool exact = (flags & PAQIF_FLAG_EXACT) != 0;
  cudaMemsetAsync(&h->d.meta[kMErr], 0, sizeof(int), h->st);
  cudaMemsetAsync(&h->d.scal[4], 0, sizeof(double), h->st);
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);  // not device-driven
  SweepCtl ctl{sel, kind == 0 ? -1 : (kind == 2 ? 1 : 0), nu_variant, omega};
  if (kind == 3) enqueue_y_sweep(h, ctl, exact);
  else enqueue_x_sweep(h, ctl, exact);
  return check_launch("paqif_ehl_point_sweep");
}

extern "C" int paqif_ehl_point_force_balance(paqif_ehl_point* h) {
  if (!h) return set_arg_error("ehl_point_force_balance");
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  pt_force_kernel<<<1, 1024, 0, h->st>>>(h->d, h->cfg, nullptr);
  return check_launch("paqif_ehl_point_force_balance");
}

extern "C" int paqif_ehl_point_residual(paqif_ehl_point* h) {
  if (!h) return set_arg_error("ehl_point_residual");
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  enqueue_residual(h);
  return check_launch("paqif_ehl_point_residual");
}

namespace {
// one outer iteration of solve_ehl (solver.py:205-216): hybrid x-sweep,
// column sweep, force balance every force_every-th iteration (drv: on the
// drive record's schedule), complementarity residual
void enqueue_step(paqif_ehl_point* h, int32_t outer, bool exact, paqif_ehl_line_drive* drv) {
  const paqif_ehl_point_cfg& c = h->cfg;
  pt_zero_kernel<<<1, 32, 0, h->st>>>(reinterpret_cast<uint32_t*>(&h->d.meta[kMErr]), 1,
                                      h->d.meta);
  pt_zero_kernel<<<1, 32, 0, h->st>>>(reinterpret_cast<uint32_t*>(&h->d.scal[4]), 2, h->d.meta);
  enqueue_x_sweep(h, SweepCtl{-1, -1, c.variant, c.omega}, exact);
  enqueue_y_sweep(h, SweepCtl{0, 0, c.variant, c.omega}, exact);
  if (drv || (outer + 1) % c.force_every == 0)
    pt_force_kernel<<<1, 1024, 0, h->st>>>(h->d, c, drv);
  enqueue_residual(h);
}
}  // namespace

extern "C" int paqif_ehl_point_step(paqif_ehl_point* h, int32_t outer, uint32_t flags) {
  if (!h) return set_arg_error("ehl_point_step");
  prepare_attrs(h);
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);  // not device-driven
  enqueue_step(h, outer, (flags & PAQIF_FLAG_EXACT) != 0, nullptr);
  return check_launch("paqif_ehl_point_step");
}

extern "C" int paqif_ehl_point_drive_steps(paqif_ehl_point* h, int32_t steps,
                                           paqif_ehl_line_drive* drive, double* hist_res,
                                           double* hist_def, int32_t hist_cap, uint32_t flags) {
  if (!h || !drive || steps < 0 || (hist_res && (!hist_def || hist_cap < 1)))
    return set_arg_error("ehl_point_drive_steps");
  prepare_attrs(h);
  const bool exact = (flags & PAQIF_FLAG_EXACT) != 0;
  // run prediction for the whole chunk: the last completed x-sweep's tags
  h->pred.clear();
  if (h->runs && h->xinfo_valid && cudaEventSynchronize(h->xinfo_ev) == cudaSuccess)
    h->pred.assign(h->xinfo_prev, h->xinfo_prev + (h->d.n - 1));
  pt_drive_begin_kernel<<<1, 32, 0, h->st>>>(h->d.meta, drive);
  for (int32_t s = 0; s < steps; ++s) {
    enqueue_step(h, 0, exact, drive);
    pt_drive_kernel<<<1, 32, 0, h->st>>>(h->d, h->cfg, drive, hist_res, hist_def, hist_cap);
  }
  h->pred.clear();
  return check_launch("paqif_ehl_point_drive_steps");
}

extern "C" int paqif_ehl_point_get(paqif_ehl_point* h, double* u, double* film, double* scal,
                                   int32_t* xinfo, int32_t* yinfo, int32_t* err) {
  if (!h) return set_arg_error("ehl_point_get");
  const size_t NN = (size_t)h->d.N * h->d.N;
  cudaStream_t st = h->st;
  if (u) cudaMemcpyAsync(u, h->d.u, NN * 8, cudaMemcpyDeviceToHost, st);
  if (film) cudaMemcpyAsync(film, h->d.film_out, NN * 8, cudaMemcpyDeviceToHost, st);
  if (scal) {
    cudaMemcpyAsync(scal, h->d.scal, 3 * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(scal + 3, h->d.scal + 4, 8, cudaMemcpyDeviceToHost, st);
  }
  if (xinfo) cudaMemcpyAsync(xinfo, h->d.xinfo, (h->d.n - 1) * 4, cudaMemcpyDeviceToHost, st);
  if (yinfo) cudaMemcpyAsync(yinfo, h->d.yinfo, (h->d.n - 1) * 4, cudaMemcpyDeviceToHost, st);
  if (err) cudaMemcpyAsync(err, &h->d.meta[kMErr], 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? PAQIF_OK : set_cuda_error("ehl_point_get", e);
}

extern "C" void* paqif_ehl_point_stream(paqif_ehl_point* h) { return h ? (void*)h->st : nullptr; }

extern "C" int paqif_ehl_point_sync(paqif_ehl_point* h) {
  if (!h) return set_arg_error("ehl_point_sync");
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? PAQIF_OK : set_cuda_error("ehl_point_sync", e);
}

extern "C" int paqif_ehl_point_deformation(paqif_ehl_point* h, const double* u, double* out) {
  if (!h) return set_arg_error("ehl_point_deformation");
  const size_t NN = (size_t)h->d.N * h->d.N;
  cudaMemcpyAsync(h->d.film_out, u, NN * 8, cudaMemcpyHostToDevice, h->st);
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  pt_set_gate_kernel<<<1, 32, 0, h->st>>>(h->d.meta, 0);
  // deformation_full: fresh base, pending line updates cleared (film.py:67-79)
  fft_deformation(h->plan, h->d.film_out, h->d.dbase, &h->d.meta[kMGate], &h->d.meta[kMCount],
                  h->st);
  if (out) cudaMemcpyAsync(out, h->d.dbase, NN * 8, cudaMemcpyDeviceToHost, h->st);
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? check_launch("ehl_point_deformation") : set_cuda_error("deformation", e);
}

namespace paqif {
// append a pending line update (FilmModel.note_line_update)
__global__ void pt_note_kernel(PointDev d, int axis, int index, const double* __restrict__ delta) {
  const int p = d.meta[kMCount];
  if (p >= kMaxPending) return;  // the caller folds before this can happen
  for (int i = threadIdx.x; i < d.N; i += blockDim.x) d.pend[(size_t)p * d.N + i] = delta[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    d.meta[kMAxis + p] = axis;
    d.meta[kMIdx + p] = index;
    d.meta[kMCount] = p + 1;
  }
}
}  // namespace paqif

extern "C" int paqif_ehl_point_note_update(paqif_ehl_point* h, int32_t axis, int32_t index,
                                           const double* delta) {
  if (!h || !delta || axis < 0 || axis > 1 || index < 0 || index > h->d.n)
    return set_arg_error("ehl_point_note_update");
  bool any = false;
  for (int i = 0; i < h->d.N; ++i) any |= delta[i] != 0.0;
  if (!any) return PAQIF_OK;  // film.py:86-87
  int count = 0;
  cudaMemcpy(&count, &h->d.meta[kMCount], sizeof(int), cudaMemcpyDeviceToHost);
  if (count >= kMaxPending) return set_arg_error("ehl_point_note_update: fold first (> 8 pending)");
  // stage delta in the films buffer's rho half (4N spare doubles)
  double* tmp = h->d.rcache + 4 * (size_t)h->d.N;
  cudaMemcpyAsync(tmp, delta, (size_t)h->d.N * 8, cudaMemcpyHostToDevice, h->st);
  pt_note_kernel<<<1, 256, 0, h->st>>>(h->d, axis, index, tmp);
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? check_launch("ehl_point_note_update") : set_cuda_error("note_update", e);
}

extern "C" int paqif_ehl_point_film_lines(paqif_ehl_point* h, int32_t mode, const int32_t* idx,
                                          int32_t L, double h0, double* out) {
  if (!h || !idx || !out || L < 0 || mode < 0 || mode > 1)
    return set_arg_error("ehl_point_film_lines");
  for (int k = 0; k < L; ++k)
    if (idx[k] < 0 || idx[k] > h->d.n) return set_arg_error("ehl_point_film_lines: index");
  const int N = h->d.N;
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  cudaMemcpyAsync(&h->d.scal[0], &h0, sizeof(double), cudaMemcpyHostToDevice, h->st);
  for (int k = 0; k < L; ++k) {
    films(h, mode, idx[k], 1, nullptr, h->d.films, h->d.rcache, 4 * (size_t)N);
    cudaMemcpyAsync(out + (size_t)k * N, h->d.films, (size_t)N * 8, cudaMemcpyDeviceToHost, h->st);
  }
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? check_launch("ehl_point_film_lines") : set_cuda_error("film_lines", e);
}


// ------------------------------------------------------- sharded folds
// IPC handles of this handle's buffers the peers write into: the
// half-spectrum buffer W, the deformation base D and the barrier words
// (3 x 64 bytes).
extern "C" int paqif_ehl_point_ipc_handles(paqif_ehl_point* h, void* out) {
  if (!h || !out) return set_arg_error("ehl_point_ipc_handles");
  cudaIpcMemHandle_t* o = reinterpret_cast<cudaIpcMemHandle_t*>(out);
  cudaError_t e;
  if ((e = cudaIpcGetMemHandle(&o[0], h->plan.W)) != cudaSuccess ||
      (e = cudaIpcGetMemHandle(&o[1], h->d.dbase)) != cudaSuccess ||
      (e = cudaIpcGetMemHandle(&o[2], h->bar)) != cudaSuccess)
    return set_cuda_error("ehl_point_ipc_handles", e);
  return PAQIF_OK;
}

// Open every peer's handles (world x 3 x 64 bytes, in rank order) and split
// every later fold of this handle over the ranks.  All ranks attach before
// any of them folds again (the caller's exchange of handles is that sync).
extern "C" int paqif_ehl_point_attach_peers(paqif_ehl_point* h, int32_t rank, int32_t world,
                                            const void* handles) {
  if (!h || !handles || world < 1 || world > kFoldMaxRanks || rank < 0 || rank >= world)
    return set_arg_error("ehl_point_attach_peers: rank / world (1..8)");
  if (h->sharded) return set_arg_error("ehl_point_attach_peers: already attached");
  const cudaIpcMemHandle_t* in = reinterpret_cast<const cudaIpcMemHandle_t*>(handles);
  FoldPeers q{};
  q.rank = rank;
  q.world = world;
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      q.W[r] = h->plan.W;
      q.D[r] = h->d.dbase;
      q.bar[r] = h->bar;
      continue;
    }
    void* ptr[3];
    for (int b = 0; b < 3; ++b) {
      cudaError_t e = cudaIpcOpenMemHandle(&ptr[b], in[3 * r + b], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return set_cuda_error("ehl_point_attach_peers: open", e);
      h->ipc_opened.push_back(ptr[b]);
    }
    q.W[r] = reinterpret_cast<double2*>(ptr[0]);
    q.D[r] = reinterpret_cast<double*>(ptr[1]);
    q.bar[r] = reinterpret_cast<unsigned*>(ptr[2]);
  }
  h->peers = q;
  h->sharded = world > 1;
  return PAQIF_OK;
}

// Dev / test: the sharded decomposition with `world` ranks emulated in
// order on this GPU, deformation of u (host, N x N) into out (host) --
// bit-identical to paqif_ehl_point_deformation for every world.
extern "C" int paqif_ehl_point_fold_emulated(paqif_ehl_point* h, int32_t world, const double* u,
                                             double* out) {
  if (!h || !u || world < 1 || world > 64) return set_arg_error("ehl_point_fold_emulated");
  const size_t NN = (size_t)h->d.N * h->d.N;
  cudaMemcpyAsync(h->d.film_out, u, NN * 8, cudaMemcpyHostToDevice, h->st);
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  pt_set_gate_kernel<<<1, 32, 0, h->st>>>(h->d.meta, 0);
  fold_sharded_emulated(h->plan, h->d.film_out, h->d.dbase, world, &h->d.meta[kMGate],
                        &h->d.meta[kMCount], h->st);
  if (out) cudaMemcpyAsync(out, h->d.dbase, NN * 8, cudaMemcpyDeviceToHost, h->st);
  cudaError_t e = cudaStreamSynchronize(h->st);
  return e == cudaSuccess ? check_launch("ehl_point_fold_emulated") : set_cuda_error("fold_emulated", e);
}

// Bench: `reps` forced folds of the resident pressure (sharded when
// attached), enqueued on the handle's stream.
extern "C" int paqif_ehl_point_fold_bench(paqif_ehl_point* h, int32_t reps) {
  if (!h || reps < 0) return set_arg_error("ehl_point_fold_bench");
  cudaMemsetAsync(&h->d.meta[kMStop], 0, sizeof(int), h->st);
  for (int r = 0; r < reps; ++r) {
    pt_set_gate_kernel<<<1, 32, 0, h->st>>>(h->d.meta, 0);
    fold(h);
  }
  return check_launch("paqif_ehl_point_fold_bench");
}
