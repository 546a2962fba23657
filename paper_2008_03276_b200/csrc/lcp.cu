// Fused batched projected LCP -- the config-2 hot path.
//
// One warp owns one banded system at a time (persistent grid, static
// striding over the batch) and runs the whole of
// paqif_solve_lcp(LcpProblem(L, f), r=1) (paqif/parallel.py:298-347) on it:
//
//   active = f <= 0                                   parallel.py:312
//   loop over passes:
//     lmod/fmod: pinned rows keep only their diagonal  parallel.py:320-327
//     paqif_solve(lmod, fmod, r=1):                    parallel.py:261-295
//       factorize_wz + solve_w (fused, register windows, aqif_warp.cuh)
//       reduced corner system (Z corner blocks, normal equations,
//         Cholesky)                                    parallel.py:184-231
//       solve_z(start_level = beta+1) for the middles  parallel.py:234-258
//     lam = L u_eval - f, u = max(u_eval, 0),
//     res = max|min(u, L u - f)|                       parallel.py:329-331
//     return / keep best / new_active = u_eval < lam   parallel.py:332-343
//
// The pinned rows are never materialised: the band is streamed straight
// from HBM and the pin is applied while loading (LcpPol::entry).  Z factor
// records (pivot rows + W-solved right side, 38 doubles/level at beta=8) go
// to a per-warp global stack and are read back outside-in by the Z solve
// through a double-buffered cp.async ring in shared memory.
#include <cfloat>
#include <mutex>
#include "aqif_warp.cuh"
#include "aqif_pipe.cuh"
#include "zsolve.cuh"
#include "capi_util.cuh"

namespace paqif {

template <int BETA>
struct LcpPol {
  static constexpr bool kFuseW = true;
  static constexpr bool kResidual = false;
  static constexpr bool kFastDiv = true;  // branch-free divisions, checked repeat
  static constexpr bool kLazyBreakdown = true;  // breakdown found after the loop
  // ... and not even tested in the loop: the Z solve and the corner system
  // read every pivot record and apply the level test there
  static constexpr bool kDeferBreakdown = true;
  static constexpr bool kRecordW = false;
  using PL = PivotLayout<BETA>;
  const double* band;
  const uint64_t* act;
  const double* f;
  double* zs;
  int n;
  bool use_act;

  __device__ __forceinline__ const double* raw_ptr(int i, int d) const {
    return band + (size_t)(d + BETA) * n + i;
  }
  __device__ __forceinline__ double raw(int i, int d) const { return *raw_ptr(i, d); }
  __device__ __forceinline__ const uint64_t* pin_ptr(int i) const {
    return use_act ? act + i : nullptr;
  }
  __device__ __forceinline__ bool pinned(int i) const { return use_act && act[i] != 0ull; }
  __device__ __forceinline__ const double* frhs_ptr(int i) const { return f + i; }
  __device__ __forceinline__ double frhs(int i) const { return f[i]; }
  // level k's pivot record (pivot rows + W-solved right sides, 38 doubles at
  // BETA = 8) to the Z stack, copied from the pivot buffer by the group's
  // lanes (16-byte coalesced stores)
  __device__ __forceinline__ double* record_out(int k) const { return zs + (size_t)k * PL::kSize; }
  __device__ __forceinline__ void on_level(int k, const double* pb, int gl, int G) {
    double2* dst = reinterpret_cast<double2*>(zs + (size_t)k * PL::kSize);
    const double2* src = reinterpret_cast<const double2*>(pb);
    constexpr int NP = PL::kSize / 2, GG = Group<BETA>::G;
#pragma unroll
    for (int t = 0; t < (NP + GG - 1) / GG; ++t) {  // straight-line, predicated
      const int idx = gl + t * G;
      if (idx < NP) dst[idx] = src[idx];
    }
  }
  __device__ __forceinline__ void on_w(int, int, double, double) {}
  __device__ __forceinline__ void on_resid(int, int, double) {}
};

__device__ __forceinline__ double fmax_(double a, double b) { return b > a ? b : a; }

// numpy maximum(x, 0.0) / minimum(a, b) semantics (NaN propagating, -0.0 kept)
__device__ __forceinline__ double np_max0(double x) { return ((x >= 0.0) | (x != x)) ? x : 0.0; }
__device__ __forceinline__ double np_min(double a, double b) {
  return ((a <= b) | (a != a)) ? a : b;
}

constexpr int kLcpWarpsPerBlock = 4;
#ifndef PAQIF_CHECK_PF
#define PAQIF_CHECK_PF 2  // complementarity-check steps the L1 prefetch runs ahead
#endif
#ifndef PAQIF_LCP_MINB
#define PAQIF_LCP_MINB 2  // resident blocks per SM the register budget is sized for
#endif

#ifdef PAQIF_PROFILE_PHASES
// dev-only phase timers (tools/phase_prof.cu): factor, corner, zsolve, check
__device__ unsigned long long g_phase_cycles[4];
#define PAQIF_TSTAMP(v) const long long v = clock64()
#define PAQIF_TACC(i, a, b) ph_acc[i] += (unsigned long long)((b) - (a))
#else
#define PAQIF_TSTAMP(v)
#define PAQIF_TACC(i, a, b)
#endif

template <int BETA>
struct LcpSmem {
  using PL = PivotLayout<BETA>;
  static constexpr int ZC = ZChunk<BETA>::ZC;
  static constexpr int kM = 2 * BETA;
  static constexpr int kCorner = 2 * kM * kM + 3 * kM;
  static constexpr int kRing = 2 * ZC * PL::kSize;
  static constexpr int kScratch = kRing > kCorner ? kRing : kCorner;
  // the factorization's prefetch slots and the Z-solve ring / corner system
  // are live in different phases and share storage
  union {
    EngineSmem<BETA> eng;
    struct {
      double pbuf_[2 * PL::kSize];
      double scratch[kScratch];
    } post;
  };
};

// Corner unknowns from the reduced system (r = 1): Rd = Z corner blocks,
// solved through R^T R Cholesky as solve_reduced does (parallel.py:227-231).
// Runs on the G lanes of the system's group; all 32 lanes call (syncs).
// Returns 0 or 1 (not SPD).
// Also applies the factorization's level test (_kernels.py:112-122; the
// LCP policy defers it) to the outermost levels s-BETA+1 .. s-1, whose
// records only the corner system reads: `fbad` = the smallest failing
// level there, or 0 (group-uniform).
template <int BETA, bool EXACT>
__device__ int corner_solve(const double* zs, int n, double* x, double* cs, int gl, bool alive,
                            int& fbad)
{
  using A = Arith<EXACT>;
  using PL = PivotLayout<BETA>;
  constexpr int BP1 = BETA + 1, m = 2 * BETA;
  constexpr int G = Group<BETA>::G;
  const int s = n / 2;
  double* rd = cs;
  double* rtr = rd + m * m;
  double* fd = rtr + m * m;
  double* rtf = fd + m;
  double* rinv = rtf + m;  // FMA arithmetic: 1 / diag of the Cholesky factor
  {
    int lv = 0;
    if (alive && gl < BETA - 1) {
      const int k = s - BETA + 1 + gl;
      const double* rec = zs + (size_t)k * PL::kSize;
      const double a11 = rec[PL::zi(0, 0, 0)], a12 = rec[PL::zi(1, 0, 0)];
      const double a21 = rec[PL::zi(0, 0, 1)], a22 = rec[PL::zi(1, 0, 1)];
      const double det = A::det2(a11, a22, a21, a12);
      const double scale = fmax(fmax(fabs(a11), fabs(a12)), fmax(fabs(a21), fabs(a22)));
      lv = fabs(det) <= 1e-14 * (scale * scale) + PAQIF_TINY ? k : 0;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const int w = __shfl_xor_sync(0xffffffffu, lv, o);
      lv = (lv == 0 || (w != 0 && w < lv)) ? w : lv;
    }
    fbad = lv;
  }
  if (alive)
    for (int idx = gl; idx < m * m; idx += G) rd[idx] = 0.0;
  __syncwarp();
  if (alive) {
    for (int idx = gl; idx < BETA * (PL::kZ + 2); idx += G) {
      const int kk = idx / (PL::kZ + 2), q = idx % (PL::kZ + 2);
      const int k = s - BETA + 1 + kk, rt = s - k, rb = n - 1 - rt;
      const double* rec = zs + (size_t)k * PL::kSize;
      const int brow = BETA + (rb - (n - BETA));
      if (q < PL::kZ) {
        const int side = q & 1, e = (q >> 1) % BP1, win = (q >> 1) / BP1;
        const int row = side == 0 ? rt : brow;
        if (win == 0) {
          const int col = rt - e;
          if (col >= 0) rd[row * m + col] = rec[q];
        } else {
          const int col = rb + e;
          if (col < n) rd[row * m + BETA + (col - (n - BETA))] = rec[q];
        }
      } else if (q == PL::kZ) {
        fd[rt] = rec[PL::kYT];
      } else {
        fd[brow] = rec[PL::kYB];
      }
    }
  }
  __syncwarp();
  if (alive) {
    for (int idx = gl; idx < m * m; idx += G) {
      const int i = idx / m, j = idx % m;
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < m; ++r) acc = A::axpy(acc, rd[r * m + i], rd[r * m + j]);
      rtr[idx] = acc;
    }
    for (int i = gl; i < m; i += G) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < m; ++r) acc = A::axpy(acc, rd[r * m + i], fd[r]);
      rtf[i] = acc;
    }
  }
  __syncwarp();
  int fail = 0;
  for (int j = 0; j < m; ++j) {
    double ajj = 0.0;
    if (alive && !fail) {
      ajj = rtr[j * m + j];
      for (int i = 0; i < j; ++i) ajj = A::sub(ajj, A::mul(rtr[i * m + j], rtr[i * m + j]));
      if (!(ajj > 0.0)) fail = 1;
      ajj = __dsqrt_rn(ajj);
    }
    __syncwarp();
    if (alive && !fail) {
      // reference rounding divides every entry; FMA arithmetic multiplies by
      // one reciprocal per column (kept for the substitutions)
      const double inv = EXACT ? 0.0 : 1.0 / ajj;
      for (int k = j + 1 + gl; k < m; k += G) {
        double v = rtr[j * m + k];
        for (int i = 0; i < j; ++i) v = A::sub(v, A::mul(rtr[i * m + j], rtr[i * m + k]));
        rtr[j * m + k] = EXACT ? A::div(v, ajj) : v * inv;
      }
      if (gl == 0) {
        rtr[j * m + j] = ajj;
        if (!EXACT) rinv[j] = inv;
      }
    }
    __syncwarp();
  }
  if (alive && !fail && gl == 0) {
    for (int j = 0; j < m; ++j) {
      double v = rtf[j];
      for (int i = 0; i < j; ++i) v = A::sub(v, A::mul(rtr[i * m + j], rtf[i]));
      rtf[j] = EXACT ? A::div(v, rtr[j * m + j]) : v * rinv[j];
    }
    for (int j = m - 1; j >= 0; --j) {
      double v = rtf[j];
      for (int k = j + 1; k < m; ++k) v = A::sub(v, A::mul(rtr[j * m + k], rtf[k]));
      rtf[j] = EXACT ? A::div(v, rtr[j * m + j]) : v * rinv[j];
    }
    for (int i = 0; i < BETA; ++i) {
      x[i] = rtf[i];
      x[n - BETA + i] = rtf[BETA + i];
    }
  }
  __syncwarp();
  return fail;
}

template <int BETA, bool EXACT, bool SOLVE_ONLY>
__global__ void __launch_bounds__(32 * kLcpWarpsPerBlock, PAQIF_LCP_MINB)
lcp_kernel(int64_t B, int n, const double* __restrict__ bands, const double* __restrict__ f,
           double tol, int max_outer, double* u_out, uint8_t* act_out, int64_t* passes_out,
           double* res_out, int64_t* status_out, char* ws, size_t ws_per_slot, int total_warps,
           unsigned long long* next_pair)
{
  using A = Arith<EXACT>;
  using PL = PivotLayout<BETA>;
  constexpr int G = Group<BETA>::G;
  constexpr int P = Group<BETA>::P;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char lcp_dyn_smem[];
  LcpSmem<BETA>* sm = reinterpret_cast<LcpSmem<BETA>*>(lcp_dyn_smem);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = lane / G, gl = lane % G;
  const int gw = blockIdx.x * kLcpWarpsPerBlock + wid;
  if (gw >= total_warps) return;
  LcpSmem<BETA>& my_sm = sm[wid * P + g];
  const int s = n / 2;
  const size_t nb = (size_t)(2 * BETA + 1) * n;
  char* my = ws + ((size_t)gw * P + g) * ws_per_slot;
  double* zs = reinterpret_cast<double*>(my);
  size_t off = (((size_t)(s + 1) * PL::kSize * sizeof(double)) + 255) & ~(size_t)255;
  double* x = reinterpret_cast<double*>(my + off);
  off += (((size_t)n * sizeof(double)) + 255) & ~(size_t)255;
  // active sets as 64-bit words: the factorization copies the flags with
  // the band values (8-byte cp.async)
  uint64_t* act = reinterpret_cast<uint64_t*>(my + off);
  off += ((size_t)n * 8 + 255) & ~(size_t)255;
  uint64_t* nact = reinterpret_cast<uint64_t*>(my + off);
#ifdef PAQIF_PROFILE_PHASES
  unsigned long long ph_acc[4] = {0, 0, 0, 0};
#endif

  // pairs of systems: the first per warp static, then taken from a global
  // counter as warps finish (pass counts differ per system)
  int64_t pair = gw;
  for (int64_t base = pair * P; base < B; base = pair * P) {
    const int64_t b = base + g;
    const bool have = b < B;
    const double* bd = bands + (have ? b : 0) * nb;
    const double* fb = f + (have ? b : 0) * (size_t)n;
    double* ub = u_out + (have ? b : 0) * (size_t)n;
    uint8_t* ab = SOLVE_ONLY ? nullptr : act_out + (have ? b : 0) * (size_t)n;
    if (have) {
      // initial policy active = f <= 0 (parallel.py:312); four loads of f in
      // flight per lane
      for (int i0 = gl; i0 < n; i0 += 4 * G) {
        double fv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) fv[u] = i0 + u * G < n ? __ldg(fb + i0 + u * G) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = i0 + u * G;
          if (i >= n) break;
          const uint64_t a = SOLVE_ONLY ? 0ull : (fv[u] <= 0.0 ? 1ull : 0ull);
          act[i] = a;
          if (!SOLVE_ONLY) {
            ub[i] = 0.0;
            ab[i] = (uint8_t)a;
          }
        }
      }
    }
    double best_res = INFINITY, res = INFINITY;
    int passes = 0, st = 0, brk_level = 0;
    bool done = false;
    bool active = have;  // this group still iterating
    uint64_t* cur = act;
    uint64_t* nxt = nact;
    for (int outer = 0; outer < max_outer; ++outer) {
      if (!__any_sync(FULL, active)) break;
      __syncwarp();
      LcpPol<BETA> pol;
      pol.band = bd;
      pol.act = cur;
      pol.f = fb;
      pol.zs = zs;
      pol.n = n;
      pol.use_act = !SOLVE_ONLY;
      if (active) passes = outer + 1;
      PAQIF_TSTAMP(t0);
      // FMA arithmetic: the software-pipelined level loop (aqif_pipe.cuh);
      // reference rounding: the general engine
      int fst = 0;
      if constexpr (EXACT)
        fst = aqif_factor_group<BETA, EXACT>(pol, n, 1e-14, my_sm.eng, gl, active);
      else
        aqif_factor_pipe<BETA>(pol, n, my_sm.eng, gl, active);
      if (EXACT && __any_sync(FULL, fst < 0)) {
        // a multiplier left the branch-free division's range: repeat this
        // system's factorization with IEEE divisions (the others idle)
        __syncwarp();
        const int f2 = aqif_factor_group<BETA, EXACT, LcpPol<BETA>, false>(
            pol, n, 1e-14, my_sm.eng, gl, active && fst < 0);
        if (fst < 0) fst = f2;
      }
      if (fst) {
        st = PAQIF_LCP_FACTOR_BREAKDOWN;
        brk_level = fst;
        active = false;
      }
      __syncwarp();  // every record stored before the corner system / Z solve read them
      PAQIF_TSTAMP(t1);
      // the factorization's breakdown test runs on the records: here for
      // the outermost levels, in the Z solve for the rest; a breakdown
      // outranks the corner system's failure (the reference raises in
      // factorize_wz first, aqif.py:133-134)
      int fbad_corner = 0;
      const bool not_pd =
          corner_solve<BETA, EXACT>(zs, n, x, my_sm.post.scratch, gl, active, fbad_corner) != 0;
      PAQIF_TSTAMP(t2);
      if (!SOLVE_ONLY && active) {
        // the band and f into L2 while the Z chain runs, for the
        // complementarity check that follows it (one bulk prefetch per lane)
        const size_t bytes = nb * 8;
        const size_t chunk = ((bytes + G - 1) / G + 15) & ~(size_t)15;
        const size_t lo = (size_t)gl * chunk;
        if (lo < bytes) {
          const size_t len = bytes - lo < chunk ? bytes - lo : chunk;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                           reinterpret_cast<const char*>(bd) + lo),
                       "r"((unsigned)len)
                       : "memory");
        }
        if (gl == G - 1)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(fb),
                       "r"((unsigned)(n * 8))
                       : "memory");
      }
      {
        const int fbad_z =
            zsolve_group<BETA, EXACT, false, Group<BETA>::G, true>(zs, n, x, my_sm.post.scratch, gl,
                                                                   active);
        const int fbad = fbad_z ? fbad_z : fbad_corner;
        if (active && fbad) {
          st = PAQIF_LCP_FACTOR_BREAKDOWN;
          brk_level = fbad;
          active = false;
        } else if (active && not_pd) {
          st = PAQIF_LCP_NOT_PD;
          active = false;
        }
      }
      PAQIF_TSTAMP(t3);
      PAQIF_TACC(0, t0, t1);
      PAQIF_TACC(1, t1, t2);
      PAQIF_TACC(2, t2, t3);
      if (SOLVE_ONLY) {
        if (active) {
          for (int i = gl; i < n; i += G) ub[i] = x[i];
          done = true;
        }
        active = false;
        continue;
      }
      // complementarity check and next policy (parallel.py:329-343)
      double r = 0.0;
      int changed = 0;
      if (active) {
        // one row of L x and L max(x, 0) against f, given its loads
        auto finish = [&](int i, double acc1, double acc2, double xi, double fi, uint64_t ci) {
          const double lam = A::sub(acc1, fi);
          const double rr = A::sub(acc2, fi);
          const double mn = fabs(np_min(np_max0(xi), rr));
          r = ((r != r) | (mn != mn)) ? __longlong_as_double(0x7ff8000000000000ll) : (mn > r ? mn : r);
          const uint64_t na = xi < lam ? 1ull : 0ull;
          nxt[i] = na;
          changed |= (na != ci);
        };
        auto edge_row = [&](int i) {  // rows whose band runs off the matrix
          double acc1 = 0.0, acc2 = 0.0;
          const int lo = i - BETA > 0 ? i - BETA : 0;
          const int hi = i + BETA + 1 < n ? i + BETA + 1 : n;
          for (int j = lo; j < hi; ++j) {
            const double a = bd[(size_t)(j - i + BETA) * n + i];
            const double xe = x[j];
            acc1 = A::axpy(acc1, a, xe);
            acc2 = A::axpy(acc2, a, np_max0(xe));
          }
          finish(i, acc1, acc2, x[i], fb[i], cur[i]);
        };
        // interior rows two per step (i, i+G): every load of the step -- 2 x
        // 17 band values, the x windows, f and the active flags -- issued
        // before the first use, so a step waits for one memory round trip
        // (the band comes from HBM here); the band lines two steps ahead are
        // prefetched into L1
        // (and the lines of x, f and the active flags those rows read)
        auto prefetch_rows = [&](int r0) {
          for (int q = gl; q < 2 * (2 * BETA + 1); q += G) {
            const int d = q >> 1, rr = r0 + (q & 1) * G;
            if (rr < n)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(bd + (size_t)d * n + rr));
          }
          if (gl < 6) {  // 2G rows: x window (3 lines), f (1-2), flags (2)
            const int q = gl;
            const void* pp = q < 3 ? (const void*)(x + min(max(r0 - BETA + 16 * q, 0), n - 1))
                             : q < 4 ? (const void*)(fb + min(r0, n - 1))
                                     : (const void*)(cur + min(r0 + 16 * (q - 4), n - 1));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(pp));
          }
        };
        constexpr int ND = 2 * BETA + 1;
        int i = gl;
        for (; i < BETA; i += G) edge_row(i);  // G >= BETA: at most one
        for (; i + G < n - BETA; i += 2 * G) {
          prefetch_rows(i - gl + 2 * PAQIF_CHECK_PF * G);
          double av0[ND], xv0[ND], av1[ND], xv1[ND];
#pragma unroll
          for (int d = 0; d < ND; ++d) {
            av0[d] = __ldg(bd + (size_t)d * n + i);
            av1[d] = __ldg(bd + (size_t)d * n + i + G);
            xv0[d] = x[i - BETA + d];
            xv1[d] = x[i + G - BETA + d];
          }
          const double f0 = __ldg(fb + i), f1 = __ldg(fb + i + G);
          const uint64_t c0 = cur[i], c1 = cur[i + G];
          double p0 = 0.0, q0 = 0.0, p1 = 0.0, q1 = 0.0;
#pragma unroll
          for (int d = 0; d < ND; ++d) {
            p0 = A::axpy(p0, av0[d], xv0[d]);
            q0 = A::axpy(q0, av0[d], np_max0(xv0[d]));
            p1 = A::axpy(p1, av1[d], xv1[d]);
            q1 = A::axpy(q1, av1[d], np_max0(xv1[d]));
          }
          finish(i, p0, q0, xv0[BETA], f0, c0);
          finish(i + G, p1, q1, xv1[BETA], f1, c1);
        }
        for (; i < n; i += G) {
          if (i >= BETA && i < n - BETA) {
            double acc1 = 0.0, acc2 = 0.0;
#pragma unroll
            for (int d = 0; d < ND; ++d) {
              const double a = __ldg(bd + (size_t)d * n + i), xe = x[i - BETA + d];
              acc1 = A::axpy(acc1, a, xe);
              acc2 = A::axpy(acc2, a, np_max0(xe));
            }
            finish(i, acc1, acc2, x[i], fb[i], cur[i]);
          } else {
            edge_row(i);
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(FULL, r, o);
        r = ((r != r) | (w != w)) ? __longlong_as_double(0x7ff8000000000000ll) : (w > r ? w : r);
        changed |= __shfl_xor_sync(FULL, changed, o);
      }
      PAQIF_TSTAMP(t4);
      PAQIF_TACC(3, t3, t4);
      if (!active) continue;
      res = r;
      if (res <= tol || res < best_res) {
        int i = gl;
        for (; i + 3 * G < n; i += 4 * G) {  // loads of four rows in flight
          const double x0 = x[i], x1 = x[i + G], x2 = x[i + 2 * G], x3 = x[i + 3 * G];
          const uint64_t c0 = cur[i], c1 = cur[i + G], c2 = cur[i + 2 * G], c3 = cur[i + 3 * G];
          ub[i] = np_max0(x0);
          ub[i + G] = np_max0(x1);
          ub[i + 2 * G] = np_max0(x2);
          ub[i + 3 * G] = np_max0(x3);
          ab[i] = (uint8_t)c0;
          ab[i + G] = (uint8_t)c1;
          ab[i + 2 * G] = (uint8_t)c2;
          ab[i + 3 * G] = (uint8_t)c3;
        }
        for (; i < n; i += G) {
          ub[i] = np_max0(x[i]);
          ab[i] = (uint8_t)cur[i];
        }
        if (res <= tol) {
          done = true;
          active = false;
          continue;
        }
        best_res = res;
      }
      if (!changed) {
        active = false;
        continue;
      }
      uint64_t* t = cur;
      cur = nxt;
      nxt = t;
    }
    if (__any_sync(FULL, have && !done && st == 0)) {
      // acceptance floor of a system that did not converge
      // (parallel.py:344-347): 1e3 eps (max row sum |L| + max |f|), only
      // needed here, so the band is not read for it otherwise
      double cmax = 0.0, fmax = 0.0;
      if (!SOLVE_ONLY && have && !done && st == 0)
        for (int i = gl; i < n; i += G) {
          double c = 0.0;
          for (int d = 0; d <= 2 * BETA; ++d) c = c + fabs(bd[(size_t)d * n + i]);
          cmax = c > cmax ? c : cmax;
          fmax = fabs(fb[i]) > fmax ? fabs(fb[i]) : fmax;
        }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) {
        cmax = fmax_(cmax, __shfl_xor_sync(FULL, cmax, o));
        fmax = fmax_(fmax, __shfl_xor_sync(FULL, fmax, o));
      }
      const double floor_ = 1e3 * DBL_EPSILON * (cmax + fmax);
      const double lim = tol > floor_ ? tol : floor_;
      if (have && !done && st == 0) {
        if (best_res <= lim) res = best_res;
        else st = PAQIF_LCP_NONCONVERGED;
      }
    }
    __syncwarp();
    if (have && gl == 0) {
#ifdef PAQIF_PROFILE_PHASES
      for (int q = 0; q < 4; ++q) { atomicAdd(&g_phase_cycles[q], ph_acc[q]); ph_acc[q] = 0; }
#endif
      if (passes_out) passes_out[b] = passes;
      // a breakdown reports -(1-based level) in res (include/paqif_b200.h)
      if (res_out) res_out[b] = brk_level ? -(double)brk_level : res;
      status_out[b] = st;
    }
    unsigned long long nx = 0;
    if (lane == 0) nx = atomicAdd(next_pair, 1ull);
    pair = total_warps + (int64_t)__shfl_sync(FULL, nx, 0);
  }
}

template <int BETA>
constexpr size_t lcp_smem_bytes() {
  return sizeof(LcpSmem<BETA>) * kLcpWarpsPerBlock * Group<BETA>::P;
}

constexpr size_t kLcpWsHead = 256;  // work counter of the persistent grid

template <int BETA>
size_t lcp_ws_per_slot(int n) {
  using PL = PivotLayout<BETA>;
  const int s = n / 2;
  size_t off = (((size_t)(s + 1) * PL::kSize * sizeof(double)) + 255) & ~(size_t)255;
  off += (((size_t)n * sizeof(double)) + 255) & ~(size_t)255;
  off += ((size_t)n * 8 + 255) & ~(size_t)255;
  off += ((size_t)n * 8 + 255) & ~(size_t)255;
  return off;
}

}  // namespace paqif

using namespace paqif;

namespace {

template <int BETA, bool EXACT, bool SOLVE_ONLY>
int lcp_grid_warps(int64_t B) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = lcp_smem_bytes<BETA>();
  cudaFuncSetAttribute(lcp_kernel<BETA, EXACT, SOLVE_ONLY>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lcp_kernel<BETA, EXACT, SOLVE_ONLY>,
                                                32 * kLcpWarpsPerBlock, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t w = (int64_t)sms * per_sm * kLcpWarpsPerBlock;
  const int64_t need = (B + Group<BETA>::P - 1) / Group<BETA>::P;
  if (w > need) w = need;
  return (int)(w < 1 ? 1 : w);
}

struct LcpDispatch {
  int64_t B;
  int n;
  const double* bands;
  const double* f;
  double tol;
  int max_outer;
  double* u;
  uint8_t* act;
  int64_t* passes;
  double* res;
  int64_t* status;
  void* ws;
  size_t ws_bytes;
  cudaStream_t st;
};

template <int BETA, bool EXACT, bool SOLVE_ONLY>
int run_lcp(const LcpDispatch& a) {
  const int warps = lcp_grid_warps<BETA, EXACT, SOLVE_ONLY>(a.B);
  const size_t per = lcp_ws_per_slot<BETA>(a.n);
  const size_t need = kLcpWsHead + per * (size_t)warps * Group<BETA>::P;
  if (a.ws_bytes < need) {
    std::snprintf(last_error_buf(), 512, "workspace too small: need %zu bytes", need);
    return PAQIF_E_WORKSPACE;
  }
  const unsigned grid = (unsigned)((warps + kLcpWarpsPerBlock - 1) / kLcpWarpsPerBlock);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(a.ws);
  cudaMemsetAsync(counter, 0, sizeof(unsigned long long), a.st);
  lcp_kernel<BETA, EXACT, SOLVE_ONLY><<<grid, 32 * kLcpWarpsPerBlock, lcp_smem_bytes<BETA>(), a.st>>>(
      a.B, a.n, a.bands, a.f, a.tol, a.max_outer, a.u, a.act, a.passes, a.res, a.status,
      (char*)a.ws + kLcpWsHead, per, warps, counter);
  return check_launch("lcp_kernel");
}

template <bool EXACT, bool SOLVE_ONLY>
int run_lcp_beta(int beta, const LcpDispatch& a) {
  switch (beta) {
    case 1: return run_lcp<1, EXACT, SOLVE_ONLY>(a);
    case 2: return run_lcp<2, EXACT, SOLVE_ONLY>(a);
    case 3: return run_lcp<3, EXACT, SOLVE_ONLY>(a);
    case 4: return run_lcp<4, EXACT, SOLVE_ONLY>(a);
    case 5: return run_lcp<5, EXACT, SOLVE_ONLY>(a);
    case 6: return run_lcp<6, EXACT, SOLVE_ONLY>(a);
    case 7: return run_lcp<7, EXACT, SOLVE_ONLY>(a);
    case 8: return run_lcp<8, EXACT, SOLVE_ONLY>(a);
    default: return set_arg_error("lcp: beta must be in 1..8");
  }
}

size_t ws_bytes_for(int64_t B, int64_t n, int64_t beta, bool exact) {
  size_t per = 0;
  int warps = 1;
  switch (beta) {
#define PAQIF_WS_CASE(BB)                                                        \
  case BB:                                                                       \
    per = lcp_ws_per_slot<BB>((int)n) * Group<BB>::P;                            \
    warps = exact ? lcp_grid_warps<BB, true, false>(B) : lcp_grid_warps<BB, false, false>(B); \
    break;
    PAQIF_WS_CASE(1)
    PAQIF_WS_CASE(2)
    PAQIF_WS_CASE(3)
    PAQIF_WS_CASE(4)
    PAQIF_WS_CASE(5)
    PAQIF_WS_CASE(6)
    PAQIF_WS_CASE(7)
    PAQIF_WS_CASE(8)
#undef PAQIF_WS_CASE
    default: return 0;
  }
  // solve-only and exact/fast variants share the layout; take the max grid
  int w2 = 1;
  switch (beta) {
#define PAQIF_WS_CASE2(BB)                                                              \
  case BB:                                                                              \
    w2 = exact ? lcp_grid_warps<BB, true, true>(B) : lcp_grid_warps<BB, false, true>(B); \
    break;
    PAQIF_WS_CASE2(1)
    PAQIF_WS_CASE2(2)
    PAQIF_WS_CASE2(3)
    PAQIF_WS_CASE2(4)
    PAQIF_WS_CASE2(5)
    PAQIF_WS_CASE2(6)
    PAQIF_WS_CASE2(7)
    PAQIF_WS_CASE2(8)
#undef PAQIF_WS_CASE2
  }
  return kLcpWsHead + per * (size_t)(warps > w2 ? warps : w2);
}

int check_lcp_args(int64_t B, int64_t n, int64_t beta) {
  if (B < 0 || n < 2 || (n & 1)) return set_arg_error("lcp: order must be even and >= 2");
  if (beta < 1 || beta > 8) return set_arg_error("lcp: beta must be in 1..8");
  if (n < 2 * beta + 2) return set_arg_error("lcp: block size must exceed 2*beta (PartitionError)");
  if (n > (1 << 26)) return set_arg_error("lcp: order too large");
  return PAQIF_OK;
}

}  // namespace

extern "C" size_t paqif_lcp_workspace_bytes(int64_t B, int64_t n, int64_t beta) {
  if (check_lcp_args(B, n, beta) || B == 0) return 0;
  const size_t a = ws_bytes_for(B, n, beta, true), b = ws_bytes_for(B, n, beta, false);
  return a > b ? a : b;
}

extern "C" int paqif_lcp_batch(int64_t B, int64_t n, int64_t beta, const double* bands,
                               const double* f, double tol, int64_t max_outer, uint32_t flags,
                               double* u, uint8_t* active, int64_t* passes, double* res,
                               int64_t* status, void* workspace, size_t workspace_bytes,
                               void* stream)
{
  if (int rc = check_lcp_args(B, n, beta)) return rc;
  if (B == 0) return PAQIF_OK;
  if (max_outer < 0 || max_outer > (1 << 30)) return set_arg_error("lcp: max_outer");
  LcpDispatch a{B, (int)n, bands, f, tol, (int)max_outer, u, active, passes, res, status,
                workspace, workspace_bytes, (cudaStream_t)stream};
  if (flags & PAQIF_FLAG_EXACT) return run_lcp_beta<true, false>((int)beta, a);
  return run_lcp_beta<false, false>((int)beta, a);
}

extern "C" int paqif_solve_r1_batch(int64_t B, int64_t n, int64_t beta, const double* bands,
                                    const double* f, double* x, int64_t* status, uint32_t flags,
                                    void* workspace, size_t workspace_bytes, void* stream)
{
  if (int rc = check_lcp_args(B, n, beta)) return rc;
  if (B == 0) return PAQIF_OK;
  LcpDispatch a{B, (int)n, bands, f, 0.0, 1, x, nullptr, nullptr, nullptr, status,
                workspace, workspace_bytes, (cudaStream_t)stream};
  if (flags & PAQIF_FLAG_EXACT) return run_lcp_beta<true, true>((int)beta, a);
  return run_lcp_beta<false, true>((int)beta, a);
}

namespace {
// Device staging reused across host-entry calls (grown on demand), so the
// host path pays for copies and the kernel, not for cudaMalloc each call.
#ifndef PAQIF_HOST_CHUNKS
#define PAQIF_HOST_CHUNKS 4
#endif
constexpr int kHostChunksMax = PAQIF_HOST_CHUNKS;

struct HostStage {
  std::mutex mu;
  char* buf = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr, st_in = nullptr, st_out = nullptr;
  cudaEvent_t ev[3][kHostChunksMax] = {};
  int device = -1;
  char* get(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != device) {
      // a different device: the old allocation belongs to another context
      buf = nullptr;
      cap = 0;
      st = st_in = st_out = nullptr;
      for (auto& row : ev)
        for (auto& e : row) e = nullptr;
      device = dev;
    }
    if (!st && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (!st_in && cudaStreamCreateWithFlags(&st_in, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (!st_out && cudaStreamCreateWithFlags(&st_out, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    for (auto& row : ev)
      for (auto& e : row)
        if (!e && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    if (bytes > cap) {
      if (buf) cudaFree(buf);
      buf = nullptr;
      cap = 0;
      if (cudaMalloc(&buf, bytes) != cudaSuccess) return nullptr;
      cap = bytes;
    }
    return buf;
  }
};
HostStage& host_stage() {
  static HostStage h;
  return h;
}
size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" int paqif_lcp_batch_host(int64_t B, int64_t n, int64_t beta, const double* bands,
                                    const double* f, double tol, int64_t max_outer,
                                    uint32_t flags, double* u, uint8_t* active, int64_t* passes,
                                    double* res, int64_t* status)
{
  if (int rc = check_lcp_args(B, n, beta)) return rc;
  if (B == 0) return PAQIF_OK;
  const size_t nb = (size_t)B * (2 * beta + 1) * n, nv = (size_t)B * n;
  const size_t wsb = paqif_lcp_workspace_bytes(B, n, beta);
  const size_t o_b = 0, o_f = o_b + al256(nb * 8), o_u = o_f + al256(nv * 8),
               o_a = o_u + al256(nv * 8), o_p = o_a + al256(nv), o_r = o_p + al256(B * 8),
               o_s = o_r + al256(B * 8), o_w = o_s + al256(B * 8), total = o_w + al256(wsb);
  HostStage& hs = host_stage();
  std::lock_guard<std::mutex> lock(hs.mu);
  char* base = hs.get(total);
  if (!base) return set_cuda_error("lcp_host: device staging", cudaErrorMemoryAllocation);
  cudaStream_t st = hs.st;
  double* d_b = (double*)(base + o_b);
  double* d_f = (double*)(base + o_f);
  double* d_u = (double*)(base + o_u);
  uint8_t* d_a = (uint8_t*)(base + o_a);
  int64_t* d_p = (int64_t*)(base + o_p);
  double* d_r = (double*)(base + o_r);
  int64_t* d_s = (int64_t*)(base + o_s);
  int rc = PAQIF_OK;
  cudaError_t e;
  // Chunked pipeline: the H2D copy of chunk c+1 (copy stream) overlaps the
  // solve of chunk c (compute stream), whose D2H overlaps chunk c+1's solve.
  // The host link, not the solve, bounds this entry point for config 2;
  // chunks below ~1000 systems would hit the solve's latency floor, so big
  // batches use up to kHostChunksMax chunks.
  const int64_t chunks = B >= 2048 ? kHostChunksMax : 1;
  const int64_t per = (B + chunks - 1) / chunks;
  const size_t rowb = (size_t)(2 * beta + 1) * n;
  for (int64_t c = 0; c < chunks && !rc; ++c) {
    const int64_t b0 = c * per, bc = (b0 + per <= B ? per : B - b0);
    if (bc <= 0) break;
    if ((e = cudaMemcpyAsync(d_b + b0 * rowb, bands + b0 * rowb, bc * rowb * 8,
                             cudaMemcpyHostToDevice, hs.st_in)) != cudaSuccess ||
        (e = cudaMemcpyAsync(d_f + b0 * n, f + b0 * n, bc * n * 8, cudaMemcpyHostToDevice,
                             hs.st_in)) != cudaSuccess ||
        (e = cudaEventRecord(hs.ev[0][c], hs.st_in)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(st, hs.ev[0][c], 0)) != cudaSuccess) {
      rc = set_cuda_error("lcp_host: h2d", e);
      break;
    }
    rc = paqif_lcp_batch(bc, n, beta, d_b + b0 * rowb, d_f + b0 * n, tol, max_outer, flags,
                         d_u + b0 * n, d_a + b0 * n, d_p + b0, d_r + b0, d_s + b0, base + o_w,
                         wsb, st);
    if (rc) break;
    if ((e = cudaEventRecord(hs.ev[1][c], st)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(hs.st_out, hs.ev[1][c], 0)) != cudaSuccess ||
        (e = cudaMemcpyAsync(u + b0 * n, d_u + b0 * n, bc * n * 8, cudaMemcpyDeviceToHost,
                             hs.st_out)) != cudaSuccess ||
        (e = cudaMemcpyAsync(active + b0 * n, d_a + b0 * n, bc * n, cudaMemcpyDeviceToHost,
                             hs.st_out)) != cudaSuccess ||
        (e = cudaMemcpyAsync(passes + b0, d_p + b0, bc * 8, cudaMemcpyDeviceToHost,
                             hs.st_out)) != cudaSuccess ||
        (e = cudaMemcpyAsync(res + b0, d_r + b0, bc * 8, cudaMemcpyDeviceToHost,
                             hs.st_out)) != cudaSuccess ||
        (e = cudaMemcpyAsync(status + b0, d_s + b0, bc * 8, cudaMemcpyDeviceToHost,
                             hs.st_out)) != cudaSuccess)
      rc = set_cuda_error("lcp_host: d2h", e);
  }
  cudaError_t e1 = cudaStreamSynchronize(hs.st_in);
  cudaError_t e2 = cudaStreamSynchronize(st);
  e = cudaStreamSynchronize(hs.st_out);
  if (!rc && e1 != cudaSuccess) rc = set_cuda_error("lcp_host: sync", e1);
  if (!rc && e2 != cudaSuccess) rc = set_cuda_error("lcp_host: sync", e2);
  if (!rc && e != cudaSuccess) rc = set_cuda_error("lcp_host: sync", e);
  return rc;
}
