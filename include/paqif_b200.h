/*
 * paqif_b200.h -- C ABI of the B200-native PAQIF / EHL Newton-step library
 * (libpaqif_b200.so).  Plain pointers and sizes only; no exceptions cross the
 * boundary.  Every function returns 0 (PAQIF_OK) or a negative PAQIF_E_*
 * error code; per-system numerical outcomes are reported through int64
 * status arrays exactly as the reference kernels do.
 *
 * Pointers marked [dev] are CUDA device pointers (or managed memory); [host]
 * pointers are host memory (pinned recommended).  `stream` is a cudaStream_t
 * (NULL = legacy default stream).  Device-pointer entry points are
 * asynchronous on `stream`; host-pointer (`*_host`) entry points copy in,
 * run and copy out synchronously.
 *
 * Array shapes follow the reference's batched kernels (all C-contiguous,
 * float64 unless noted; s = n/2, n even):
 *   band, anti  (B, 2*beta+1, n)   diagonal-major: band[b,d,i] = A(i, i+d-beta)
 *   z2x2        (B, s+1, 2, 2)     level corners (level index 0 unused)
 *   zl, zr      (B, s+1, 2, beta+1)
 *   ww          (B, s+1, 2*beta, 2)
 *   status      (B,) int64         0 or the 1-based breakdown level
 *   trace       (B, n) int64       resolution order, -1 padded
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/paqif):
 *   paqif_factor_batch        _kernels.factor_batch       _kernels.py:62-149
 *   paqif_solve_w_batch       _kernels.solve_w_batch      _kernels.py:152-172
 *   paqif_solve_z_batch       _kernels.solve_z_batch      _kernels.py:175-225
 *   paqif_band_matvec_batch   _kernels.band_matvec_batch  _kernels.py:228-241
 *   paqif_psor_sweeps         _kernels.psor_sweeps        _kernels.py:244-276
 *   paqif_lcp_batch(_host)    parallel.paqif_solve_lcp(problem, r=1) per system,
 *                             parallel.py:298-347 (fused: factor + W + corner
 *                             normal equations + Z + complementarity loop)
 *   paqif_solve_r1_batch      parallel.paqif_solve(l, f, r=1) per system,
 *                             parallel.py:261-295
 */
#ifndef PAQIF_B200_H
#define PAQIF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define PAQIF_OK 0
#define PAQIF_E_ARG (-1)        /* bad size / odd order / unsupported beta   */
#define PAQIF_E_CUDA (-2)       /* CUDA runtime error (see paqif_last_error) */
#define PAQIF_E_WORKSPACE (-3)  /* workspace too small                        */

/* per-system LCP status (paqif_lcp_batch status[]) */
#define PAQIF_LCP_OK 0
#define PAQIF_LCP_FACTOR_BREAKDOWN 1 /* FactorizationBreakdownError (aqif.py:133-134) */
#define PAQIF_LCP_ZSOLVE_BREAKDOWN 2 /* FactorizationBreakdownError "z-solve" (aqif.py:174-175) */
#define PAQIF_LCP_NOT_PD 3           /* NotPositiveDefiniteError (bandcore.py:179-182) */
#define PAQIF_LCP_NONCONVERGED 4     /* NonConvergenceError (parallel.py:346-347) */

/* flags */
#define PAQIF_FLAG_EXACT 1u /* reference rounding: no FMA, IEEE division (bit-exact kernels) */
/* EHL line steps (paqif_ehl.h): the path for a batch of cases.  Default:
 * the fused one-CTA-per-case kernel below 2 x SM-count cases, the split
 * three-kernel path (phase A / batched rung solves / phase C) from there. */
#define PAQIF_FLAG_LINE_SPLIT 2u /* force the split path */
#define PAQIF_FLAG_LINE_FUSED 4u /* force the fused path */

/* library identity / diagnostics */
const char *paqif_version(void);
const char *paqif_last_error(void);
int paqif_device_count(void);

/* ------------------------------------------------------------------ AQIF kernels */
/* In-place W0 Z0 factorization of B banded systems (band consumed, anti zero on entry). */
int paqif_factor_batch(int64_t B, int64_t n, int64_t beta, double *band /*[dev]*/,
                       double *anti /*[dev]*/, double *z2x2 /*[dev]*/, double *zl /*[dev]*/,
                       double *zr /*[dev]*/, double *ww /*[dev]*/, double tol,
                       int64_t *status /*[dev]*/, uint32_t flags, void *stream);

/* Middle-out solve W0 y = rhs in place. */
int paqif_solve_w_batch(int64_t B, int64_t n, int64_t beta, const double *ww /*[dev]*/,
                        double *rhs /*[dev]*/, uint32_t flags, void *stream);

/* Outside-in solve Z0 x = y from pair level `start` (x prefilled below it). */
int paqif_solve_z_batch(int64_t B, int64_t n, int64_t beta, const double *z2x2 /*[dev]*/,
                        const double *zl /*[dev]*/, const double *zr /*[dev]*/,
                        const double *y /*[dev]*/, double *x /*[dev]*/, int64_t start,
                        double tol, int64_t *status /*[dev]*/, int64_t *trace /*[dev], may be NULL*/,
                        uint32_t flags, void *stream);

/* out = A x for diagonal-major banded A. */
int paqif_band_matvec_batch(int64_t B, int64_t n, int64_t beta, const double *bands /*[dev]*/,
                            const double *x /*[dev]*/, double *out /*[dev]*/, void *stream);

/* Projected SOR on one banded LCP (sequential oracle; returns sweeps via *sweeps). */
int paqif_psor_sweeps(int64_t n, int64_t beta, const double *bands /*[dev]*/,
                      const double *f /*[dev]*/, double *u /*[dev]*/, double omega, double tol,
                      int64_t max_sweeps, int64_t *sweeps /*[host]*/, double *change /*[host]*/,
                      void *stream);

/* ------------------------------------------------------------------ solvers */
/* paqif_solve(L_b, f_b, r=1) for every system b (status 0/1/2/3 as LCP codes). */
int paqif_solve_r1_batch(int64_t B, int64_t n, int64_t beta, const double *bands /*[dev]*/,
                         const double *f /*[dev]*/, double *x /*[dev]*/,
                         int64_t *status /*[dev]*/, uint32_t flags, void *workspace /*[dev]*/,
                         size_t workspace_bytes, void *stream);

/* Workspace needed by paqif_lcp_batch / paqif_solve_r1_batch for (B, n, beta). */
/* r-block partitioned PAQIF, all seven steps on the device (paqif_solve,
 * parallel.py:106-295): B systems of order n = r*t (t even, t > 2 beta),
 * beta <= 16.  bands [dev] (B, 2beta+1, n), f [dev] (B, n), x [dev] (B, n)
 * out; project != 0 clamps corners and middles at zero (the LCP pass);
 * status [dev] (B,) PAQIF_LCP_* (factor / z-solve breakdown, reduced system
 * not SPD).  The reduced system (order 2 beta r) is solved through its
 * normal equations with a banded Cholesky; rounding differs from the
 * reference's numpy/LAPACK there. */
size_t paqif_solve_rblock_workspace_bytes(int64_t B, int64_t n, int64_t beta, int64_t r);
int paqif_solve_rblock_batch(int64_t B, int64_t n, int64_t beta, int64_t r,
                             const double *bands, const double *f, double *x, int32_t project,
                             int64_t *status, uint32_t flags, void *workspace,
                             size_t workspace_bytes, void *stream);

/* Active-set pass helpers for paqif_solve_lcp with r > 1 (parallel.py:
 * 312-343), batched, [dev] pointers.  _pin: lmod/fmod of the active rows
 * (diagonal kept, 1 if zero; right side 0).  _pass: lam = L u_eval - f,
 * u = max(u_eval, 0), res[b] = max|min(u, L u - f)|, new_active = u_eval < lam,
 * changed[b] = new_active differs from active. */
int paqif_lcp_pin_batch(int64_t B, int64_t n, int64_t beta, const double *bands, const double *f,
                        const uint8_t *active, double *lmod, double *fmod, void *stream);
int paqif_lcp_pass_batch(int64_t B, int64_t n, int64_t beta, const double *bands,
                         const double *f, const double *u_eval, const uint8_t *active,
                         double *u, uint8_t *new_active, double *res, int32_t *changed,
                         void *stream);

size_t paqif_lcp_workspace_bytes(int64_t B, int64_t n, int64_t beta);

/* Fused batched projected LCP: u >= 0, L u >= f, u.(L u - f) = 0 for every
 * system, following paqif_solve_lcp(problem, r=1, tol, max_outer) exactly:
 * same active-set policy, same pass count, same termination rules.
 * Outputs: u (B,n) solution, active (B,n) uint8 pinned set of the returned
 * pass, passes (B,) int64, res (B,) final complementarity residual,
 * status (B,) int64 PAQIF_LCP_*.  On a breakdown (status 1 or 2) res[b]
 * holds -(the 1-based breakdown level), which the Python layer passes on as
 * FactorizationBreakdownError.level (aqif.py:133-134, 174-175). */
int paqif_lcp_batch(int64_t B, int64_t n, int64_t beta, const double *bands /*[dev]*/,
                    const double *f /*[dev]*/, double tol, int64_t max_outer, uint32_t flags,
                    double *u /*[dev]*/, uint8_t *active /*[dev]*/, int64_t *passes /*[dev]*/,
                    double *res /*[dev]*/, int64_t *status /*[dev]*/, void *workspace /*[dev]*/,
                    size_t workspace_bytes, void *stream);

/* Same, host buffers in and out (H2D, kernel, D2H on an internal stream). */
int paqif_lcp_batch_host(int64_t B, int64_t n, int64_t beta, const double *bands /*[host]*/,
                         const double *f /*[host]*/, double tol, int64_t max_outer,
                         uint32_t flags, double *u /*[host]*/, uint8_t *active /*[host]*/,
                         int64_t *passes /*[host]*/, double *res /*[host]*/,
                         int64_t *status /*[host]*/);

#ifdef __cplusplus
}
#endif
#endif /* PAQIF_B200_H */
