/* C ABI of the TVD kappa-scheme line-splitting sweeps (the paper's Sec. 6
 * linear study) -- paqif/tvdcd.py of the reference.  [dev] pointers are
 * device memory; every call is asynchronous on `stream` (NULL = legacy
 * default stream); return 0 or a PAQIF_E_* code (paqif_last_error()). */
#ifndef PAQIF_TVD_H
#define PAQIF_TVD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One discrete problem (ConvectionDiffusionProblem, tvdcd.py:312-343) and
 * its x-line splitting (tvdcd.py:374-416).  Fields are u[j, i], x-lines
 * contiguous; planes are ny x nx. */
typedef struct {
  int32_t nx, ny;        /* solved grid */
  int32_t kx, ky;        /* StencilOperator.cx / .cy entries (<= 4 each) */
  int32_t ox[4], oy[4];  /* their offsets, in the dicts' iteration order */
  int32_t line_mask;     /* bit t: line band offset t-2 present (t = 0..3:
                            offsets -2, -1, 0, +1 of _line_system_coeffs) */
  int32_t reserved;
  double omega;          /* relaxation of the line changes */
  double h2;             /* grid.h ** 2 (the residual norm's weight) */
  const double *f;       /* [dev] ny x nx right side */
  const double *c0;      /* [dev] ny x nx operator centre */
  const double *cx;      /* [dev] kx planes */
  const double *cy;      /* [dev] ky planes */
  const double *lb;      /* [dev] 4 planes: line bands at offsets -2..+1 */
  /* Shared line factorization (constant-coefficient lines, as the
   * reference caches it, tvdcd.py:466-477): the WZFactors arrays of
   * paqif_factor_batch for one system of the padded line order, [dev];
   * z2x2 NULL = factor every line.  Then each line is solve_w + solve_z
   * (aqif.py:138-178) on the shared factors. */
  const double *z2x2, *zl, *zr, *ww;
  int32_t zf_beta;
  int32_t reserved2;
} paqif_tvd_problem;

/* sweep_splitting(problem, u, variant in {Ls0, Ls1, Ls2}, omega, order)
 * (tvdcd.py:449-489): u_full [dev] (ny+4) x (nx+4), the data ring with the
 * iterate embedded (ConvectionDiffusionProblem.embed), updated in place
 * line by line; backward = 1 scans lines ny-1..0.  want_norm = 1 also
 * writes residual_norm(u_next) to norm [dev] 1, using resid [dev]
 * (paqif_tvd_resid_bytes) as scratch.  status [dev] 1: 0, or 1 + the line
 * whose factorization broke down (FactorizationBreakdownError). */
int paqif_tvd_sweep(const paqif_tvd_problem *p, double *u_full, int32_t backward,
                    int32_t want_norm, double *resid, double *norm, int32_t *status,
                    void *stream);
size_t paqif_tvd_resid_bytes(int32_t nx, int32_t ny);

/* sweep_splitting(problem, u, "Ls3", omega) (tvdcd.py:615-656): every
 * x-line's change from the current iterate (one CTA per line), then
 * u += omega (sigma - spread / 4) and residual_norm(u_next) into norm [dev].
 * a_over_h [dev] ny x nx = a / h; line_bands [dev] 5 planes (offsets -2..2
 * of the distributive line operator); k1 = (1 + kappa) / 4, k2 =
 * (1 - kappa) / 4; sigma [dev] ny x nx and line_status [dev] ny scratch;
 * status [dev] 1: 0 or 1 + the first line whose factorization broke down
 * (then u_full is unchanged). */
int paqif_tvd_distributive(const paqif_tvd_problem *p, double *u_full, const double *a_over_h,
                           const double *line_bands, double k1, double k2, double *sigma,
                           int32_t *line_status, double *resid, double *norm, int32_t *status,
                           void *stream);

/* Interior of src_full (ny+4) x (nx+4) into the interior of dst_full
 * (nx+4) x (ny+4), transposed: the hand-over to transposed_problem's twin
 * (tvdcd.py:492-511, solve_by_sweeps' "t" passes). */
int paqif_tvd_transpose(const double *src_full, int32_t ny, int32_t nx, double *dst_full,
                        void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PAQIF_TVD_H */
