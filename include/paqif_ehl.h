/*
 * paqif_ehl.h -- C ABI of the fused EHL Newton steps (libpaqif_b200.so).
 * Same conventions as paqif_b200.h (return codes, [dev] pointers, streams).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/paqif):
 *   paqif_ehl_line_step   one outer iteration of ehl.solver.solve_ehl for the
 *                         line contact, for B independent load cases:
 *                         _line_contact_sweep (ehl/solver.py:131-183),
 *                         force_balance_update (ehl/sweeps.py:521-535, when
 *                         (outer+1) % force_every == 0) and
 *                         EhlState.complementarity_residual (ehl/solver.py:43-51).
 */
#ifndef PAQIF_EHL_H
#define PAQIF_EHL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Line-contact step configuration, common to the batch (EhlParams fields,
 * ehl/params.py:40-58, plus the solve_ehl arguments). */
typedef struct {
  int32_t n;            /* grid intervals; nodes = n + 1                     */
  int32_t limiter;      /* 0 kappa, 1 none, 2 van-albada, 3 minmod, 4 koren  */
  int32_t variant;      /* 0 Lhs1 (Ls1/Ls4), 1 Lhs2 (Ls0/Ls5)                */
  int32_t compressible; /* Dowson-Higginson + Roelands (1) or unit (0)       */
  int32_t force_every;  /* force-balance period                              */
  int32_t outer;        /* 0-based outer iteration index of this step        */
  double h, lo;         /* spacing and left end of the domain                */
  double kappa, omega, max_change, relax_c, max_h0_step, load_target;
  double alpha, z, p0;  /* pressure-viscosity constants                      */
} paqif_ehl_line_cfg;

/* Workspace for paqif_ehl_line_step (B cases on n intervals). */
size_t paqif_ehl_line_workspace_bytes(int64_t B, int64_t n);

/* One outer iteration for every case b (one CTA per case).
 *   table   [dev] (n+1)      line kernel cell integrals (kernels.kernel_line)
 *   p_hertz [dev] (B)        per-case p_H;  lam [dev] (B) per-case lambda
 *   u       [dev] (B, n+1)   pressure in, updated pressure out
 *   h0      [dev] (B)        offset in/out
 *   film    [dev] (B, n+1)   film of the new state (out)
 *   res     [dev] (B)        complementarity residual of the new state (out)
 *   deficit [dev] (B)        load deficit target - h*sum(u) if the force balance
 *                            ran this step, else NaN (out, may be NULL)
 *   info    [dev] (B) int32  bits 0-1: solve rung (0 combined system, 1..3 Ls4
 *                            ladder scheme / first-order / diagonal), bit 2:
 *                            force balance applied, bit 3: non-finite change,
 *                            bit 8: every rung broke down, bits 16..: number of
 *                            weighted (eps/h <= 0.6) rows */
int paqif_ehl_line_step(const paqif_ehl_line_cfg *cfg, int64_t B, const double *table,
                        const double *p_hertz, const double *lam, double *u, double *h0,
                        double *film, double *res, double *deficit, int32_t *info,
                        uint32_t flags, void *workspace, size_t workspace_bytes, void *stream);

/* Device-side solve_ehl loop for line contacts (ehl/solver.py:210-240), one
 * record per case.  The stop and divergence tests run in the kernel epilogue
 * with the reference's comparisons, so a case that stopped turns every later
 * launch into a no-op and the host only synchronises once per chunk. */
typedef struct {
  double tol, tol_fb;   /* stop test: res <= tol and |deficit| <= tol_fb       */
  double best;          /* best residual so far (start +inf)                   */
  double deficit;       /* |deficit| of the last force balance (start +inf)    */
  int32_t max_outer;    /* iteration budget                                    */
  int32_t outer;        /* iterations done (also the force-balance phase)      */
  int32_t grow;         /* iterations without a new best residual              */
  int32_t done;         /* 0 running, 1 converged, 2 diverging (grow >= 20 and
                           res > 1e3 max(best, tol)), 3 budget spent, 4 every
                           Ls4 rung broke down, 5 non-finite change            */
} paqif_ehl_line_drive;

/* Enqueues `steps` outer iterations of paqif_ehl_line_step for every case
 * still running (drive[b].done == 0), taking the iteration index from
 * drive[b].outer.  Iteration k of case b writes its residual and its load
 * deficit (NaN when no force balance ran) to hist_res / hist_def
 * [b * hist_cap + k % hist_cap] ([dev], may be NULL).  Other arguments as in
 * paqif_ehl_line_step; cfg->outer is ignored. */
int paqif_ehl_line_drive_steps(const paqif_ehl_line_cfg *cfg, int64_t B, int32_t steps,
                               const double *table, const double *p_hertz, const double *lam,
                               double *u, double *h0, double *film, double *res,
                               double *deficit, int32_t *info, paqif_ehl_line_drive *drive,
                               double *hist_res, double *hist_def, int32_t hist_cap,
                               uint32_t flags, void *workspace, size_t workspace_bytes,
                               void *stream);

/* Complementarity residual max|min(u, -R(u))|/h and film of B line states
 * (EhlState.complementarity_residual / film_field, ehl/solver.py:40-51);
 * [dev] pointers as in paqif_ehl_line_step, film may be NULL. */
int paqif_ehl_line_residual(const paqif_ehl_line_cfg *cfg, int64_t B, const double *table,
                            const double *p_hertz, const double *lam, const double *u,
                            const double *h0, double *film, double *res, void *stream);

/* Line deformation  d_b[i] = -(1/pi) sum_j table[|i-j|] u_b[j]  for B pressure
 * vectors of n+1 nodes (FilmModel.deformation_full, ehl/film.py:67-71). */
int paqif_line_deformation(int64_t B, int64_t n, const double *table /*[dev] n+1*/,
                           const double *u /*[dev] (B, n+1)*/, double *out /*[dev] (B, n+1)*/,
                           void *stream);

/* ------------------------------------------------------- line systems
 * The per-line building blocks of paqif/ehl/sweeps.py on the GPU, for
 * callers that work line by line with the reference's arrays ([dev]
 * pointers, one CTA per call). */
typedef struct {
  int32_t n;        /* intervals: nodes n + 1, unknowns n - 1               */
  int32_t limiter;  /* 0 kappa, 1 none, 2 van-albada, 3 minmod, 4 koren    */
  int32_t weighted; /* 1: Ls4/Ls5 distributive pattern, 0: Ls1/Ls0         */
  int32_t reserved;
  double kappa;
  double ks0, ks1;  /* kernel strengths (film sensitivity x kernel_nu,
                       sweeps.py:190-199, computed by the caller)          */
  double h, hy;     /* spacing; hy = h (point contact) or 1 (line)         */
  const double *q, *rho;                              /* [dev] n + 1       */
  const double *ex_p, *ex_m, *ey_p, *ey_m, *resid;    /* [dev] n - 1       */
} paqif_ehl_linesys;

/* assemble_line_system (ehl/sweeps.py:157-267; splitting_ls4/ls5 are the
 * weighted pattern): the padded change matrix of order n_sys (n - 1 rounded
 * up to even) in BandedMatrix layout bands[(d + 2) * n_sys + i] (beta = 2)
 * and its right side rhs[n_sys].  jacobian: 0 scheme, 1 first-order,
 * 2 diagonal. */
int paqif_ehl_assemble_line(const paqif_ehl_linesys *a, int32_t jacobian,
                            double *bands /*[dev] 5 x n_sys*/, double *rhs /*[dev] n_sys*/,
                            void *stream);

/* robust_line_solve (ehl/sweeps.py:270-295): scheme, first-order, diagonal
 * Jacobians until the AQIF factorization succeeds; sigma[n - 1] and the rung
 * that solved (-1: every rung broke down, the reference re-raises). */
int paqif_ehl_robust_line_solve(const paqif_ehl_linesys *a, double *sigma /*[dev] n-1*/,
                                int32_t *rung /*[dev] 1*/, void *stream);

typedef struct {
  int32_t compressible;
  int32_t reserved;
  double alpha, z, p0, p_hertz, lam;
} paqif_ehl_rheo;

/* reynolds_residual_field (ehl/sweeps.py:106-138): the residual of the
 * discrete balance on every interior node, boundary entries zero; u and
 * film are (n+1) (point = 0) or (n+1) x (n+1) (point = 1). */
int paqif_ehl_residual_field(const double *u, const double *film, int64_t n, int32_t point,
                             const paqif_ehl_rheo *rheo, double h, int32_t limiter,
                             double kappa, double *r, void *stream);

/* ------------------------------------------------------------ point contact
 * One outer iteration of ehl.solver.solve_ehl for the circular point contact
 * (configs 4/5) on an (n+1)^2 grid, in the reference's Gauss-Seidel order:
 *   _hybrid_x_sweep (ehl/solver.py:76-128; per-row Newton Ls1 or weighted Ls4
 *   by min(eps)/h > 0.6), column_sweep (ehl/sweeps.py:421-518),
 *   force_balance_update (ehl/sweeps.py:521-535, weight h^2) and
 *   complementarity_residual (ehl/solver.py:43-51).
 * The deformation is FilmModel('point') (ehl/film.py:43-155): fp64 FFT
 * convolution plus exact pending-line corrections, folded after > 8 pending
 * updates.  The handle owns all device state (one CUDA stream, HBM resident
 * pressure / deformation / film fields); a native host loop drives the
 * 2(n-1) line kernels. */
typedef struct {
  int32_t n;            /* grid intervals per axis                            */
  int32_t limiter;      /* 0 kappa, 1 none, 2 van-albada, 3 minmod, 4 koren   */
  int32_t variant;      /* 0 Lhs1 (Ls1/Ls4), 1 Lhs2 (Ls0/Ls5)                 */
  int32_t compressible; /* Dowson-Higginson + Roelands (1) or unit (0)        */
  int32_t force_every;  /* force-balance period                               */
  int32_t outer;        /* ignored in the cfg; passed to _step                */
  double h;             /* spacing (both axes)                                */
  double kappa, omega, max_change, relax_c, max_h0_step, load_target;
  double alpha, z, p0;  /* pressure-viscosity constants                       */
  double p_hertz, lam;  /* case constants (EhlParams.point_from_moes)          */
} paqif_ehl_point_cfg;

typedef struct paqif_ehl_point paqif_ehl_point;

/* Creates the solver state; table (kernels.kernel_point) and geometry
 * (0.5 (x^2 + y^2)) are HOST (n+1)^2 row-major arrays [j][i].  NULL on error
 * (paqif_last_error). */
paqif_ehl_point *paqif_ehl_point_create(const paqif_ehl_point_cfg *cfg, const double *table,
                                        const double *geometry);
void paqif_ehl_point_destroy(paqif_ehl_point *h);

/* Loads pressure u (HOST (n+1)^2) and offset h0; recomputes the deformation. */
int paqif_ehl_point_set_state(paqif_ehl_point *h, const double *u, double h0);

/* Enqueues one outer iteration (asynchronous on the handle's stream). */
int paqif_ehl_point_step(paqif_ehl_point *h, int32_t outer, uint32_t flags);

/* Device-side solve_ehl loop for the point contact (ehl/solver.py:210-240):
 * enqueues `steps` outer iterations; after each, the stop / divergence tests
 * run on the device against `drive` ([dev], the line contact's record type;
 * its `outer` is the iteration index and sets the force-balance schedule).
 * Once the record is done (1 converged, 2 diverging, 3 budget, 4 every rung
 * of a line solve broke down, 5 non-finite change -- 4/5 stop before the
 * residual is recorded) every later enqueued kernel returns at once, so the
 * host synchronises once per chunk.  hist_res / hist_def ([dev], may be
 * NULL) receive the residual and the load deficit (NaN without a force
 * balance) of iteration k at k % hist_cap. */
int paqif_ehl_point_drive_steps(paqif_ehl_point *h, int32_t steps, paqif_ehl_line_drive *drive,
                                double *hist_res, double *hist_def, int32_t hist_cap,
                                uint32_t flags);

/* Enqueues one sweep of the public sweep functions on the resident state:
 *   kind 0  _hybrid_x_sweep         (ehl/solver.py:76-128)
 *   kind 1  newton_line_sweep       (ehl/sweeps.py:344-379; immediate updates)
 *   kind 2  weighted_change_sweep   (ehl/sweeps.py:382-418; deferred, spread)
 *   kind 3  column_sweep            (ehl/sweeps.py:421-518)
 * sel: line system of the x-sweeps, -1 by min(eps)/h > 0.6 (hybrid_select),
 * 0 Newton (Ls0/Ls1), 1 weighted (Ls4/Ls5); nu_variant 0 Ls1/Ls4, 1 Ls0/Ls5
 * (kernel_nu); omega the under-relaxation.  The sweep's worst |resid|
 * (the functions' return value) is reported by _get. */
int paqif_ehl_point_sweep(paqif_ehl_point *h, int32_t kind, int32_t sel, int32_t nu_variant,
                          double omega, uint32_t flags);

/* force_balance_update (ehl/sweeps.py:521-535), enqueued. */
int paqif_ehl_point_force_balance(paqif_ehl_point *h);

/* EhlState.complementarity_residual and film_full (ehl/solver.py:40-51),
 * enqueued; read with _get. */
int paqif_ehl_point_residual(paqif_ehl_point *h);

/* Synchronises and copies results to HOST buffers (any may be NULL):
 *   u, film (n+1)^2;  scal[4] = {h0, complementarity residual, deficit of the
 *   last force balance, worst |resid| of the last sweep / step};
 *   xinfo (n-1): bit 0 Newton system (Ls0/Ls1), bit 1 deferred update,
 *                bits 4..5 ladder rung (3 = failed);
 *   yinfo (n-1): rung (0 tridiagonal, 1 diagonal, 3 failed);
 *   err: bit 0/2 an x/y line broke down on every rung, 1/3 non-finite change */
int paqif_ehl_point_get(paqif_ehl_point *h, double *u, double *film, double *scal,
                        int32_t *xinfo, int32_t *yinfo, int32_t *err);
int paqif_ehl_point_sync(paqif_ehl_point *h);

/* The handle's CUDA stream (cudaStream_t), for event timing and ordering. */
void *paqif_ehl_point_stream(paqif_ehl_point *h);

/* FilmModel.note_line_update (ehl/film.py:83-91): record an applied line
 * change -- axis 0 row / 1 column at `index`, delta [host] (n+1) -- as a
 * pending update; an all-zero delta is ignored.  At most 9 may be pending:
 * the caller folds (paqif_ehl_point_deformation clears the list) once more
 * than 8 are, as the reference does. */
int paqif_ehl_point_note_update(paqif_ehl_point *h, int32_t axis, int32_t index,
                                const double *delta);

/* FilmModel.film_rows / film_cols (ehl/film.py:125-146): h0 + geometry +
 * base deformation + pending corrections on L lines (mode 0 rows, 1
 * columns; indices idx [host] L) -> out [host] L x (n+1). */
int paqif_ehl_point_film_lines(paqif_ehl_point *h, int32_t mode, const int32_t *idx, int32_t L,
                               double h0, double *out);

/* Deformation of HOST pressure u into HOST out (FilmModel.deformation_full). */
int paqif_ehl_point_deformation(paqif_ehl_point *h, const double *u, double *out);

/* Config 5 on several GPUs: every rank runs the same
 * contact (the line chains in the reference's order, replicated); after
 * attach_peers every full deformation of the handle is split over the
 * ranks -- row FFTs, column FFTs x kernel spectrum, inverse row FFTs, each
 * rank its slab, written straight into the peers' buffers over NVLink with
 * a system-scope barrier between the phases -- bit-identical to the
 * one-GPU fold.  ipc_handles: this handle's 3 x 64-byte CUDA IPC handles;
 * attach_peers: all ranks' handles (world x 3 x 64 bytes, rank order),
 * world <= 8.  A peer that never reaches a barrier sets err bit 64
 * (PaqifError) after ~seconds instead of hanging. */
int paqif_ehl_point_ipc_handles(paqif_ehl_point *h, void *out /*[host] 192 bytes*/);
int paqif_ehl_point_attach_peers(paqif_ehl_point *h, int32_t rank, int32_t world,
                                 const void *handles /*[host] world x 192 bytes*/);
/* test: the sharded decomposition with `world` ranks emulated in order on
 * one GPU, deformation of u [host] into out [host] */
int paqif_ehl_point_fold_emulated(paqif_ehl_point *h, int32_t world, const double *u,
                                  double *out);
/* bench: `reps` forced folds of the resident pressure (sharded when
 * attached), enqueued on the handle's stream */
int paqif_ehl_point_fold_bench(paqif_ehl_point *h, int32_t reps);

/* Deformation kernel tables on the device (ehl/kernels.py:64-100,
 * kernel_line / kernel_point): table [dev] nx+1 doubles, the cell integrals
 * of log|x - x'| for offsets 0..nx; or (nx+1) x (ny+1) row-major, the
 * eight-term asinh form times `scale` (the caller passes 2.0 / np.pi**2 so
 * the constant is the reference's).  Within a few ulp of the host tables
 * (library log / asinh rounding). */
int paqif_ehl_kernel_line(int64_t nx, double h, double *table, void *stream);
int paqif_ehl_kernel_point(int64_t nx, int64_t ny, double h, double scale, double *table,
                           void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PAQIF_EHL_H */
