/*
 * oracle/paqif_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference's PAQIF numerical kernels and
 * of the r=1 projected-LCP driver.  It exists so that tests/, bench.py's
 * cpu_baseline / --impl reference arm and __graft_entry__.smoke() have a
 * checker that travels to the GPU box (where /root/reference is absent).
 * Nothing in the product package links or calls this file.
 *
 * Compiled with -O2 -ffp-contract=off so every expression rounds exactly
 * like the reference (numba @njit with fastmath off == pure Python, no FMA
 * contraction).  The AQIF kernels are therefore
 * bit-identical to the reference; this is pinned against golden vectors
 * produced by the reference itself (tests/golden/make_golden.py).
 *
 * Reference functions restated (paths relative to /root/reference/pkg/src/paqif):
 *   _cget / _cadd               _kernels.py:40-59
 *   factor_batch                _kernels.py:62-149
 *   solve_w_batch               _kernels.py:152-172
 *   solve_z_batch               _kernels.py:175-225
 *   band_matvec_batch           _kernels.py:228-241  (== bandcore.band_matvec order, bandcore.py:150-162)
 *   psor_sweeps                 _kernels.py:244-276
 *   paqif_solve (r = 1)         parallel.py:261-295 (+ partition/_block_forward/
 *                               build_reduced_system/solve_reduced/back_substitute_middle,
 *                               parallel.py:106-258; cholesky_spd_solve bandcore.py:165-186)
 *   paqif_solve_lcp (r = 1)     parallel.py:298-347
 *
 * Known, documented deviation: the reference solves the 2*beta x 2*beta
 * corner system through BLAS (R^T R) and LAPACK dpotrf/dpotrs; this oracle
 * uses textbook loops, so corner unknowns agree to rounding (~1e-16 rel),
 * not bit-for-bit.  Everything else is bit-exact.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#include <pthread.h>

#define OR_TINY 1e-300

/* ---------------------------------------------------------------- cross layout */
static inline double cget(const double *band, const double *anti, int64_t beta,
                          int64_t n, int64_t i, int64_t j)
{
    int64_t d = j - i;
    if (-beta <= d && d <= beta) return band[(d + beta) * n + i];
    int64_t c = i + j - (n - 1);
    if (-beta <= c && c <= beta) return anti[(c + beta) * n + i];
    return 0.0;
}

static inline void cadd(double *band, double *anti, int64_t beta, int64_t n,
                        int64_t i, int64_t j, double val)
{
    int64_t d = j - i;
    if (-beta <= d && d <= beta) { band[(d + beta) * n + i] += val; return; }
    int64_t c = i + j - (n - 1);
    if (-beta <= c && c <= beta) anti[(c + beta) * n + i] += val;
}

/* ---------------------------------------------------------------- factor (one system) */
static void factor_one(int64_t n, int64_t beta, double *band, double *anti,
                       double *z2x2, double *zl, double *zr, double *ww,
                       double tol, int64_t *status)
{
    const int64_t s = n / 2, bp1 = beta + 1, tb = 2 * beta;
    *status = 0;
    for (int64_t k = 1; k <= s; ++k) {
        const int64_t rt = s - k, rb = s + k - 1;
        double *zlk = zl + k * 2 * bp1, *zrk = zr + k * 2 * bp1;
        for (int64_t t = 0; t <= beta; ++t) {
            int64_t jl = rt - beta + t;
            if (jl >= 0) {
                zlk[t] = cget(band, anti, beta, n, rt, jl);
                zlk[bp1 + t] = cget(band, anti, beta, n, rb, jl);
            }
            int64_t jr = rb + t;
            if (jr < n) {
                zrk[t] = cget(band, anti, beta, n, rt, jr);
                zrk[bp1 + t] = cget(band, anti, beta, n, rb, jr);
            }
        }
        const double a11 = zlk[beta], a12 = zrk[0], a21 = zlk[bp1 + beta], a22 = zrk[bp1];
        double *zk = z2x2 + k * 4;
        zk[0] = a11; zk[1] = a12; zk[2] = a21; zk[3] = a22;
        int64_t top_lo = rt - beta > 0 ? rt - beta : 0;
        int64_t bot_hi = rb + beta < n - 1 ? rb + beta : n - 1;
        int have_wings = (top_lo <= rt - 1) || (rb + 1 <= bot_hi);
        if (!have_wings) continue;
        double det = a11 * a22 - a21 * a12;
        double scale = fabs(a11);
        if (fabs(a12) > scale) scale = fabs(a12);
        if (fabs(a21) > scale) scale = fabs(a21);
        if (fabs(a22) > scale) scale = fabs(a22);
        if (fabs(det) <= tol * (scale * scale) + OR_TINY) { *status = k; break; }
        double *wk = ww + k * tb * 2;
        for (int64_t t = 0; t < tb; ++t) {
            int64_t i;
            if (t < beta) { i = rt - beta + t; if (i < 0) continue; }
            else { i = rb + 1 + (t - beta); if (i >= n) continue; }
            double b1 = cget(band, anti, beta, n, i, rt);
            double b2 = cget(band, anti, beta, n, i, rb);
            double w1 = (a22 * b1 - a21 * b2) / det;
            double w2 = (a11 * b2 - a12 * b1) / det;
            wk[t * 2] = w1; wk[t * 2 + 1] = w2;
            if (w1 == 0.0 && w2 == 0.0) continue;
            for (int64_t u = 0; u <= beta; ++u) {
                int64_t jl = rt - beta + u;
                if (jl >= 0)
                    cadd(band, anti, beta, n, i, jl, -(w1 * zlk[u] + w2 * zlk[bp1 + u]));
                int64_t jr = rb + u;
                if (jr < n)
                    cadd(band, anti, beta, n, i, jr, -(w1 * zrk[u] + w2 * zrk[bp1 + u]));
            }
        }
    }
}

static void solve_w_one(int64_t n, int64_t beta, const double *ww, double *rhs)
{
    const int64_t s = n / 2, tb = 2 * beta;
    for (int64_t k = 1; k <= s; ++k) {
        const int64_t rt = s - k, rb = s + k - 1;
        const double yt = rhs[rt], yb = rhs[rb];
        const double *wk = ww + k * tb * 2;
        for (int64_t t = 0; t < beta; ++t) {
            int64_t i = rt - beta + t;
            if (i >= 0) rhs[i] -= yt * wk[t * 2] + yb * wk[t * 2 + 1];
            int64_t i2 = rb + 1 + t;
            if (i2 < n) rhs[i2] -= yt * wk[(beta + t) * 2] + yb * wk[(beta + t) * 2 + 1];
        }
    }
}

static void solve_z_one(int64_t n, int64_t beta, const double *z2x2, const double *zl,
                        const double *zr, const double *y, double *x, int64_t start,
                        double tol, int64_t *status, int64_t *trace)
{
    const int64_t s = n / 2, bp1 = beta + 1;
    int64_t pos = 0;
    *status = 0;
    for (int64_t level = start; level <= s; ++level) {
        const int64_t p = level - 1, q = n - 1 - p, k = s - p;
        const double *zlk = zl + k * 2 * bp1, *zrk = zr + k * 2 * bp1;
        double rt_rhs = y[p], rb_rhs = y[q];
        for (int64_t t = 0; t < beta; ++t) {
            int64_t j = p - beta + t;
            if (j >= 0) { rt_rhs -= zlk[t] * x[j]; rb_rhs -= zlk[bp1 + t] * x[j]; }
            int64_t j2 = q + 1 + t;
            if (j2 < n) { rt_rhs -= zrk[1 + t] * x[j2]; rb_rhs -= zrk[bp1 + 1 + t] * x[j2]; }
        }
        const double *zk = z2x2 + k * 4;
        const double a11 = zk[0], a12 = zk[1], a21 = zk[2], a22 = zk[3];
        double det = a11 * a22 - a12 * a21;
        double scale = fabs(a11);
        if (fabs(a12) > scale) scale = fabs(a12);
        if (fabs(a21) > scale) scale = fabs(a21);
        if (fabs(a22) > scale) scale = fabs(a22);
        if (fabs(det) <= tol * (scale * scale) + OR_TINY) { *status = level; break; }
        x[p] = (a22 * rt_rhs - a12 * rb_rhs) / det;
        x[q] = (a11 * rb_rhs - a21 * rt_rhs) / det;
        if (trace) { trace[pos] = p; trace[pos + 1] = q; }
        pos += 2;
    }
}

/* ---------------------------------------------------------------- batched exports */
void or_factor_batch(int64_t B, int64_t n, int64_t beta, double *band, double *anti,
                     double *z2x2, double *zl, double *zr, double *ww, double tol,
                     int64_t *status)
{
    const int64_t s = n / 2, nb = (2 * beta + 1) * n;
    for (int64_t b = 0; b < B; ++b)
        factor_one(n, beta, band + b * nb, anti + b * nb, z2x2 + b * (s + 1) * 4,
                   zl + b * (s + 1) * 2 * (beta + 1), zr + b * (s + 1) * 2 * (beta + 1),
                   ww + b * (s + 1) * 4 * beta, tol, status + b);
}

void or_solve_w_batch(int64_t B, int64_t n, int64_t beta, const double *ww, double *rhs)
{
    const int64_t s = n / 2;
    for (int64_t b = 0; b < B; ++b)
        solve_w_one(n, beta, ww + b * (s + 1) * 4 * beta, rhs + b * n);
}

void or_solve_z_batch(int64_t B, int64_t n, int64_t beta, const double *z2x2,
                      const double *zl, const double *zr, const double *y, double *x,
                      int64_t start, double tol, int64_t *status, int64_t *trace)
{
    const int64_t s = n / 2;
    for (int64_t b = 0; b < B; ++b)
        solve_z_one(n, beta, z2x2 + b * (s + 1) * 4, zl + b * (s + 1) * 2 * (beta + 1),
                    zr + b * (s + 1) * 2 * (beta + 1), y + b * n, x + b * n, start, tol,
                    status + b, trace ? trace + b * n : NULL);
}

static void matvec_one(int64_t n, int64_t beta, const double *bands, const double *x, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        int64_t lo = i - beta > 0 ? i - beta : 0;
        int64_t hi = i + beta + 1 < n ? i + beta + 1 : n;
        for (int64_t j = lo; j < hi; ++j) acc += bands[(j - i + beta) * n + i] * x[j];
        out[i] = acc;
    }
}

void or_band_matvec_batch(int64_t B, int64_t n, int64_t beta, const double *bands,
                          const double *x, double *out)
{
    const int64_t nb = (2 * beta + 1) * n;
    for (int64_t b = 0; b < B; ++b) matvec_one(n, beta, bands + b * nb, x + b * n, out + b * n);
}

/* psor_sweeps (_kernels.py:244-276); returns sweeps, writes last change */
int64_t or_psor_sweeps(int64_t n, int64_t beta, const double *bands, const double *f,
                       double *u, double omega, double tol, int64_t max_sweeps,
                       double *change_out)
{
    int64_t sweeps = 0;
    double change = 0.0;
    for (int64_t sweep = 0; sweep < max_sweeps; ++sweep) {
        change = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            int64_t lo = i - beta > 0 ? i - beta : 0;
            int64_t hi = i + beta + 1 < n ? i + beta + 1 : n;
            for (int64_t j = lo; j < hi; ++j)
                if (j != i) acc += bands[(j - i + beta) * n + i] * u[j];
            double diag = bands[beta * n + i];
            double unew = (1.0 - omega) * u[i] + omega * (f[i] - acc) / diag;
            if (unew < 0.0) unew = 0.0;
            double d = fabs(unew - u[i]);
            if (d > change) change = d;
            u[i] = unew;
        }
        sweeps = sweep + 1;
        if (change <= tol) break;
    }
    *change_out = change;
    return sweeps;
}

/* ---------------------------------------------------------------- r=1 paqif_solve */
/* Status codes shared with the CUDA product (include/paqif_b200.h). */
#define OR_OK 0
#define OR_FACTOR_BREAKDOWN 1
#define OR_ZSOLVE_BREAKDOWN 2
#define OR_NOT_PD 3
#define OR_NONCONVERGED 4

typedef struct {
    double *band, *anti, *z2x2, *zl, *zr, *ww, *y, *x;
    double *rd, *rtr, *rtf;
    int64_t *trace;
    /* LCP driver buffers (allocated once per worker: per-call malloc of
       >128 KB goes through mmap and serialises threads on page faults) */
    double *lmod, *fmod, *ue, *lam, *u, *lu, *best_u;
    uint8_t *active, *nact, *best_act;
} work_t;

static void work_alloc(work_t *w, int64_t n, int64_t beta)
{
    const int64_t s = n / 2, nb = (2 * beta + 1) * n, m = 2 * beta;
    w->band = malloc(sizeof(double) * nb);
    w->anti = malloc(sizeof(double) * nb);
    w->z2x2 = malloc(sizeof(double) * (s + 1) * 4);
    w->zl = malloc(sizeof(double) * (s + 1) * 2 * (beta + 1));
    w->zr = malloc(sizeof(double) * (s + 1) * 2 * (beta + 1));
    w->ww = malloc(sizeof(double) * (s + 1) * 4 * beta);
    w->y = malloc(sizeof(double) * n);
    w->x = malloc(sizeof(double) * n);
    w->rd = malloc(sizeof(double) * m * m);
    w->rtr = malloc(sizeof(double) * m * m);
    w->rtf = malloc(sizeof(double) * m);
    w->trace = NULL;
    w->lmod = malloc(sizeof(double) * nb);
    w->fmod = malloc(sizeof(double) * n);
    w->ue = malloc(sizeof(double) * n);
    w->lam = malloc(sizeof(double) * n);
    w->u = malloc(sizeof(double) * n);
    w->lu = malloc(sizeof(double) * n);
    w->best_u = malloc(sizeof(double) * n);
    w->active = malloc(n);
    w->nact = malloc(n);
    w->best_act = malloc(n);
}

static void work_free(work_t *w)
{
    free(w->band); free(w->anti); free(w->z2x2); free(w->zl); free(w->zr); free(w->ww);
    free(w->y); free(w->x); free(w->rd); free(w->rtr); free(w->rtf);
    free(w->lmod); free(w->fmod); free(w->ue); free(w->lam); free(w->u); free(w->lu);
    free(w->best_u); free(w->active); free(w->nact); free(w->best_act);
}

/* Cholesky of the SPD normal matrix (upper, A = U^T U) + two triangular
 * solves: restates cholesky_spd_solve (bandcore.py:165-186) textbook-style. */
static int chol_solve(int64_t m, double *a, double *rhs)
{
    for (int64_t j = 0; j < m; ++j) {
        double ajj = a[j * m + j];
        for (int64_t i = 0; i < j; ++i) ajj -= a[i * m + j] * a[i * m + j];
        if (!(ajj > 0.0)) return -1;
        ajj = sqrt(ajj);
        a[j * m + j] = ajj;
        for (int64_t k = j + 1; k < m; ++k) {
            double v = a[j * m + k];
            for (int64_t i = 0; i < j; ++i) v -= a[i * m + j] * a[i * m + k];
            a[j * m + k] = v / ajj;
        }
    }
    for (int64_t j = 0; j < m; ++j) {           /* U^T z = rhs */
        double v = rhs[j];
        for (int64_t i = 0; i < j; ++i) v -= a[i * m + j] * rhs[i];
        rhs[j] = v / a[j * m + j];
    }
    for (int64_t j = m - 1; j >= 0; --j) {      /* U x = z */
        double v = rhs[j];
        for (int64_t k = j + 1; k < m; ++k) v -= a[j * m + k] * rhs[k];
        rhs[j] = v / a[j * m + j];
    }
    return 0;
}

/* u = L^{-1} f through the seven-step method with a single block. */
static int paqif_solve_r1(int64_t n, int64_t beta, const double *bands, const double *f,
                          double *u, work_t *w)
{
    const int64_t s = n / 2, nb = (2 * beta + 1) * n, m = 2 * beta, bp1 = beta + 1;
    int64_t st = 0;
    memcpy(w->band, bands, sizeof(double) * nb);
    memset(w->anti, 0, sizeof(double) * nb);
    memset(w->z2x2, 0, sizeof(double) * (s + 1) * 4);
    memset(w->zl, 0, sizeof(double) * (s + 1) * 2 * bp1);
    memset(w->zr, 0, sizeof(double) * (s + 1) * 2 * bp1);
    memset(w->ww, 0, sizeof(double) * (s + 1) * 4 * beta);
    factor_one(n, beta, w->band, w->anti, w->z2x2, w->zl, w->zr, w->ww, 1e-14, &st);
    if (st) return OR_FACTOR_BREAKDOWN;
    memcpy(w->y, f, sizeof(double) * n);
    solve_w_one(n, beta, w->ww, w->y);
    /* reduced corner system: rows/cols (first beta, last beta) of Z */
    double *rd = w->rd;
    memset(rd, 0, sizeof(double) * m * m);
    for (int64_t k = s - beta + 1; k <= s; ++k) {
        const int64_t rt = s - k, rb = s + k - 1;
        const double *zlk = w->zl + k * 2 * bp1, *zrk = w->zr + k * 2 * bp1;
        for (int64_t t = 0; t <= beta; ++t) {
            int64_t jl = rt - beta + t, jr = rb + t;
            if (jl >= 0) {           /* column jl < beta -> reduced col jl */
                rd[rt * m + jl] = zlk[t];
                rd[(beta + (rb - (n - beta))) * m + jl] = zlk[bp1 + t];
            }
            if (jr < n) {            /* column jr >= n-beta -> reduced col beta + jr-(n-beta) */
                rd[rt * m + beta + (jr - (n - beta))] = zrk[t];
                rd[(beta + (rb - (n - beta))) * m + beta + (jr - (n - beta))] = zrk[bp1 + t];
            }
        }
    }
    double fd[64];
    for (int64_t i = 0; i < beta; ++i) { fd[i] = w->y[i]; fd[beta + i] = w->y[n - beta + i]; }
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < m; ++j) {
            double acc = 0.0;
            for (int64_t r = 0; r < m; ++r) acc += rd[r * m + i] * rd[r * m + j];
            w->rtr[i * m + j] = acc;
        }
    for (int64_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int64_t r = 0; r < m; ++r) acc += rd[r * m + i] * fd[r];
        w->rtf[i] = acc;
    }
    if (chol_solve(m, w->rtr, w->rtf)) return OR_NOT_PD;
    memset(w->x, 0, sizeof(double) * n);
    for (int64_t i = 0; i < beta; ++i) { w->x[i] = w->rtf[i]; w->x[n - beta + i] = w->rtf[beta + i]; }
    solve_z_one(n, beta, w->z2x2, w->zl, w->zr, w->y, w->x, beta + 1, 1e-14, &st, NULL);
    if (st) return OR_ZSOLVE_BREAKDOWN;
    memcpy(u, w->x, sizeof(double) * n);
    return OR_OK;
}

int or_paqif_solve_r1(int64_t n, int64_t beta, const double *bands, const double *f, double *u)
{
    work_t w;
    work_alloc(&w, n, beta);
    int rc = paqif_solve_r1(n, beta, bands, f, u, &w);
    work_free(&w);
    return rc;
}

/* ---------------------------------------------------------------- LCP driver */
static int lcp_one(int64_t n, int64_t beta, const double *bands, const double *f,
                   double tol, int64_t max_outer, double *u_out, uint8_t *active_out,
                   int64_t *passes_out, double *res_out, work_t *w)
{
    const int64_t nb = (2 * beta + 1) * n;
    double *lmod = w->lmod, *fmod = w->fmod, *ue = w->ue, *lam = w->lam, *u = w->u, *lu = w->lu;
    double *best_u = w->best_u;
    uint8_t *active = w->active, *nact = w->nact, *best_act = w->best_act;
    memset(best_u, 0, sizeof(double) * n);
    int rc = OR_NONCONVERGED;
    int64_t passes = 0;
    double res = INFINITY, best_res = INFINITY;
    for (int64_t i = 0; i < n; ++i) active[i] = (f[i] <= 0.0);
    memcpy(best_act, active, n);
    /* scale = max_i sum_d |bands[d,i]| + max|f| (parallel.py:317) */
    double scale = 0.0, fmax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double c = 0.0;
        for (int64_t d = 0; d <= 2 * beta; ++d) c += fabs(bands[d * n + i]);
        if (c > scale) scale = c;
        if (fabs(f[i]) > fmax) fmax = fabs(f[i]);
    }
    scale += fmax;
    const double floor_ = 1e3 * DBL_EPSILON * scale;
    const double lim = tol > floor_ ? tol : floor_;
    for (int64_t outer = 0; outer < max_outer; ++outer) {
        memcpy(lmod, bands, sizeof(double) * nb);
        for (int64_t i = 0; i < n; ++i) {
            fmod[i] = active[i] ? 0.0 : f[i];
            if (active[i]) {
                double dg = bands[beta * n + i];
                for (int64_t d = 0; d <= 2 * beta; ++d) lmod[d * n + i] = 0.0;
                lmod[beta * n + i] = fabs(dg) > 0.0 ? dg : 1.0;
            }
        }
        passes = outer + 1;
        int st = paqif_solve_r1(n, beta, lmod, fmod, ue, w);
        if (st) { rc = st; goto done; }
        matvec_one(n, beta, bands, ue, lam);
        for (int64_t i = 0; i < n; ++i) {
            lam[i] -= f[i];
            /* np.maximum(x, 0.0): (x >= 0 || isnan(x)) ? x : 0.0 (keeps -0.0) */
            u[i] = (ue[i] >= 0.0 || ue[i] != ue[i]) ? ue[i] : 0.0;
        }
        matvec_one(n, beta, bands, u, lu);
        res = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double r = lu[i] - f[i];
            /* np.minimum(a, b): (a <= b || isnan(a)) ? a : b (NaN propagates) */
            double mn = (u[i] <= r || u[i] != u[i]) ? u[i] : r;
            double a = fabs(mn);
            if (a > res || a != a) res = a;
        }
        if (res <= tol) {
            memcpy(u_out, u, sizeof(double) * n);
            memcpy(active_out, active, n);
            rc = OR_OK; goto done;
        }
        if (res < best_res) {
            best_res = res; memcpy(best_u, u, sizeof(double) * n); memcpy(best_act, active, n);
        }
        int same = 1;
        for (int64_t i = 0; i < n; ++i) {
            nact[i] = ue[i] < lam[i];
            if (nact[i] != active[i]) same = 0;
        }
        if (same) break;
        memcpy(active, nact, n);
    }
    if (best_res <= lim) {
        memcpy(u_out, best_u, sizeof(double) * n);
        memcpy(active_out, best_act, n);
        res = best_res;
        rc = OR_OK;
    } else {
        rc = OR_NONCONVERGED;
        memcpy(u_out, best_u, sizeof(double) * n);
        memcpy(active_out, best_act, n);
    }
done:
    *passes_out = passes;
    *res_out = res;
    return rc;
}

typedef struct {
    int64_t B, n, beta, max_outer, next;
    const double *bands, *f;
    double tol, *u, *res;
    uint8_t *active;
    int64_t *passes, *status;
    pthread_mutex_t *mu;
} lcp_job_t;

static void *lcp_worker(void *arg)
{
    lcp_job_t *J = arg;
    work_t w;
    work_alloc(&w, J->n, J->beta);
    const int64_t nb = (2 * J->beta + 1) * J->n;
    for (;;) {
        pthread_mutex_lock(J->mu);
        int64_t b = J->next++;
        pthread_mutex_unlock(J->mu);
        if (b >= J->B) break;
        J->status[b] = lcp_one(J->n, J->beta, J->bands + b * nb, J->f + b * J->n, J->tol,
                               J->max_outer, J->u + b * J->n, J->active + b * J->n,
                               J->passes + b, J->res + b, &w);
    }
    work_free(&w);
    return NULL;
}

/* Batched paqif_solve_lcp(LcpProblem(L_b, f_b), r=1) over `threads` host threads. */
void or_lcp_batch(int64_t B, int64_t n, int64_t beta, const double *bands, const double *f,
                  double tol, int64_t max_outer, double *u, uint8_t *active,
                  int64_t *passes, double *res, int64_t *status, int64_t threads)
{
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    lcp_job_t J = {B, n, beta, max_outer, 0, bands, f, tol, u, res, active, passes, status, &mu};
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t tid[512];
    for (int64_t t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, lcp_worker, &J);
    for (int64_t t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* Raw single-pass factor+W+Z over a batch (the reference's _kernels pass), threaded. */
typedef struct {
    int64_t B, n, beta, next;
    const double *bands, *f;
    double *x;
    int64_t *status;
    pthread_mutex_t *mu;
} pass_job_t;

static void *pass_worker(void *arg)
{
    pass_job_t *J = arg;
    work_t w;
    work_alloc(&w, J->n, J->beta);
    const int64_t nb = (2 * J->beta + 1) * J->n;
    for (;;) {
        pthread_mutex_lock(J->mu);
        int64_t b = J->next++;
        pthread_mutex_unlock(J->mu);
        if (b >= J->B) break;
        J->status[b] = paqif_solve_r1(J->n, J->beta, J->bands + b * nb, J->f + b * J->n,
                                      J->x + b * J->n, &w);
    }
    work_free(&w);
    return NULL;
}

void or_paqif_solve_r1_batch(int64_t B, int64_t n, int64_t beta, const double *bands,
                             const double *f, double *x, int64_t *status, int64_t threads)
{
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    pass_job_t J = {B, n, beta, 0, bands, f, x, status, &mu};
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t tid[512];
    for (int64_t t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, pass_worker, &J);
    for (int64_t t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}
