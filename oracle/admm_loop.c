/*
 * ORACLE — Algorithm 1 of arXiv 2310.09410, plain C, one thread.
 * TEST INFRASTRUCTURE ONLY: called from oracle/admm.py (ctypes) by tests/, smoke()
 * and bench.py's cpu_baseline leg.  Shares nothing with paper_2310_09410_b200/.
 * Built with: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction, IEEE
 * round-to-nearest-even, fixed summation orders as stated below).  The `omp` pragmas are inert in that
 * (parity) build; the same file built with -fopenmp is the multi-core CPU baseline of bench.py (SURVEY
 * §8(d) mode (ii)): each loop split statically over the host cores, residual sums by an OpenMP
 * reduction (summation order then differs, so that build is for timing only, never for parity).
 *
 * Data (all in canonical order, DESIGN.md §3 C12):
 *   n globals: c, lo, hi                      (LP_model)
 *   nc copies: copy_global[k] = global of copy k (B_s as index lists)
 *   seg_ptr[n+1], seg_copy[nc]: copies of global i ascending (I_si)
 *   S subsystems: sub_ptr[S+1] copy offsets; abar_ptr[S+1] offsets of the dense
 *   row-major n_s x n_s Abar_s; bbar[nc] (closed_2)
 * State: x[n], xl[nc] = x_s concatenated, lam[nc] = lambda_s concatenated.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

typedef struct {
    int64_t n, S, nc;
    const double *c, *lo, *hi;
    const int64_t *seg_ptr;
    const int32_t *seg_copy;
    const int32_t *copy_global;
    const int64_t *sub_ptr;
    const int64_t *abar_ptr;
    const double *abar, *bbar;
    double rho, eps_rel;
} oracle_problem;

/* Global update, closed_1 with the rho restored (reading C1):
 *   x_i = min(max(xhat_i, lo_i), hi_i),
 *   xhat_i = (rho * sum_k x_k - (c_i + sum_k lam_k)) / (rho nu_i)
 *          = (sum_k (x_k - lam_k/rho) - c_i/rho) / nu_i,   k over seg(i) ascending. */
void oracle_global_update(const oracle_problem *p, const double *xl, const double *lam, double *x)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < p->n; ++i) {
        double sigma = 0.0;
        int64_t nu = p->seg_ptr[i + 1] - p->seg_ptr[i];
        for (int64_t q = p->seg_ptr[i]; q < p->seg_ptr[i + 1]; ++q) {
            int32_t k = p->seg_copy[q];
            sigma += xl[k] - lam[k] / p->rho;
        }
        double xhat = (sigma - p->c[i] / p->rho) / (double)nu;
        x[i] = fmin(fmax(xhat, p->lo[i]), p->hi[i]);   /* IEEE +-inf bounds = no clamp (C8) */
    }
}

/* Local update, closed_2: for each s,
 *   v = B_s x,  d = -rho v - lam_s,  x_s[r] = (sum_k Abar[r][k] d[k]) / rho + bbar[r]  (k ascending). */
void oracle_local_update(const oracle_problem *p, const double *x, const double *lam, double *xl_new)
{
#pragma omp parallel
    {
    double *d = NULL;
    int64_t dcap = 0;
#pragma omp for schedule(static)
    for (int64_t s = 0; s < p->S; ++s) {
        int64_t o = p->sub_ptr[s], ns = p->sub_ptr[s + 1] - o;
        if (ns > dcap) { free(d); dcap = ns; d = (double *)malloc(sizeof(double) * (size_t)dcap); }
        for (int64_t k = 0; k < ns; ++k) {
            double v = x[p->copy_global[o + k]];
            d[k] = -p->rho * v - lam[o + k];
        }
        const double *Ab = p->abar + p->abar_ptr[s];
        for (int64_t r = 0; r < ns; ++r) {
            double acc = 0.0;
            for (int64_t k = 0; k < ns; ++k) acc += Ab[r * ns + k] * d[k];
            xl_new[o + r] = acc / p->rho + p->bbar[o + r];
        }
    }
    free(d);
    }
}

/* Dual update ADMM-3: lam_s += rho (B_s x - x_s). */
void oracle_dual_update(const oracle_problem *p, const double *x, const double *xl, double *lam)
{
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < p->nc; ++k) {
        double v = x[p->copy_global[k]];
        lam[k] = lam[k] + p->rho * (v - xl[k]);
    }
}

/* Residuals of (termination), readings C3/C4 (B_s^T is an isometry):
 *   pres = sqrt(sum (v - x_s)^2), dres = rho sqrt(sum (x_s - x_s_old)^2),
 *   eps_prim = eps_rel max(sqrt(sum v^2), sqrt(sum x_s^2)), eps_dual = eps_rel sqrt(sum lam^2);
 * all sums sequential over copies in ascending order. out = {pres, dres, eps_prim, eps_dual}. */
void oracle_residuals(const oracle_problem *p, const double *x, const double *xl, const double *xl_old,
                      const double *lam, double *out)
{
    double sp = 0.0, sd = 0.0, sv = 0.0, sx = 0.0, sl = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : sp, sd, sv, sx, sl)
    for (int64_t k = 0; k < p->nc; ++k) {
        double v = x[p->copy_global[k]];
        double r = v - xl[k];
        double dx = xl[k] - xl_old[k];
        sp += r * r;
        sd += dx * dx;
        sv += v * v;
        sx += xl[k] * xl[k];
        sl += lam[k] * lam[k];
    }
    out[0] = sqrt(sp);
    out[1] = p->rho * sqrt(sd);
    out[2] = p->eps_rel * fmax(sqrt(sv), sqrt(sx));
    out[3] = p->eps_rel * sqrt(sl);
}

/* Algorithm 1 loop: while not (termination): global; local; dual.
 * The test is applied after every full sweep on that sweep's x, x_s, lambda and the previous
 * x_s (reading C5); K = number of sweeps executed.  test = 0 runs exactly max_iter sweeps.
 * trace (optional, may be NULL): rows of {pres, dres, eps_prim, eps_dual} every trace_every sweeps.
 * Returns K; res receives the last residuals; converged = 1 iff the test fired. */
int64_t oracle_run(const oracle_problem *p, double *x, double *xl, double *lam, int64_t max_iter,
                   int32_t test, double *res, int32_t *converged, double *trace, int64_t trace_cap,
                   int32_t trace_every, int64_t *trace_rows)
{
    double *xl_old = (double *)malloc(sizeof(double) * (size_t)(p->nc > 0 ? p->nc : 1));
    int64_t t = 0, nrow = 0;
    *converged = 0;
    res[0] = res[1] = res[2] = res[3] = 0.0;
    while (t < max_iter) {
        memcpy(xl_old, xl, sizeof(double) * (size_t)p->nc);
        oracle_global_update(p, xl, lam, x);          /* line 5 */
        oracle_local_update(p, x, lam, xl);           /* line 7 */
        oracle_dual_update(p, x, xl, lam);            /* line 8 */
        ++t;
        oracle_residuals(p, x, xl, xl_old, lam, res);
        if (trace && trace_every > 0 && (t % trace_every) == 0 && nrow < trace_cap) {
            memcpy(trace + 4 * nrow, res, 4 * sizeof(double));
            ++nrow;
        }
        if (test && res[0] <= res[2] && res[1] <= res[3]) { *converged = 1; break; }
    }
    if (trace_rows) *trace_rows = nrow;
    free(xl_old);
    return t;
}

/* ---- residual balancing ("residual balancing [wohlberg2017admm]") ----------
 * Algorithm 1 with the penalty adapted by the residual-balancing rule of Boyd et al. (2011) §3.4.1 /
 * Wohlberg (2017): after the test of sweep t has failed, and if t is a multiple of `every`,
 *     rho <- tau rho   if pres > mu dres,      rho <- rho / tau   if dres > mu pres,
 * and rho is unchanged otherwise.  lambda is the unscaled multiplier, so nothing else is
 * rescaled, and Abar_s, bbar_s contain no rho: only the scalar changes.  Sweep t uses
 * the rho in force when it starts everywhere (u = x_s - lambda/rho and c/rho of closed_1, d = -rho v -
 * lambda and the 1/rho of closed_2, ADMM-3, and dres = rho ||x_s - x_s_old||).  rho_out: the final rho. */
int64_t oracle_run_adaptive(const oracle_problem *p, double *x, double *xl, double *lam, int64_t max_iter,
                            int32_t test, double *res, int32_t *converged, int32_t every, double mu, double tau,
                            double *rho_out, int64_t *n_changes)
{
    double *xl_old = (double *)malloc(sizeof(double) * (size_t)(p->nc > 0 ? p->nc : 1));
    oracle_problem q = *p;
    int64_t t = 0, nch = 0;
    *converged = 0;
    res[0] = res[1] = res[2] = res[3] = 0.0;
    while (t < max_iter) {
        memcpy(xl_old, xl, sizeof(double) * (size_t)p->nc);
        oracle_global_update(&q, xl, lam, x);
        oracle_local_update(&q, x, lam, xl);
        oracle_dual_update(&q, x, xl, lam);
        ++t;
        oracle_residuals(&q, x, xl, xl_old, lam, res);
        if (test && res[0] <= res[2] && res[1] <= res[3]) { *converged = 1; break; }
        if (every > 0 && (t % every) == 0) {
            if (res[0] > mu * res[1]) { q.rho = tau * q.rho; ++nch; }
            else if (res[1] > mu * res[0]) { q.rho = q.rho / tau; ++nch; }
        }
    }
    *rho_out = q.rho;
    *n_changes = nch;
    free(xl_old);
    return t;
}

/* ---- fp32 variant (the paper's GPU precision; reading F1) --------
 * The same Algorithm 1 with every datum of the iteration in binary32: Abar_s, bbar_s, c, lo, hi, rho
 * and the initial point are the fp64 values rounded once to nearest (IEEE +-inf stays +-inf), and every
 * operation of closed_1, closed_2 and ADMM-3 is a binary32 operation in the order written above.  The
 * five residual terms are formed in binary32 and summed in binary64 (sequentially, ascending copy), and
 * the test of (termination) is evaluated in binary64 from those sums — the paper does not say how its
 * fp32 norms are reduced; an fp64 sum keeps the decision independent of the summation order. */
typedef struct {
    int64_t n, S, nc;
    const float *c, *lo, *hi;
    const int64_t *seg_ptr;
    const int32_t *seg_copy;
    const int32_t *copy_global;
    const int64_t *sub_ptr;
    const int64_t *abar_ptr;
    const float *abar, *bbar;
    float rho;
    double rho64, eps_rel;
} oracle_problem_f32;

int64_t oracle_run_f32(const oracle_problem_f32 *p, float *x, float *xl, float *lam, int64_t max_iter,
                       int32_t test, double *res, int32_t *converged)
{
    float *xl_old = (float *)malloc(sizeof(float) * (size_t)(p->nc > 0 ? p->nc : 1));
    float *d = NULL;
    int64_t dcap = 0, t = 0;
    *converged = 0;
    res[0] = res[1] = res[2] = res[3] = 0.0;
    while (t < max_iter) {
        memcpy(xl_old, xl, sizeof(float) * (size_t)p->nc);
        /* line 5: closed_1 with rho restored (C1) */
        for (int64_t i = 0; i < p->n; ++i) {
            float sigma = 0.0f;
            int64_t nu = p->seg_ptr[i + 1] - p->seg_ptr[i];
            for (int64_t q = p->seg_ptr[i]; q < p->seg_ptr[i + 1]; ++q) {
                int32_t k = p->seg_copy[q];
                sigma += xl[k] - lam[k] / p->rho;
            }
            float xhat = (sigma - p->c[i] / p->rho) / (float)nu;
            x[i] = fminf(fmaxf(xhat, p->lo[i]), p->hi[i]);
        }
        /* line 7: closed_2 */
        for (int64_t s = 0; s < p->S; ++s) {
            int64_t o = p->sub_ptr[s], ns = p->sub_ptr[s + 1] - o;
            if (ns > dcap) { free(d); dcap = ns; d = (float *)malloc(sizeof(float) * (size_t)dcap); }
            for (int64_t k = 0; k < ns; ++k) d[k] = -p->rho * x[p->copy_global[o + k]] - lam[o + k];
            const float *Ab = p->abar + p->abar_ptr[s];
            for (int64_t r = 0; r < ns; ++r) {
                float acc = 0.0f;
                for (int64_t k = 0; k < ns; ++k) acc += Ab[r * ns + k] * d[k];
                xl[o + r] = acc / p->rho + p->bbar[o + r];
            }
        }
        /* line 8: ADMM-3 */
        for (int64_t k = 0; k < p->nc; ++k) lam[k] = lam[k] + p->rho * (x[p->copy_global[k]] - xl[k]);
        ++t;
        /* (termination): binary32 terms, binary64 sums */
        double sp = 0.0, sd = 0.0, sv = 0.0, sx = 0.0, sl = 0.0;
        for (int64_t k = 0; k < p->nc; ++k) {
            float v = x[p->copy_global[k]];
            float r = v - xl[k], dx = xl[k] - xl_old[k];
            sp += (double)(r * r);
            sd += (double)(dx * dx);
            sv += (double)(v * v);
            sx += (double)(xl[k] * xl[k]);
            sl += (double)(lam[k] * lam[k]);
        }
        res[0] = sqrt(sp);
        res[1] = p->rho64 * sqrt(sd);
        res[2] = p->eps_rel * fmax(sqrt(sv), sqrt(sx));
        res[3] = p->eps_rel * sqrt(sl);
        if (test && res[0] <= res[2] && res[1] <= res[3]) { *converged = 1; break; }
    }
    free(d);
    free(xl_old);
    return t;
}
