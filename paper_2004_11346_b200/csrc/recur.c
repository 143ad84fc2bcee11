/*
 * Host-side normalized associated Legendre recurrence (plan time only).
 *
 * Produces one parity half of an order-m ALT matrix as a dense table,
 * entry (r, j) = Pbar_{m + offset + 2j}^m(x[r]).  The per-point operation
 * sequence is the reference kernel's (pkg/src/bfsht/kernels/_recur_cy.pyx:
 * 18-67 and its numpy twin _recur_np.py:12-51): the scaled three-term step
 * p_next = alpha[s]*(x*p_cur) - beta[s]*p_prev, a (mantissa, 2^exp) pair
 * rescaled by exact powers of two whenever max(|p_cur|,|p_prev|) leaves
 * [2^-500, 2^500], and emission ldexp(p, e) flushed to 0 below MAG_MIN.
 * Compiled with -ffp-contract=off so no FMA contraction changes a bit; the
 * values therefore equal the reference entry oracle's bitwise, which is what
 * makes the plans built from them identical to the reference planner's.
 *
 * Evaluating a whole half table once per (m, parity) replaces the
 * reference's checkpointed per-block re-evaluation
 * (pkg/src/bfsht/partition.py:91-169); resumed evaluation there is bitwise
 * equal to seeded evaluation, so the table entries are the same numbers.
 */
#include <math.h>
#include <stdint.h>

#include "recur.h"

static inline double emit(double p_cur, int e, double mag_min) {
    double v = ldexp(p_cur, e);
    return fabs(v) < mag_min ? 0.0 : v;
}

/* out is row-major n x ncols; degrees m + offset + 2j, j < ncols. */
int bfsht_legendre_half_table(int64_t m, int64_t offset, int64_t n,
                              int64_t ncols, const double *x,
                              const double *alpha, const double *beta,
                              const double *mant0, const int32_t *exp0,
                              double mag_min, double *out)
{
    if (n <= 0 || ncols <= 0) return 0;
    const int64_t k_first = m + offset;
    const int64_t k_last = m + offset + 2 * (ncols - 1);
    for (int64_t r = 0; r < n; ++r) {
        const double xr = x[r];
        double p_prev = 0.0, p_cur = mant0[r];
        int e = exp0[r];
        double *row = out + r * ncols;
        int64_t j = 0;
        if (k_first == m) {
            row[j++] = emit(p_cur, e, mag_min);
        }
        for (int64_t k = m; k < k_last; ++k) {
            const int64_t s = k - m;
            bfr_step(xr, alpha[s], beta[s], &p_prev, &p_cur, &e);
            if (j < ncols && k + 1 == k_first + 2 * j) {
                row[j++] = emit(p_cur, e, mag_min);
            }
        }
    }
    return 0;
}

/* Arbitrary ascending degree list for a set of points (dense references). */
int bfsht_legendre_table(int64_t m, int64_t npts, const double *x,
                         int64_t ndeg, const int64_t *degrees,
                         const double *alpha, const double *beta,
                         const double *mant0, const int32_t *exp0,
                         double mag_min, double *out)
{
    if (npts <= 0 || ndeg <= 0) return 0;
    const int64_t k_stop = degrees[ndeg - 1];
    for (int64_t r = 0; r < npts; ++r) {
        const double xr = x[r];
        double p_prev = 0.0, p_cur = mant0[r];
        int e = exp0[r];
        double *row = out + r * ndeg;
        int64_t d = 0;
        if (degrees[0] == m) {
            row[d++] = emit(p_cur, e, mag_min);
        }
        for (int64_t k = m; k < k_stop; ++k) {
            const int64_t s = k - m;
            bfr_step(xr, alpha[s], beta[s], &p_prev, &p_cur, &e);
            if (d < ndeg && degrees[d] == k + 1) {
                row[d++] = emit(p_cur, e, mag_min);
            }
        }
    }
    return 0;
}
