/*
 * The normalized associated Legendre degree recurrence, one step, shared by
 * the host table builder (recur.c), the packer's seed computation
 * (packer.cpp) and the GPU tile regeneration (engine.cu).
 *
 * Operation sequence of the reference kernel
 * (pkg/src/bfsht/kernels/_recur_cy.pyx:45-66):
 *     p_next = alpha[s] * (x * p_cur) - beta[s] * p_prev
 * with a (mantissa, 2^e) pair rescaled by exact powers of two when
 * max(|p_cur|, |p_prev|) leaves [2^-500, 2^500].  No FMA contraction
 * anywhere (host: -ffp-contract=off; device: __dmul_rn/__dsub_rn), and the
 * 2^-+1000 rescales are exact, so host and device produce the same bits.
 */
#ifndef BFSHT_RECUR_H
#define BFSHT_RECUR_H
#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define BFR_HD __host__ __device__ __forceinline__
#ifdef __CUDA_ARCH__
#define BFR_MUL(a, b) __dmul_rn((a), (b))
#define BFR_SUB(a, b) __dsub_rn((a), (b))
#else
#define BFR_MUL(a, b) ((a) * (b))
#define BFR_SUB(a, b) ((a) - (b))
#endif
#else
#define BFR_HD static inline
#define BFR_MUL(a, b) ((a) * (b))
#define BFR_SUB(a, b) ((a) - (b))
#endif

#define BFR_BIG 0x1p500
#define BFR_SMALL 0x1p-500
#define BFR_RESCALE 1000

BFR_HD void bfr_step(double xr, double a, double b, double *p_prev, double *p_cur, int *e) {
    const double t1 = BFR_MUL(xr, *p_cur);
    const double t2 = BFR_MUL(a, t1);
    const double t3 = BFR_MUL(b, *p_prev);
    const double p_next = BFR_SUB(t2, t3);
    *p_prev = *p_cur;
    *p_cur = p_next;
    const double aa = fabs(*p_cur), bb = fabs(*p_prev);
    const double mx = aa > bb ? aa : bb;
    if (mx > BFR_BIG) {
        *p_cur = BFR_MUL(*p_cur, 0x1p-1000);
        *p_prev = BFR_MUL(*p_prev, 0x1p-1000);
        *e += BFR_RESCALE;
    } else if (mx < BFR_SMALL && mx > 0.0) {
        *p_cur = BFR_MUL(*p_cur, 0x1p1000);
        *p_prev = BFR_MUL(*p_prev, 0x1p1000);
        *e -= BFR_RESCALE;
    }
}

/* alpha_s, beta_s for k = m + s, exact integer products then one correctly
 * rounded division and square root (kernels/common.py:37-53). */
BFR_HD void bfr_coeffs(int64_t m, int64_t k, double *alpha, double *beta) {
    const double kd = (double)k, md = (double)m;
    const double den = (kd + 1.0 - md) * (kd + 1.0 + md);
    *alpha = sqrt((2.0 * kd + 1.0) * (2.0 * kd + 3.0) / den);
    if (k == m) {
        *beta = 0.0;
    } else {
        const double num_b = (2.0 * kd + 3.0) * (kd - md) * (kd + md);
        *beta = sqrt(num_b / ((2.0 * kd - 1.0) * den));
    }
}

#endif
