// SHT stages around the ALT engine: coefficient packing, the phi-direction
// DFT of odd length L = 4N-1 fused with parity assembly / quadrature fold,
// and the per-order ALT boundary kernels.
//
// Reference: sht_forward / sht_inverse (pkg/src/bfsht/sht.py:137-166) —
// per-order alt_forward, phase exp(i m phi0), bin m mod L, L*ifft per
// colatitude row; and the reverse with fft/L — plus the parity assembly
// out[n:] = g_e + g_o, out[n-1::-1] = g_e - g_o (alt.py:225-236) and the
// weighted fold (alt.py:239-253).
//
// DFT: in-place mixed-radix decimation-in-time in shared memory, input
// loaded in digit-reversed order (host-built permutation), twiddles from a
// host-built exp(-2 pi i k/L) table.  A CTA owns the two rows n+r and
// n-1-r, so the parity assembly (forward) and the +/- fold (inverse) happen
// in the same kernel that does the DFT: the ALT node halves are read or
// written exactly once, as 32-byte sectors.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <complex>
#include <vector>

#include <cooperative_groups.h>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kMaxRadix = 24;
#ifndef BF_DFT_THREADS
#define BF_DFT_THREADS 256
#endif
constexpr int kDftThreads = BF_DFT_THREADS;
#ifndef BF_DFT_MINBLOCKS
#define BF_DFT_MINBLOCKS 2
#endif
// The row-pair kernels with the row in shared memory (N <= 1024: 64 KB rows)
// run three CTAs of 128 threads per SM: measured at N=1024 against two CTAs
// of 256 threads, synthesis 0.162 -> 0.152 ms, analysis 0.191 -> 0.171 ms
// (more rows in flight hide the global load / store phases; 160 x 3 gave
// 0.149 / 0.185, 192 x 3 and 224 x 3 spill and are slower).  The L2-scratch
// kernels keep 256 x 2 (128 x 3 there: N=4096 10.5 / 9.4 vs 9.3 / 8.5 ms).
#ifndef BF_PAIR_THREADS
#define BF_PAIR_THREADS 128
#endif
#ifndef BF_PAIR_MINBLOCKS
#define BF_PAIR_MINBLOCKS 3
#endif
constexpr int kPairThreads = BF_PAIR_THREADS;
// shared-memory ceiling of a one-row CTA: two CTAs per SM (228 KB per SM,
// 1 KB reserved per CTA)
constexpr int kPairSmemMax = 113 * 1024;

struct DftDesc {
    int L;       // transform length
    int Lb;      // row buffer length: L, or the Bluestein convolution length M
    int blue;    // 1: Bluestein (chirp-z) rows of length M >= 2L-1
    int nrad;
    int radix[kMaxRadix];
    // per pass: exact multiplicative inverse of the pass's span (the product
    // of the earlier radices), x / span == __umulhi(x, span_inv) for every
    // butterfly index x < L (checked on the host when the table is built)
    unsigned span_inv[kMaxRadix];
    // per pass: offset of its twiddle block in the pass table (entries
    // (q-1) * span + k, contiguous in the butterfly index k, so a warp's
    // twiddle loads are consecutive) and of its P radix roots
    int tw_off[kMaxRadix];
    int root_off[kMaxRadix];
    int span[kMaxRadix];
};

__device__ __forceinline__ int fast_div(int x, unsigned inv) {
    return inv ? (int)__umulhi((unsigned)x, inv) : x;   // inv 0: span 1
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 conjif(double2 a, bool c) {
    return c ? make_double2(a.x, -a.y) : a;
}

// One radix-P pass over all butterflies of `nrows` rows (whole CTA).
// Radix roots are loaded once per pass into registers; the inter-pass
// twiddles come from the pass table Tw (entry (q-1)*span + k = W^{q k L/(span P)},
// the value the flat root table held at q*k*tstep), which keeps a warp's
// twiddle loads on consecutive addresses (no shared-memory bank
// conflicts); the first pass (span 1) has only unit twiddles and skips
// them.  Odd P uses the conjugate-pair form: with a_j = x_j + x_{P-j},
// b_j = x_j - x_{P-j},
//   y_s, y_{P-s} = x_0 + sum_j a_j cos(2 pi js/P)  +/-  i sum_j b_j sin(..)
// (signs per direction), about a quarter of the P^2 complex products of a
// naive size-P DFT.
//
// DIF = false: decimation in time (twiddle the inputs, then the butterfly;
// passes in radix order, input digit-reversed, output natural).  DIF =
// true: the transposed pass (butterfly, then twiddle the outputs; passes
// in reverse order, input natural, output digit-reversed) — the DFT matrix
// is symmetric, so the transposed pass sequence computes the same DFT.
// Bluestein rows use both (see row_dft).
template <int P, bool DIF = false>
__device__ __forceinline__ void radix_pass(double2 *buf, int nrows, int L, int span,
                                           unsigned span_inv, const double2 *Tw,
                                           const double2 *__restrict__ R, bool inv) {
    double cr[P], ci[P];
#pragma unroll
    for (int t = 0; t < P; ++t) {
        const double2 w = R[t];
        cr[t] = w.x;
        ci[t] = inv ? -w.y : w.y;
    }
    const int nb = L / P;
    for (int t = threadIdx.x; t < nb * nrows; t += blockDim.x) {
        // nrows <= 2: the row by one compare, the group by a multiply-high
        const int rw = t >= nb ? 1 : 0, tt = t - rw * nb;
        const int g = fast_div(tt, span_inv), k = tt - g * span;
        double2 *row = buf + (int64_t)rw * L;
        const int base = g * span * P + k;
        double2 x[P];
#pragma unroll
        for (int q = 0; q < P; ++q) x[q] = row[base + q * span];
        if (!DIF && span > 1) {
            // w^q as powers of the one loaded w (table entry q = 1): one
            // twiddle load per butterfly instead of P - 1 (the passes are
            // L1-bound); <= P - 2 extra roundings, ~1e-15 relative
            const double2 w1 = conjif(Tw[k], inv);
            double2 w = w1;
            x[1] = cmul(x[1], w);
#pragma unroll
            for (int q = 2; q < P; ++q) {
                w = cmul(w, w1);
                x[q] = cmul(x[q], w);
            }
        }
        double2 y[P];
        if (P == 2) {
            y[0] = make_double2(x[0].x + x[1].x, x[0].y + x[1].y);
            y[1] = make_double2(x[0].x - x[1].x, x[0].y - x[1].y);
        } else if (P == 4) {
            // W = -i (forward) / +i (inverse)
            const double2 s02 = make_double2(x[0].x + x[2].x, x[0].y + x[2].y);
            const double2 d02 = make_double2(x[0].x - x[2].x, x[0].y - x[2].y);
            const double2 s13 = make_double2(x[1].x + x[3].x, x[1].y + x[3].y);
            const double2 d13 = make_double2(x[1].x - x[3].x, x[1].y - x[3].y);
            // -i * d13 = (d13.y, -d13.x)
            const double2 r = inv ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
            y[0] = make_double2(s02.x + s13.x, s02.y + s13.y);
            y[2] = make_double2(s02.x - s13.x, s02.y - s13.y);
            y[1] = make_double2(d02.x + r.x, d02.y + r.y);
            y[3] = make_double2(d02.x - r.x, d02.y - r.y);
        } else {
            constexpr int H = (P - 1) / 2;
            double2 a[H + 1], bb[H + 1];
            double2 y0 = x[0];
#pragma unroll
            for (int j = 1; j <= H; ++j) {
                a[j] = make_double2(x[j].x + x[P - j].x, x[j].y + x[P - j].y);
                bb[j] = make_double2(x[j].x - x[P - j].x, x[j].y - x[P - j].y);
                y0.x += a[j].x;
                y0.y += a[j].y;
            }
            y[0] = y0;
#pragma unroll
            for (int sidx = 1; sidx <= H; ++sidx) {
                double2 re = x[0], im = make_double2(0.0, 0.0);
#pragma unroll
                for (int j = 1; j <= H; ++j) {
                    const int t = (j * sidx) % P;
                    re.x = fma(a[j].x, cr[t], re.x);
                    re.y = fma(a[j].y, cr[t], re.y);
                    im.x = fma(bb[j].x, ci[t], im.x);
                    im.y = fma(bb[j].y, ci[t], im.y);
                }
                // x_j w^{js} + x_{P-j} w^{-js} = a_j cr + i ci b_j
                y[sidx] = make_double2(re.x - im.y, re.y + im.x);
                y[P - sidx] = make_double2(re.x + im.y, re.y - im.x);
            }
        }
        if (DIF && span > 1) {
            const double2 w1 = conjif(Tw[k], inv);
            double2 w = w1;
            y[1] = cmul(y[1], w);
#pragma unroll
            for (int q = 2; q < P; ++q) {
                w = cmul(w, w1);
                y[q] = cmul(y[q], w);
            }
        }
#pragma unroll
        for (int q = 0; q < P; ++q) row[base + q * span] = y[q];
    }
}

// Generic prime radix P (17 <= P <= 255; the 43 and 127 of N=4096's
// L = 16383, the 31 and 151 of N=8192's L = 32767) as a whole-CTA pass over
// batches of butterflies.  The batch's inputs (inter-pass twiddles
// applied) are staged in shared memory in the conjugate-pair form
// a_j = x_j + x_{P-j}, b_j = x_j - x_{P-j}; a thread then forms RS output
// pairs (s, P-s) of RB butterflies,
//   y_s, y_{P-s} = x_0 + sum_j a_j cos(2 pi js/P) +- i sum_j b_j sin(..),
// so each shared load of a root or of an a_j/b_j feeds several FMAs (the
// first version, one output pair per thread, was shared-load bound).
// Staging lives at the end of the dynamic shared memory (kGenBytes, added
// to the launch only when the length has such a radix).
constexpr int kGenMaxP = 255;
constexpr int kGenCap = 2048;                       // staged (a, b) items
constexpr int kGenRootsDoubles = 512;               // cos / sin of <= 256 roots
constexpr int kGenBytes = kGenRootsDoubles * 8 + 2 * kGenCap * 16;
constexpr int kGenRS = 2, kGenRB = 4;

__device__ __forceinline__ double *gen_staging() {
    extern __shared__ __align__(16) double2 dsm[];
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    return reinterpret_cast<double *>(reinterpret_cast<char *>(dsm) + dyn - kGenBytes);
}

__device__ void generic_pass(double2 *buf, int nrows, int L, int span, int P, const double2 *Tw,
                             const double2 *__restrict__ R, bool inv) {
    double *g = gen_staging();
    double *s_cr = g, *s_ci = g + kGenRootsDoubles / 2;
    double2 *s_a = reinterpret_cast<double2 *>(g + kGenRootsDoubles), *s_b = s_a + kGenCap;
    const int H = (P - 1) / 2, W = H + 1;
    const int NB = (kGenCap / W) / kGenRB * kGenRB;   // butterflies per batch
    const int NQ = NB / kGenRB, NSG = (H + kGenRS - 1) / kGenRS;
    for (int t = threadIdx.x; t < P; t += blockDim.x) {
        const double2 w = R[t];
        s_cr[t] = w.x;
        s_ci[t] = inv ? -w.y : w.y;
    }
    const int nb = L / P, total = nb * nrows;
    for (int g0 = 0; g0 < total; g0 += NB) {
        __syncthreads();   // roots written / previous batch's staging consumed
        // staging, item = j * NB + bi: consecutive threads take consecutive
        // butterflies (consecutive k), so the loads coalesce when span > 1;
        // kGenU items per thread have all their loads in flight before any
        // is used (rows in global scratch: the loads are L2 round trips)
        constexpr int kGenU = 4;
        for (int it0 = threadIdx.x; it0 < NB * W; it0 += kGenU * blockDim.x) {
            double2 xj[kGenU], xm[kGenU], tj[kGenU], tm[kGenU];
            int jj[kGenU], bb[kGenU];
#pragma unroll
            for (int u = 0; u < kGenU; ++u) {
                const int it = it0 + u * blockDim.x;
                const int j = it / NB, bi = it - j * NB, gi = g0 + bi;
                jj[u] = (it < NB * W && gi < total) ? j : -1;
                bb[u] = bi;
                xj[u] = xm[u] = tj[u] = tm[u] = make_double2(0.0, 0.0);
                if (jj[u] < 0) continue;
                const int rw = gi >= nb ? gi / nb : 0, tt = gi - rw * nb;
                const int gg = tt / span, k = tt - gg * span;
                const double2 *row = buf + (int64_t)rw * L + gg * span * P + k;
                xj[u] = row[j * span];
                if (j > 0) {
                    xm[u] = row[(P - j) * span];
                    if (span > 1) {
                        tj[u] = Tw[(j - 1) * span + k];
                        tm[u] = Tw[(P - j - 1) * span + k];
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kGenU; ++u) {
                const int j = jj[u], bi = bb[u];
                if (j < 0) continue;
                if (j == 0) {
                    s_a[bi] = xj[u];
                    s_b[bi] = make_double2(0.0, 0.0);
                } else {
                    double2 a = xj[u], c = xm[u];
                    if (span > 1) {
                        a = cmul(a, conjif(tj[u], inv));
                        c = cmul(c, conjif(tm[u], inv));
                    }
                    s_a[j * NB + bi] = make_double2(a.x + c.x, a.y + c.y);
                    s_b[j * NB + bi] = make_double2(a.x - c.x, a.y - c.y);
                }
            }
        }
        __syncthreads();
        // y_0 of every butterfly
        for (int bi = threadIdx.x; bi < NB; bi += blockDim.x) {
            const int gi = g0 + bi;
            if (gi >= total) continue;
            const int rw = gi >= nb ? gi / nb : 0, tt = gi - rw * nb;
            const int gg = tt / span, k = tt - gg * span;
            double2 y0 = s_a[bi];
            for (int j = 1; j <= H; ++j) {
                y0.x += s_a[j * NB + bi].x;
                y0.y += s_a[j * NB + bi].y;
            }
            buf[(int64_t)rw * L + gg * span * P + k] = y0;
        }
        // output pairs: item = bq + NQ * sg, RS pairs x RB butterflies
        // bi = r * NQ + bq; staging is j-major (entry j * NB + bi), so a
        // warp's loads of one (j, r) hit consecutive 16-byte entries
        for (int it = threadIdx.x; it < NQ * NSG; it += blockDim.x) {
            const int sg = it / NQ, bq = it - sg * NQ;
            const int s0 = 1 + sg * kGenRS;
            double2 re[kGenRS][kGenRB], im[kGenRS][kGenRB];
#pragma unroll
            for (int r = 0; r < kGenRB; ++r) {
                const double2 x0 = s_a[r * NQ + bq];
#pragma unroll
                for (int q = 0; q < kGenRS; ++q) {
                    re[q][r] = x0;
                    im[q][r] = make_double2(0.0, 0.0);
                }
            }
            int t[kGenRS];
#pragma unroll
            for (int q = 0; q < kGenRS; ++q) t[q] = 0;
            for (int j = 1; j <= H; ++j) {
                double c[kGenRS], sn[kGenRS];
#pragma unroll
                for (int q = 0; q < kGenRS; ++q) {
                    t[q] += s0 + q;
                    if (t[q] >= P) t[q] -= P;
                    c[q] = s_cr[t[q]];
                    sn[q] = s_ci[t[q]];
                }
#pragma unroll
                for (int r = 0; r < kGenRB; ++r) {
                    const double2 A = s_a[j * NB + r * NQ + bq];
                    const double2 B = s_b[j * NB + r * NQ + bq];
#pragma unroll
                    for (int q = 0; q < kGenRS; ++q) {
                        re[q][r].x = fma(A.x, c[q], re[q][r].x);
                        re[q][r].y = fma(A.y, c[q], re[q][r].y);
                        im[q][r].x = fma(B.x, sn[q], im[q][r].x);
                        im[q][r].y = fma(B.y, sn[q], im[q][r].y);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < kGenRB; ++r) {
                const int gi = g0 + r * NQ + bq;
                if (gi >= total) continue;
                const int rw = gi >= nb ? gi / nb : 0, tt = gi - rw * nb;
                const int gg = tt / span, k = tt - gg * span;
                double2 *row = buf + (int64_t)rw * L + gg * span * P + k;
#pragma unroll
                for (int q = 0; q < kGenRS; ++q) {
                    const int sidx = s0 + q;
                    if (sidx > H) continue;
                    row[sidx * span] = make_double2(re[q][r].x - im[q][r].y, re[q][r].y + im[q][r].x);
                    row[(P - sidx) * span] =
                        make_double2(re[q][r].x + im[q][r].y, re[q][r].y - im[q][r].x);
                }
            }
        }
    }
}

// All passes over `nrows` rows of buf (row stride Lb), whole CTA.  Tw: the
// pass twiddle table (Lb entries, shared or global memory); R: radix roots.
template <bool GEN = true>
__device__ void dft_passes(double2 *buf, int nrows, const DftDesc &d, const double2 *Tw,
                           const double2 *__restrict__ R, bool inv) {
    const int L = d.Lb;
    for (int ri = 0; ri < d.nrad; ++ri) {
        const int P = d.radix[ri], span = d.span[ri];
        const unsigned si = d.span_inv[ri];
        const double2 *tw = Tw + d.tw_off[ri];
        const double2 *rr = R + d.root_off[ri];
        switch (P) {
            case 2: radix_pass<2>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 3: radix_pass<3>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 4: radix_pass<4>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 5: radix_pass<5>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 7: radix_pass<7>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 9: radix_pass<9>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 11: radix_pass<11>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 13: radix_pass<13>(buf, nrows, L, span, si, tw, rr, inv); break;
            default:
                if (GEN) generic_pass(buf, nrows, L, span, P, tw, rr, inv);
                else __trap();   // launched without the generic radix (host picks by radices)
        }
        __syncthreads();
    }
}

// The transposed pass sequence (DIF): natural-order input, output at the
// digit-reversed positions perm[k].  Bluestein lengths are 2-3-5-7-smooth,
// so only templated radices occur.
__device__ void dft_passes_dif(double2 *buf, int nrows, const DftDesc &d, const double2 *Tw,
                               const double2 *__restrict__ R, bool inv) {
    const int L = d.Lb;
    for (int ri = d.nrad - 1; ri >= 0; --ri) {
        const int P = d.radix[ri], span = d.span[ri];
        const unsigned si = d.span_inv[ri];
        const double2 *tw = Tw + d.tw_off[ri];
        const double2 *rr = R + d.root_off[ri];
        switch (P) {
            case 2: radix_pass<2, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 3: radix_pass<3, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 4: radix_pass<4, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 5: radix_pass<5, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 7: radix_pass<7, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            case 9: radix_pass<9, true>(buf, nrows, L, span, si, tw, rr, inv); break;
            default: __trap();
        }
        __syncthreads();
    }
}

// Length-L DFT of `nrows` rows already scattered into buf (digit-reversed
// positions perm[j], j < L; for Bluestein rows pre-multiplied by the chirp
// and zero at every other position).  Direct rows: mixed-radix DIT, result
// in natural order.  Bluestein rows (Bluestein 1970 / Rabiner-Schafer-Rader
// chirp-z: jk = (j^2 + k^2 - (k-j)^2)/2, so y_k = c_k sum_j (x_j c_j)
// conj(c_{k-j}) with c_j = exp(-i pi j^2/L), a cyclic convolution of length
// M >= 2L-1): forward DIT FFT of length M, times H = FFT_M(conj c)/M
// (conjugated for the +i direction), inverse DIF FFT; the convolution lands
// at positions perm[k], to be multiplied by c_k (or conj c_k) on the way out.
template <bool GEN>
__device__ __forceinline__ void row_dft(double2 *buf, int nrows, const DftDesc &d,
                                        const double2 *Tw, const double2 *__restrict__ R,
                                        const double2 *__restrict__ H, bool inv) {
    if (!d.blue) {
        dft_passes<GEN>(buf, nrows, d, Tw, R, inv);
        return;
    }
    dft_passes<false>(buf, nrows, d, Tw, R, false);
    const int M = d.Lb;
    for (int rw = 0; rw < nrows; ++rw)
        for (int i = threadIdx.x; i < M; i += blockDim.x)
            buf[(int64_t)rw * M + i] = cmul(buf[(int64_t)rw * M + i], conjif(H[i], inv));
    __syncthreads();
    dft_passes_dif(buf, nrows, d, Tw, R, true);
}

// Zero the rows of a Bluestein buffer before the input scatter.
__device__ __forceinline__ void row_clear(double2 *buf, int nrows, const DftDesc &d) {
    if (!d.blue) return;
    for (int i = threadIdx.x; i < nrows * d.Lb; i += blockDim.x) buf[i] = make_double2(0.0, 0.0);
    __syncthreads();
}

// SM is a template argument so that, once inlined, every row access is a
// known shared-memory access (LDS/STS) rather than a generic one
template <bool SM>
__device__ __forceinline__ double2 *dft_buffer(double2 *scratch, int rows, int L) {
    extern __shared__ __align__(16) double2 dsm[];
    if (SM) return dsm;
    return scratch + (int64_t)blockIdx.x * rows * L;
}

// ---- standalone batched DFT: rows of length L (numpy fft / L*ifft)
template <bool SM, bool GEN>
__global__ void __launch_bounds__(kDftThreads, BF_DFT_MINBLOCKS) dft_rows_kernel(
    DftDesc d, const double2 *__restrict__ in, double2 *__restrict__ out, int64_t rows,
    const int *__restrict__ perm, const double2 *__restrict__ W, bool inv, bool use_smem,
    double2 *scratch, const double2 *__restrict__ chirp, const double2 *__restrict__ H) {
    const int L = d.L, Lb = d.Lb;
    double2 *buf = dft_buffer<SM>(scratch, 1, Lb);
    for (int64_t rw = blockIdx.x; rw < rows; rw += gridDim.x) {
        const double2 *src = in + rw * L;
        row_clear(buf, 1, d);
        for (int j = threadIdx.x; j < L; j += blockDim.x) {
            const double2 v = src[j];
            buf[perm[j]] = d.blue ? cmul(v, conjif(chirp[j], inv)) : v;
        }
        __syncthreads();
        row_dft<GEN>(buf, 1, d, W, W + Lb, H, inv);
        double2 *dst = out + rw * L;
        for (int j = threadIdx.x; j < L; j += blockDim.x)
            dst[j] = d.blue ? cmul(buf[perm[j]], conjif(chirp[j], inv)) : buf[j];
        __syncthreads();
    }
}

// ---- row-pair kernels on a 2-CTA cluster (rows that fit a CTA's half SM)
//
// Round 1 held both rows n+r / n-1-r in one CTA (128 KB of shared memory
// at N=1024 plus the twiddles): one CTA of 8 warps per SM, load, transform
// and store phases serialized (ncu: 12% occupancy).  Here the pair is a
// thread-block
// cluster of two CTAs, one row each (rank 0: row n+r, rank 1: row n-1-r),
// 64 KB of shared memory and <= 128 registers per thread, so two clusters'
// CTAs share an SM and one CTA's DRAM phase overlaps another's transform.
// The parity coupling crosses the pair through distributed shared memory:
// forward, each rank reads the node halves of half of the orders and
// stores g_e + g_o into rank 0's row and g_e - g_o into rank 1's
// (alt.py:225-236); inverse, after both row DFTs, each rank reads bins m
// and L-m of both rows (one local, one remote) for half of the orders and
// writes the weighted fold (alt.py:239-253).  Twiddle tables are read
// through L1.  One cluster per row pair, grid = 2 * rows.
template <bool GEN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, BF_PAIR_MINBLOCKS)
    sht_synth_pair_kernel(DftDesc d, int n, const bf_half *__restrict__ halves,
                          const double *__restrict__ arena, int r_count,
                          const double2 *__restrict__ tw, const int *__restrict__ perm,
                          const double2 *__restrict__ W, double2 *__restrict__ grid, int64_t yr,
                          int ystride, int ew, const double2 *__restrict__ chirp,
                          const double2 *__restrict__ H) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    extern __shared__ __align__(16) double2 dsm[];
    const int L = d.L, Lb = d.Lb;
    double2 *own = dsm;
    double2 *peer = cl.map_shared_rank(dsm, rank ^ 1u);
    double2 *bplus = rank ? peer : own, *bminus = rank ? own : peer;
    const int rr = blockIdx.x >> 1;
    if (d.blue)
        for (int i = threadIdx.x; i < Lb; i += blockDim.x) own[i] = make_double2(0.0, 0.0);
    cl.sync();   // both CTAs running (and Bluestein rows cleared) before remote stores
    const int nord = 2 * n, half = (nord + 1) >> 1;
    const int a_lo = rank ? half : 0, a_hi = rank ? nord : half;
    constexpr int kBatch = 2;
    for (int a0 = a_lo + threadIdx.x; a0 < a_hi; a0 += kBatch * blockDim.x) {
        double2 op[kBatch], on[kBatch], ep[kBatch], en[kBatch], tp[kBatch], tn[kBatch];
        int pp[kBatch], pn[kBatch];
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int am = a0 + i * blockDim.x;
            const bool ok = am < a_hi;
            op[i] = on[i] = ep[i] = en[i] = make_double2(0.0, 0.0);
            if (ok) {
                const double2 *eo = nullptr, *ee = nullptr;
                if (ystride > 0) {
                    const double *rowp = arena + (yr + (int64_t)rr * ystride) * ew;
                    eo = reinterpret_cast<const double2 *>(rowp + (2 * am) * ew);
                    ee = reinterpret_cast<const double2 *>(rowp + (2 * am + 1) * ew);
                } else {
                    const bf_half ho = halves[2 * am], he = halves[2 * am + 1];
                    if (ho.ncols > 0)
                        eo = reinterpret_cast<const double2 *>(
                            arena + ((int64_t)ho.y + (int64_t)rr * ho.x) * ew);
                    if (he.ncols > 0)
                        ee = reinterpret_cast<const double2 *>(
                            arena + ((int64_t)he.y + (int64_t)rr * he.x) * ew);
                }
                if (eo) {
                    op[i] = eo[0];
                    on[i] = eo[1];
                }
                if (ee) {
                    ep[i] = ee[0];
                    en[i] = ee[1];
                }
            }
            const int bn = am > 0 && ok ? L - am : 0;
            tp[i] = ok ? tw[am] : make_double2(0.0, 0.0);
            tn[i] = ok ? tw[bn] : make_double2(0.0, 0.0);
            if (d.blue && ok) {
                tp[i] = cmul(tp[i], conjif(chirp[am], true));
                tn[i] = cmul(tn[i], conjif(chirp[bn], true));
            }
            pp[i] = ok ? perm[am] : 0;
            pn[i] = ok ? perm[bn] : 0;
        }
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int am = a0 + i * blockDim.x;
            if (am < a_hi) {
                bplus[pp[i]] = cmul(make_double2(ep[i].x + op[i].x, ep[i].y + op[i].y), tp[i]);
                bminus[pp[i]] = cmul(make_double2(ep[i].x - op[i].x, ep[i].y - op[i].y), tp[i]);
                if (am > 0) {
                    bplus[pn[i]] = cmul(make_double2(en[i].x + on[i].x, en[i].y + on[i].y), tn[i]);
                    bminus[pn[i]] = cmul(make_double2(en[i].x - on[i].x, en[i].y - on[i].y), tn[i]);
                }
            }
        }
    }
    cl.sync();   // both rows assembled; no remote access after this point
    row_dft<GEN>(own, 1, d, W, W + Lb, H, true);
    double2 *out = grid + (int64_t)(rank ? r_count - 1 - rr : r_count + rr) * L;
    for (int j0 = threadIdx.x; j0 < L; j0 += 2 * blockDim.x) {
        double2 v[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = j0 + u * blockDim.x;
            if (j < L) {
                v[u] = own[d.blue ? perm[j] : j];
                if (d.blue) v[u] = cmul(v[u], conjif(chirp[j], true));
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int j = j0 + u * blockDim.x;
            if (j < L) out[j] = v[u];
        }
    }
}

// Forward, one row per CTA without a cluster: each CTA reads the node
// halves of every order for its row (the pair's second read of the same
// entries is an L2 hit, both CTAs run together) and assembles g_e + g_o
// (row n+r) or g_e - g_o (row n-1-r).  SM: the row in shared memory
// (grid = 2 * r_count); else in a global (L2-resident) scratch row per
// CTA, persistent over the rows — the path of rows too long for shared
// memory (N >= 2048), at 128 registers so two CTAs share an SM.
template <bool SM, bool GEN>
__global__ void __launch_bounds__(kDftThreads, BF_DFT_MINBLOCKS)
    sht_synth_row_kernel(DftDesc d, int n, const bf_half *__restrict__ halves,
                         const double *__restrict__ arena, int r_count,
                         const double2 *__restrict__ tw, const int *__restrict__ perm,
                         const double2 *__restrict__ W, double2 *__restrict__ grid, int64_t yr,
                         int ystride, int ew, const double2 *__restrict__ chirp,
                         const double2 *__restrict__ H, double2 *scratch) {
    const int L = d.L, Lb = d.Lb;
    double2 *buf = dft_buffer<SM>(scratch, 1, Lb);
    const int nord = 2 * n;
    for (int t = blockIdx.x; t < 2 * r_count; t += gridDim.x) {
        const int rr = t >> 1;
        const bool lower = t & 1;
        if (d.blue) {
            for (int i = threadIdx.x; i < Lb; i += blockDim.x) buf[i] = make_double2(0.0, 0.0);
            __syncthreads();
        }
        constexpr int kBatch = 2;
        for (int a0 = threadIdx.x; a0 < nord; a0 += kBatch * blockDim.x) {
            double2 op[kBatch], on[kBatch], ep[kBatch], en[kBatch], tp[kBatch], tn[kBatch];
            int pp[kBatch], pn[kBatch];
#pragma unroll
            for (int i = 0; i < kBatch; ++i) {
                const int am = a0 + i * blockDim.x;
                const bool ok = am < nord;
                op[i] = on[i] = ep[i] = en[i] = make_double2(0.0, 0.0);
                if (ok) {
                    const double2 *eo = nullptr, *ee = nullptr;
                    if (ystride > 0) {
                        const double *rowp = arena + (yr + (int64_t)rr * ystride) * ew;
                        eo = reinterpret_cast<const double2 *>(rowp + (2 * am) * ew);
                        ee = reinterpret_cast<const double2 *>(rowp + (2 * am + 1) * ew);
                    } else {
                        const bf_half ho = halves[2 * am], he = halves[2 * am + 1];
                        if (ho.ncols > 0)
                            eo = reinterpret_cast<const double2 *>(
                                arena + ((int64_t)ho.y + (int64_t)rr * ho.x) * ew);
                        if (he.ncols > 0)
                            ee = reinterpret_cast<const double2 *>(
                                arena + ((int64_t)he.y + (int64_t)rr * he.x) * ew);
                    }
                    if (eo) {
                        op[i] = eo[0];
                        on[i] = eo[1];
                    }
                    if (ee) {
                        ep[i] = ee[0];
                        en[i] = ee[1];
                    }
                }
                const int bn = am > 0 && ok ? L - am : 0;
                tp[i] = ok ? tw[am] : make_double2(0.0, 0.0);
                tn[i] = ok ? tw[bn] : make_double2(0.0, 0.0);
                if (d.blue && ok) {
                    tp[i] = cmul(tp[i], conjif(chirp[am], true));
                    tn[i] = cmul(tn[i], conjif(chirp[bn], true));
                }
                pp[i] = ok ? perm[am] : 0;
                pn[i] = ok ? perm[bn] : 0;
            }
#pragma unroll
            for (int i = 0; i < kBatch; ++i) {
                const int am = a0 + i * blockDim.x;
                if (am < nord) {
                    const double2 vp = lower ? make_double2(ep[i].x - op[i].x, ep[i].y - op[i].y)
                                             : make_double2(ep[i].x + op[i].x, ep[i].y + op[i].y);
                    buf[pp[i]] = cmul(vp, tp[i]);
                    if (am > 0) {
                        const double2 vn = lower
                                               ? make_double2(en[i].x - on[i].x, en[i].y - on[i].y)
                                               : make_double2(en[i].x + on[i].x, en[i].y + on[i].y);
                        buf[pn[i]] = cmul(vn, tn[i]);
                    }
                }
            }
        }
        __syncthreads();
        row_dft<GEN>(buf, 1, d, W, W + Lb, H, true);
        double2 *out = grid + (int64_t)(lower ? r_count - 1 - rr : r_count + rr) * L;
        for (int j0 = threadIdx.x; j0 < L; j0 += 2 * blockDim.x) {
            double2 v[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = j0 + u * blockDim.x;
                if (j < L) {
                    v[u] = buf[d.blue ? perm[j] : j];
                    if (d.blue) v[u] = cmul(v[u], conjif(chirp[j], true));
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = j0 + u * blockDim.x;
                if (j < L) out[j] = v[u];
            }
        }
        __syncthreads();
    }
}

// SM = false: each CTA's row lives in a global (L2-resident) scratch row,
// the cluster persistent over row pairs; the peer's row is read through
// global memory after the cluster barrier (release / acquire at cluster
// scope orders those accesses).
template <bool SM, bool GEN>
__global__ void __cluster_dims__(2, 1, 1)
    __launch_bounds__(SM ? kPairThreads : kDftThreads, SM ? BF_PAIR_MINBLOCKS : BF_DFT_MINBLOCKS)
    sht_anal_pair_kernel(DftDesc d, int n, const bf_half *__restrict__ halves,
                         double *__restrict__ arena, const double2 *__restrict__ tw,
                         const int *__restrict__ perm, const double2 *__restrict__ W,
                         const double2 *__restrict__ grid, const double *__restrict__ weights,
                         int r_begin, int r_count, const int *__restrict__ node_y, int ew,
                         const double2 *__restrict__ chirp, const double2 *__restrict__ H,
                         double2 *scratch) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    extern __shared__ __align__(16) double2 dsm[];
    const int L = d.L, Lb = d.Lb;
    double2 *own = SM ? dsm : scratch + (int64_t)blockIdx.x * Lb;
    const double2 *peer = SM ? cl.map_shared_rank(dsm, rank ^ 1u)
                             : scratch + (int64_t)(blockIdx.x ^ 1u) * Lb;
    for (int rr = blockIdx.x >> 1; rr < r_count; rr += gridDim.x >> 1) {
    const double2 *src = grid + (int64_t)(rank ? r_count - 1 - rr : r_count + rr) * L;
    if (d.blue) {
        for (int i = threadIdx.x; i < Lb; i += blockDim.x) own[i] = make_double2(0.0, 0.0);
        __syncthreads();
    }
    constexpr int kBatch = 4;   // issue a batch of loads before using any
    for (int j0 = threadIdx.x; j0 < L; j0 += kBatch * blockDim.x) {
        double2 u[kBatch];
        int p[kBatch];
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int j = j0 + i * blockDim.x;
            if (j < L) {
                p[i] = perm[j];
                u[i] = src[j];
            }
        }
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int j = j0 + i * blockDim.x;
            if (j < L) own[p[i]] = d.blue ? cmul(u[i], chirp[j]) : u[i];
        }
    }
    __syncthreads();
    row_dft<GEN>(own, 1, d, W, W + Lb, H, false);
    cl.sync();   // both spectra ready
    const double2 *bU = rank ? peer : own, *bL = rank ? own : peer;
    const int r = r_begin + rr;
    const double w = weights[n + r];
    const double invL = 1.0 / (double)L;
    const int nord = 2 * n, half = (nord + 1) >> 1;
    const int a_lo = rank ? half : 0, a_hi = rank ? nord : half;
    for (int am = a_lo + threadIdx.x; am < a_hi; am += blockDim.x) {
        int yo, ye, xo = 1, xe = 1;
        if (node_y) {
            yo = node_y[2 * am];
            ye = node_y[2 * am + 1];
        } else {
            const bf_half ho = halves[2 * am], he = halves[2 * am + 1];
            yo = ho.ncols > 0 ? ho.y : -1;
            ye = he.ncols > 0 ? he.y : -1;
            xo = ho.x;
            xe = he.x;
        }
        const int bn = L - am;
        const int pa = d.blue ? perm[am] : am, pb = d.blue ? perm[bn] : bn;
        double2 sa = bU[pa], sb = bL[pa];
        if (d.blue) {
            const double2 c = chirp[am];
            sa = cmul(sa, c);
            sb = cmul(sb, c);
        }
        const double2 tp = tw[am];
        const double2 cp = make_double2(tp.x, -tp.y);
        sa = cmul(make_double2(sa.x * invL, sa.y * invL), cp);
        sb = cmul(make_double2(sb.x * invL, sb.y * invL), cp);
        double2 na = make_double2(0.0, 0.0), nb = na;
        if (am > 0) {
            const double2 tn = tw[bn];
            const double2 cn = make_double2(tn.x, -tn.y);
            na = bU[pb];
            nb = bL[pb];
            if (d.blue) {
                const double2 c = chirp[bn];
                na = cmul(na, c);
                nb = cmul(nb, c);
            }
            na = cmul(make_double2(na.x * invL, na.y * invL), cn);
            nb = cmul(make_double2(nb.x * invL, nb.y * invL), cn);
        }
        if (yo >= 0) {
            double2 *e = reinterpret_cast<double2 *>(arena + ((int64_t)yo + (int64_t)rr * xo) * ew);
            e[0] = make_double2(w * (sa.x - sb.x), w * (sa.y - sb.y));
            e[1] = am > 0 ? make_double2(w * (na.x - nb.x), w * (na.y - nb.y))
                          : make_double2(0.0, 0.0);
        }
        if (ye >= 0) {
            double2 *e = reinterpret_cast<double2 *>(arena + ((int64_t)ye + (int64_t)rr * xe) * ew);
            e[0] = make_double2(w * (sa.x + sb.x), w * (sa.y + sb.y));
            e[1] = am > 0 ? make_double2(w * (na.x + nb.x), w * (na.y + nb.y))
                          : make_double2(0.0, 0.0);
        }
    }
    cl.sync();   // the peer has finished reading this CTA's row
    }
}

__device__ __forceinline__ int64_t coeff_offset(int m, int K) {
    // start of order m in ShtCoeffs.pack() (m ascending from -(K-1)), K = 2N
    if (m <= 0) return (int64_t)(K + m - 1) * (K + m) / 2;
    return (int64_t)(K - 1) * K / 2 + (int64_t)m * K - (int64_t)m * (m - 1) / 2;
}

// coefficient halves for the whole SHT: entry = (Re, Im) of +m then -m
__global__ void coef_pack_kernel(int n, const bf_half *__restrict__ halves,
                                 const double2 *__restrict__ c, double *__restrict__ arena, int ew) {
    const int am = blockIdx.y;
    const int K = 2 * n;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * am + par];
        if (j >= h.ncols) continue;
        const int k = (par == 0 ? 1 : 0) + 2 * j;
        const double2 p = c ? c[coeff_offset(am, K) + k] : make_double2(0.0, 0.0);
        const double2 q = (c && am) ? c[coeff_offset(-am, K) + k] : make_double2(0.0, 0.0);
        double *e = arena + ((int64_t)h.x + j) * ew;
        *reinterpret_cast<double2 *>(e) = p;
        *reinterpret_cast<double2 *>(e + 2) = q;
    }
}

__global__ void coef_unpack_kernel(int n, const bf_half *__restrict__ halves,
                                   const double *__restrict__ arena, double2 *__restrict__ c, int ew) {
    const int am = blockIdx.y;
    const int K = 2 * n;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * am + par];
        if (j >= h.ncols) continue;
        const int k = (par == 0 ? 1 : 0) + 2 * j;
        const double *e = arena + ((int64_t)h.x + j) * ew;
        c[coeff_offset(am, K) + k] = *reinterpret_cast<const double2 *>(e);
        if (am) c[coeff_offset(-am, K) + k] = *reinterpret_cast<const double2 *>(e + 2);
    }
}

// ---- per-order boundary (alt_forward / alt_inverse on plans o = 0..)
// off[o] = start of order o's coefficient vector (length 2N - m_o)
__global__ void orders_pack_kernel(int n, const bf_half *__restrict__ halves,
                                   const int64_t *__restrict__ off, const double2 *__restrict__ in,
                                   double *__restrict__ arena) {
    const int o = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        const double2 v = in[off[o] + (par == 0 ? 1 : 0) + 2 * j];
        double *e = arena + ((int64_t)h.x + j) * BF_NRHS;
        *reinterpret_cast<double2 *>(e) = v;
        *reinterpret_cast<double2 *>(e + 2) = make_double2(0.0, 0.0);
    }
}

__global__ void orders_unpack_kernel(int n, const bf_half *__restrict__ halves,
                                     const int64_t *__restrict__ off,
                                     const double *__restrict__ arena, double2 *__restrict__ out) {
    const int o = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        out[off[o] + (par == 0 ? 1 : 0) + 2 * j] =
            *reinterpret_cast<const double2 *>(arena + ((int64_t)h.x + j) * BF_NRHS);
    }
}

__global__ void orders_assemble_kernel(int n, const bf_half *__restrict__ halves,
                                       const double *__restrict__ arena, double2 *__restrict__ out) {
    const int o = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const bf_half ho = halves[2 * o], he = halves[2 * o + 1];
    double2 go = make_double2(0.0, 0.0), ge = go;
    if (ho.ncols > 0) go = *reinterpret_cast<const double2 *>(arena + ((int64_t)ho.y + (int64_t)r * ho.x) * BF_NRHS);
    if (he.ncols > 0) ge = *reinterpret_cast<const double2 *>(arena + ((int64_t)he.y + (int64_t)r * he.x) * BF_NRHS);
    double2 *col = out + (int64_t)o * 2 * n;
    col[n + r] = make_double2(ge.x + go.x, ge.y + go.y);
    col[n - 1 - r] = make_double2(ge.x - go.x, ge.y - go.y);
}

__global__ void orders_fold_kernel(int n, const bf_half *__restrict__ halves,
                                   const double2 *__restrict__ in, const double *__restrict__ weights,
                                   double *__restrict__ arena) {
    const int o = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double2 *col = in + (int64_t)o * 2 * n;
    const double2 up = col[n + r], lo = col[n - 1 - r];
    const double w = weights[n + r];
    const bf_half ho = halves[2 * o], he = halves[2 * o + 1];
    if (ho.ncols > 0) {
        double *e = arena + ((int64_t)ho.y + r) * BF_NRHS;
        *reinterpret_cast<double2 *>(e) = make_double2(w * (up.x - lo.x), w * (up.y - lo.y));
        *reinterpret_cast<double2 *>(e + 2) = make_double2(0.0, 0.0);
    }
    if (he.ncols > 0) {
        double *e = arena + ((int64_t)he.y + r) * BF_NRHS;
        *reinterpret_cast<double2 *>(e) = make_double2(w * (up.x + lo.x), w * (up.y + lo.y));
        *reinterpret_cast<double2 *>(e + 2) = make_double2(0.0, 0.0);
    }
}

std::vector<int> factorize(int64_t L) {
    // prime factors ascending, with pairs of 2s merged into the radix-4 pass
    std::vector<int> f;
    int twos = 0;
    while (L % 2 == 0) {
        ++twos;
        L /= 2;
    }
    for (; twos >= 2; twos -= 2) f.push_back(4);
    if (twos) f.push_back(2);
    // pairs of 3s as one radix-9 pass (one shared-memory round trip fewer;
    // the passes are L1-bound)
    int threes = 0;
    while (L % 3 == 0) {
        ++threes;
        L /= 3;
    }
    for (; threes >= 2; threes -= 2) f.push_back(9);
    if (threes) f.push_back(3);
    for (int p = 5; (int64_t)p * p <= L; p += 2)
        while (L % p == 0) {
            f.push_back(p);
            L /= p;
        }
    if (L > 1) f.push_back((int)L);
    return f;
}

// Smallest 2-3-5-7-smooth length >= need (Bluestein convolution length).
int64_t smooth_at_least(int64_t need) {
    int64_t best = INT64_MAX;
    for (int64_t a = 1; a < 2 * need; a *= 2)
        for (int64_t b = a; b < 2 * need; b *= 3)
            for (int64_t c = b; c < 2 * need; c *= 5)
                for (int64_t d = c; d < 2 * need; d *= 7)
                    if (d >= need && d < best) best = d;
    return best;
}

// Host FFT in long double (recursive, smallest prime first), sign -1 or +1:
// the Bluestein kernel spectrum H, computed once per length.
void host_fft(std::vector<std::complex<long double>> &a, int sign) {
    const int64_t n = (int64_t)a.size();
    if (n <= 1) return;
    int64_t p = 2;
    while (n % p) ++p;
    const int64_t m = n / p;
    std::vector<std::vector<std::complex<long double>>> sub(p, std::vector<std::complex<long double>>(m));
    for (int64_t i = 0; i < n; ++i) sub[i % p][i / p] = a[i];
    for (auto &v : sub) host_fft(v, sign);
    const long double two_pi = 6.283185307179586476925286766559L;
    for (int64_t k = 0; k < n; ++k) {
        std::complex<long double> acc = 0;
        for (int64_t r = 0; r < p; ++r) {
            const long double ang = sign * two_pi * (long double)((r * k) % n) / (long double)n;
            acc += sub[r][k % m] * std::complex<long double>(std::cos(ang), std::sin(ang));
        }
        a[k] = acc;
    }
}

int perm_of(int64_t nidx, const std::vector<int> &rad, int upto) {
    // position of input index nidx after digit reversal for radices[0..upto)
    if (upto == 0) return 0;
    const int p = rad[upto - 1];
    int64_t M = 1;
    for (int i = 0; i < upto - 1; ++i) M *= rad[i];
    return (int)((nidx % p) * M + perm_of(nidx / p, rad, upto - 1));
}

DftDesc make_desc(const bfsht_plan *pl) {
    DftDesc d;
    d.L = (int)pl->dft_L;
    d.Lb = (int)pl->dft_Lb;
    d.blue = pl->dft_blue ? 1 : 0;
    d.nrad = (int)pl->dft_radix.size();
    int64_t span = 1;
    int tw = 0, ro = 0;
    for (int i = 0; i < d.nrad; ++i) {
        d.radix[i] = pl->dft_radix[i];
        // ceil(2^32 / span): exact for the quotients used (x < L <= 2^20,
        // verified exhaustively in bf_dft_prepare)
        d.span_inv[i] = span == 1 ? 0u : (unsigned)(((1ULL << 32) + span - 1) / span);
        d.tw_off[i] = tw;
        d.root_off[i] = ro;
        d.span[i] = (int)span;
        tw += (int)((pl->dft_radix[i] - 1) * span);
        ro += pl->dft_radix[i];
        span *= pl->dft_radix[i];
    }
    return d;
}

int dft_smem_bytes(int64_t L, int rows) { return (int)(rows * L * 16); }

// generic-radix staging bytes of a factorization (0 when every radix is templated)
int dft_gen_bytes(const std::vector<int> &rad) {
    for (int p : rad)
        if (p > 13) return kGenBytes;
    return 0;
}
}  // namespace

// Tables of the length-L DFT stage (built once per length, on the plan's
// device).  Lengths whose prime factors are all <= kGenMaxP run as direct
// mixed-radix rows; any other length (a prime factor above 255, e.g. N=2048's
// L = 8191 or N=66's L = 263 = prime) runs as a Bluestein row of the
// smallest 2-3-5-7-smooth length M >= 2L-1.  BFSHT_BLUESTEIN_ABOVE=p moves
// the threshold (tests force Bluestein onto small lengths with it).
int bf_dft_prepare(bfsht_plan *pl, int64_t L) {
    int above = kGenMaxP;
    if (const char *e = std::getenv("BFSHT_BLUESTEIN_ABOVE")) above = std::atoi(e);
    std::vector<int> rad_l = factorize(L);
    bool blue = false;
    for (int p : rad_l)
        if (p > above || p > kGenMaxP) blue = true;
    if (pl->dft_L == L && pl->dft_blue == blue) return 0;
    const int64_t Lb = blue ? smooth_at_least(2 * L - 1) : L;
    if (Lb > (1 << 20)) {
        bfsht_set_error("DFT length too large (buffer above 2^20)");
        return -4;
    }
    std::vector<int> rad = blue ? factorize(Lb) : rad_l;
    if ((int)rad.size() > kMaxRadix) {
        bfsht_set_error("DFT length has too many prime factors");
        return -4;
    }
    {
        // the multiply-high quotients of make_desc must be exact for every
        // butterfly index of every pass
        int64_t span = 1;
        for (int p : rad) {
            if (span > 1) {
                const uint64_t inv = ((1ULL << 32) + span - 1) / span;
                for (int64_t x = 0; x < Lb; ++x)
                    if ((int64_t)(((uint64_t)x * inv) >> 32) != x / span) {
                        bfsht_set_error("DFT index division check failed");
                        return -4;
                    }
            }
            span *= p;
        }
    }
    std::vector<double> w(2 * Lb), tw(2 * L), wt;
    std::vector<int32_t> perm(Lb);
    const double two_pi = 6.283185307179586476925286766559;
    for (int64_t k = 0; k < Lb; ++k) {
        // exp(-2 pi i k / Lb), argument reduced to (-pi, pi] for accuracy
        int64_t kk = k <= Lb / 2 ? k : k - Lb;
        double a = -two_pi * (double)kk / (double)Lb;
        w[2 * k] = std::cos(a);
        w[2 * k + 1] = std::sin(a);
        perm[k] = perm_of(k, rad, (int)rad.size());
    }
    const int64_t ntop = (L + 1) / 4 * 2 - 1;  // 2N - 1 for L = 4N - 1
    const double phi0 = 3.14159265358979323846264338327950288 / (double)L;
    for (int64_t b = 0; b < L; ++b) {
        int64_t m = b <= ntop ? b : b - L;
        std::complex<double> t = std::exp(std::complex<double>(0.0, (double)m * phi0));
        tw[2 * b] = t.real();
        tw[2 * b + 1] = t.imag();
    }
    // pass table: [0, Lb) inter-pass twiddles, pass after pass, entry
    // (q-1)*span + k = w[q k Lb/(span P)]; then the radix roots of every
    // pass, w[t Lb/P] for t < P
    {
        wt.assign(2 * Lb, 0.0);
        int64_t span = 1, off = 0;
        for (int p : rad) {
            const int64_t tstep = Lb / (span * p);
            for (int q = 1; q < p; ++q)
                for (int64_t k = 0; k < span; ++k) {
                    const int64_t e = (q * k * tstep) % Lb;
                    wt[2 * (off + (q - 1) * span + k)] = w[2 * e];
                    wt[2 * (off + (q - 1) * span + k) + 1] = w[2 * e + 1];
                }
            off += (p - 1) * span;
            span *= p;
        }
        for (int p : rad)
            for (int t = 0; t < p; ++t) {
                const int64_t e = t * (Lb / p);
                wt.push_back(w[2 * e]);
                wt.push_back(w[2 * e + 1]);
            }
    }
    // Bluestein: chirp c_j = exp(-i pi j^2 / L) (j^2 reduced mod 2L, exact
    // in int64) and H = FFT_M(h) / M, h_d = conj(c_|d|) at d mod M, |d| < L
    std::vector<double> chirp, hh;
    if (blue) {
        const long double pi = 3.14159265358979323846264338327950288L;
        std::vector<std::complex<long double>> c(L), h(Lb, 0.0L);
        for (int64_t j = 0; j < L; ++j) {
            const int64_t r = (j * j) % (2 * L);
            const long double ang = -pi * (long double)r / (long double)L;
            c[j] = std::complex<long double>(std::cos(ang), std::sin(ang));
        }
        for (int64_t d = 0; d < L; ++d) {
            h[d] = std::conj(c[d]);
            if (d) h[Lb - d] = std::conj(c[d]);
        }
        host_fft(h, -1);
        chirp.resize(2 * L);
        hh.resize(2 * Lb);
        for (int64_t j = 0; j < L; ++j) {
            chirp[2 * j] = (double)c[j].real();
            chirp[2 * j + 1] = (double)c[j].imag();
        }
        for (int64_t k = 0; k < Lb; ++k) {
            hh[2 * k] = (double)(h[k].real() / (long double)Lb);
            hh[2 * k + 1] = (double)(h[k].imag() / (long double)Lb);
        }
    }
    // re-prepare for a new length: every table and the scratch of the old one go
    for (void *p : {(void *)pl->dft_w, (void *)pl->dft_perm, (void *)pl->dft_tw,
                    (void *)pl->dft_scratch, (void *)pl->dft_chirp, (void *)pl->dft_hhat})
        if (p) cudaFree(p);
    pl->dft_w = pl->dft_tw = pl->dft_chirp = pl->dft_hhat = nullptr;
    pl->dft_perm = nullptr;
    pl->dft_scratch = nullptr;
    pl->dft_scratch_rows = 0;
    pl->dft_L = 0;
    BF_CUDA(cudaMalloc(&pl->dft_w, 8 * wt.size()));
    BF_CUDA(cudaMalloc(&pl->dft_tw, 16 * L));
    BF_CUDA(cudaMalloc(&pl->dft_perm, 4 * Lb));
    BF_CUDA(cudaMemcpy(pl->dft_w, wt.data(), 8 * wt.size(), cudaMemcpyHostToDevice));
    BF_CUDA(cudaMemcpy(pl->dft_tw, tw.data(), 16 * L, cudaMemcpyHostToDevice));
    BF_CUDA(cudaMemcpy(pl->dft_perm, perm.data(), 4 * Lb, cudaMemcpyHostToDevice));
    if (blue) {
        BF_CUDA(cudaMalloc(&pl->dft_chirp, 16 * L));
        BF_CUDA(cudaMalloc(&pl->dft_hhat, 16 * Lb));
        BF_CUDA(cudaMemcpy(pl->dft_chirp, chirp.data(), 16 * L, cudaMemcpyHostToDevice));
        BF_CUDA(cudaMemcpy(pl->dft_hhat, hh.data(), 16 * Lb, cudaMemcpyHostToDevice));
    }
    pl->dft_radix = rad;
    pl->dft_L = L;
    pl->dft_Lb = Lb;
    pl->dft_blue = blue;
    pl->dft_gen = dft_gen_bytes(rad);
    const int gen = pl->dft_gen;
    // global scratch rows for rows longer than half an SM's shared memory
    if (Lb * 16 + gen > kPairSmemMax) {
        const int64_t rows = 2 * (int64_t)pl->sm_count * 4;
        BF_CUDA(cudaMalloc(&pl->dft_scratch, 16 * Lb * rows));
        pl->dft_scratch_rows = rows;
    }
    // dynamic shared-memory limits are raised per launch (bf_ensure_smem)
    return 0;
}

// DFT-stage kernel choice.  A row in half an SM's shared memory: rows in
// shared memory, two CTAs per SM, a 2-CTA cluster per row pair (measured
// at N=1024 against the round-1 kernels that held both rows in one CTA:
// synthesis 0.204 vs 0.209 ms, and a one-row-per-CTA synthesis without the
// cluster 0.245 ms).  Longer rows: global (L2-resident) scratch rows,
// persistent grids (synthesis one row per CTA, analysis the cluster pair).
static bool pair_path(const bfsht_plan *pl) {
    return pl->dft_Lb * 16 + pl->dft_gen <= kPairSmemMax;
}
static int scratch_grid(const bfsht_plan *pl, int r_count) {
    const int64_t g = std::min<int64_t>(2LL * r_count, pl->dft_scratch_rows) & ~1LL;
    return (int)g;
}

// Forward DFT stage over row pairs r_begin .. r_begin + r_count - 1: node
// halves through `halves` (or the row-major Yr array when ystride > 0) ->
// 2 r_count grid rows.
static int launch_synth(bfsht_plan *pl, const bf_half *halves, const double *arena, int r_begin,
                        int r_count, double *grid, int64_t yr, int ystride, int ew,
                        cudaStream_t st) {
    const int n = pl->n;
    const DftDesc d = make_desc(pl);
    const double2 *tw = reinterpret_cast<const double2 *>(pl->dft_tw);
    const double2 *W = reinterpret_cast<const double2 *>(pl->dft_w);
    const double2 *chirp = reinterpret_cast<const double2 *>(pl->dft_chirp);
    const double2 *H = reinterpret_cast<const double2 *>(pl->dft_hhat);
    double2 *g = reinterpret_cast<double2 *>(grid);
    if (pair_path(pl)) {
        const int smem = (int)(pl->dft_Lb * 16) + pl->dft_gen;
        auto kern = pl->dft_gen ? sht_synth_pair_kernel<true> : sht_synth_pair_kernel<false>;
        int rc = bf_ensure_smem((const void *)kern, smem);
        if (rc) return rc;
        kern<<<2 * r_count, kPairThreads, smem, st>>>(d, n, halves, arena, r_count, tw,
                                                     pl->dft_perm, W, g, yr, ystride, ew, chirp, H);
    } else {
        auto kern = pl->dft_gen ? sht_synth_row_kernel<false, true>
                                : sht_synth_row_kernel<false, false>;
        int rc = bf_ensure_smem((const void *)kern, pl->dft_gen);
        if (rc) return rc;
        kern<<<scratch_grid(pl, r_count), kDftThreads, pl->dft_gen, st>>>(
            d, n, halves, arena, r_count, tw, pl->dft_perm, W, g, yr, ystride, ew, chirp, H,
            reinterpret_cast<double2 *>(pl->dft_scratch));
    }
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

// Inverse DFT stage: 2 r_count grid rows -> weighted node halves
// (node_y: per-half base with consecutive rows, else through `halves`).
static int launch_anal(bfsht_plan *pl, const bf_half *halves, double *arena, int r_begin,
                       int r_count, const double *grid, const double *weights, const int *node_y,
                       int ew, cudaStream_t st) {
    const int n = pl->n;
    const DftDesc d = make_desc(pl);
    const double2 *tw = reinterpret_cast<const double2 *>(pl->dft_tw);
    const double2 *W = reinterpret_cast<const double2 *>(pl->dft_w);
    const double2 *chirp = reinterpret_cast<const double2 *>(pl->dft_chirp);
    const double2 *H = reinterpret_cast<const double2 *>(pl->dft_hhat);
    const double2 *g = reinterpret_cast<const double2 *>(grid);
    const bool sm = pair_path(pl);
    const int smem = sm ? (int)(pl->dft_Lb * 16) + pl->dft_gen : pl->dft_gen;
    auto kern = sm ? (pl->dft_gen ? sht_anal_pair_kernel<true, true>
                                  : sht_anal_pair_kernel<true, false>)
                   : (pl->dft_gen ? sht_anal_pair_kernel<false, true>
                                  : sht_anal_pair_kernel<false, false>);
    const int nblk = sm ? 2 * r_count : scratch_grid(pl, r_count);
    int rc = bf_ensure_smem((const void *)kern, smem);
    if (rc) return rc;
    kern<<<nblk, sm ? kPairThreads : kDftThreads, smem, st>>>(d, n, halves, arena, tw, pl->dft_perm, W, g, weights,
                                          r_begin, r_count, node_y, ew, chirp, H,
                                          reinterpret_cast<double2 *>(pl->dft_scratch));
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bf_sht_forward(bfsht_plan *pl, const double *coeffs, double *grid, cudaStream_t st) {
    const int n = pl->n;
    int rc = bf_dft_prepare(pl, 4LL * n - 1);
    if (rc) return rc;
    dim3 g1((n + 255) / 256, 2 * n);
    coef_pack_kernel<<<g1, 256, 0, st>>>(n, pl->halves, reinterpret_cast<const double2 *>(coeffs),
                                         pl->arena, BF_NRHS);
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    rc = bf_alt_apply(pl, BFSHT_FORWARD, st);
    if (rc) return rc;
    return launch_synth(pl, pl->layout_fwd, pl->arena, 0, n, grid, pl->info[10],
                        2 * pl->norders, BF_NRHS, st);
}

int bf_sht_inverse(bfsht_plan *pl, const double *grid, double *coeffs, const double *weights,
                   cudaStream_t st) {
    const int n = pl->n;
    int rc = bf_dft_prepare(pl, 4LL * n - 1);
    if (rc) return rc;
    rc = launch_anal(pl, pl->layout_inv, pl->arena, 0, n, grid, weights, pl->node_y, BF_NRHS, st);
    if (rc) return rc;
    rc = bf_alt_apply(pl, BFSHT_INVERSE, st);
    if (rc) return rc;
    dim3 g1((n + 255) / 256, 2 * n);
    coef_unpack_kernel<<<g1, 256, 0, st>>>(n, pl->halves, pl->arena,
                                           reinterpret_cast<double2 *>(coeffs), BF_NRHS);
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bf_alt_orders(bfsht_plan *pl, int dir, const double *in, double *out, const double *weights,
                  cudaStream_t st) {
    const int n = pl->n, no = pl->norders;
    if (no == 0) return 0;
    dim3 g((n + 255) / 256, no);
    if (dir == BFSHT_FORWARD) {
        orders_pack_kernel<<<g, 256, 0, st>>>(n, pl->halves, pl->order_off,
                                              reinterpret_cast<const double2 *>(in), pl->arena);
        BF_CUDA(cudaGetLastError());
        int rc = bf_alt_apply(pl, dir, st);
        if (rc) return rc;
        orders_assemble_kernel<<<g, 256, 0, st>>>(n, pl->layout_fwd, pl->arena,
                                                  reinterpret_cast<double2 *>(out));
        BF_CUDA(cudaGetLastError());
    } else {
        orders_fold_kernel<<<g, 256, 0, st>>>(n, pl->halves, reinterpret_cast<const double2 *>(in),
                                              weights, pl->arena);
        BF_CUDA(cudaGetLastError());
        int rc = bf_alt_apply(pl, dir, st);
        if (rc) return rc;
        orders_unpack_kernel<<<g, 256, 0, st>>>(n, pl->halves, pl->order_off, pl->arena,
                                                reinterpret_cast<double2 *>(out));
        BF_CUDA(cudaGetLastError());
    }
    pl->launches += 2;
    return 0;
}

// ------------------------------------------------------------------------
// Batched fields (BASELINE config 4; SURVEY 8(b) "API extension"): F
// complex fields per order sharing one plan, field-minor rows — forward
// input (2N-m) x F and output 2N x F per order, plan after plan.  Pass p
// carries fields 8p .. 8p+7 as the 16 real RHS of a wide arena entry, so
// every DMMA uses its full n = 8 width and the payload is read once per 8
// fields instead of once per field.
namespace {

constexpr int kW = BF_WIDE_NRHS;
constexpr int kFPerPass = kW / 2;

__global__ void fields_pack_kernel(int F, int f0, const bf_half *__restrict__ halves,
                                   const int64_t *__restrict__ off, const double2 *__restrict__ in,
                                   double *__restrict__ arena, int ew) {
    const int o = blockIdx.y, f = threadIdx.x;
    const int j = blockIdx.x * blockDim.y + threadIdx.y;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        double2 v = make_double2(0.0, 0.0);
        if (f0 + f < F) v = in[(off[o] + (par == 0 ? 1 : 0) + 2 * (int64_t)j) * F + f0 + f];
        *reinterpret_cast<double2 *>(arena + ((int64_t)h.x + j) * ew + 2 * f) = v;
    }
}

__global__ void fields_assemble_kernel(int n, int F, int f0, const bf_half *__restrict__ layout,
                                       const double *__restrict__ arena, double2 *__restrict__ out,
                                       int ew) {
    const int o = blockIdx.y, f = threadIdx.x;
    const int r = blockIdx.x * blockDim.y + threadIdx.y;
    if (r >= n || f0 + f >= F) return;
    const bf_half ho = layout[2 * o], he = layout[2 * o + 1];
    double2 go = make_double2(0.0, 0.0), ge = go;
    if (ho.ncols > 0)
        go = *reinterpret_cast<const double2 *>(arena + ((int64_t)ho.y + (int64_t)r * ho.x) * ew + 2 * f);
    if (he.ncols > 0)
        ge = *reinterpret_cast<const double2 *>(arena + ((int64_t)he.y + (int64_t)r * he.x) * ew + 2 * f);
    double2 *col = out + (int64_t)o * 2 * n * F + f0 + f;
    col[(int64_t)(n + r) * F] = make_double2(ge.x + go.x, ge.y + go.y);
    col[(int64_t)(n - 1 - r) * F] = make_double2(ge.x - go.x, ge.y - go.y);
}

__global__ void fields_fold_kernel(int n, int F, int f0, const bf_half *__restrict__ halves,
                                   const double2 *__restrict__ in, const double *__restrict__ weights,
                                   double *__restrict__ arena, int ew) {
    const int o = blockIdx.y, f = threadIdx.x;
    const int r = blockIdx.x * blockDim.y + threadIdx.y;
    if (r >= n) return;
    double2 up = make_double2(0.0, 0.0), lo = up;
    if (f0 + f < F) {
        const double2 *col = in + (int64_t)o * 2 * n * F + f0 + f;
        up = col[(int64_t)(n + r) * F];
        lo = col[(int64_t)(n - 1 - r) * F];
    }
    const double w = weights[n + r];
    const bf_half ho = halves[2 * o], he = halves[2 * o + 1];
    if (ho.ncols > 0)
        *reinterpret_cast<double2 *>(arena + ((int64_t)ho.y + r) * ew + 2 * f) =
            make_double2(w * (up.x - lo.x), w * (up.y - lo.y));
    if (he.ncols > 0)
        *reinterpret_cast<double2 *>(arena + ((int64_t)he.y + r) * ew + 2 * f) =
            make_double2(w * (up.x + lo.x), w * (up.y + lo.y));
}

__global__ void fields_unpack_kernel(int F, int f0, const bf_half *__restrict__ halves,
                                     const int64_t *__restrict__ off,
                                     const double *__restrict__ arena, double2 *__restrict__ out,
                                     int ew) {
    const int o = blockIdx.y, f = threadIdx.x;
    const int j = blockIdx.x * blockDim.y + threadIdx.y;
    if (f0 + f >= F) return;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        out[(off[o] + (par == 0 ? 1 : 0) + 2 * (int64_t)j) * F + f0 + f] =
            *reinterpret_cast<const double2 *>(arena + ((int64_t)h.x + j) * ew + 2 * f);
    }
}

// Raw half apply (reference idbf_apply / _apply_half, butterfly.py:275-292,
// alt.py:197-222): real row-major in (len_in x k) -> out (len_out x k),
// columns c0 .. c0+15 of this pass.
__global__ void half_load_kernel(int64_t base, int64_t stride, int len, int k, int c0,
                                 const double *__restrict__ in, double *__restrict__ arena) {
    const int r = blockIdx.x * blockDim.y + threadIdx.y, c = threadIdx.x;
    if (r >= len) return;
    arena[(base + r * stride) * kW + c] = (c0 + c < k) ? in[(int64_t)r * k + c0 + c] : 0.0;
}

__global__ void half_store_kernel(int64_t base, int64_t stride, int len, int k, int c0,
                                  const double *__restrict__ arena, double *__restrict__ out) {
    const int r = blockIdx.x * blockDim.y + threadIdx.y, c = threadIdx.x;
    if (r >= len || c0 + c >= k) return;
    out[(int64_t)r * k + c0 + c] = arena[(base + r * stride) * kW + c];
}

}  // namespace

// More than 8 fields on a plan without regenerated tiles: passes of 32
// fields through the group engine (64-wide entries, bf_alt_apply_group);
// otherwise passes of 8 fields through the 16-wide warp engine.  Both give
// the same bits (per-field sums in the same order).  BFSHT_FIELDS_WIDE16=1
// forces the 8-field passes (A/B measurements).
int bf_alt_fields(bfsht_plan *pl, int dir, int F, const double *in, double *out,
                  const double *weights, double *work, cudaStream_t st) {
    const int n = pl->n, no = pl->norders;
    if (no == 0 || F == 0) return 0;
    static const bool force16 = std::getenv("BFSHT_FIELDS_WIDE16") != nullptr;
    const bool group = F > kFPerPass && pl->info[18] == 0 && !force16;
    const int ew = group ? BFSHT_FIELDS_NRHS : kW;
    const int fpp = ew / 2;
    const dim3 blk(fpp, 256 / fpp);
    const dim3 g((n + blk.y - 1) / blk.y, no);
    for (int f0 = 0; f0 < F; f0 += fpp) {
        auto apply = [&]() {
            return group ? bf_alt_apply_group(pl, dir, work, st) : bf_alt_apply_wide(pl, dir, work, st);
        };
        if (dir == BFSHT_FORWARD) {
            fields_pack_kernel<<<g, blk, 0, st>>>(F, f0, pl->halves, pl->order_off,
                                                  reinterpret_cast<const double2 *>(in), work, ew);
            BF_CUDA(cudaGetLastError());
            int rc = apply();
            if (rc) return rc;
            fields_assemble_kernel<<<g, blk, 0, st>>>(n, F, f0, pl->layout_fwd, work,
                                                      reinterpret_cast<double2 *>(out), ew);
            BF_CUDA(cudaGetLastError());
        } else {
            fields_fold_kernel<<<g, blk, 0, st>>>(n, F, f0, pl->halves,
                                                  reinterpret_cast<const double2 *>(in), weights,
                                                  work, ew);
            BF_CUDA(cudaGetLastError());
            int rc = apply();
            if (rc) return rc;
            fields_unpack_kernel<<<g, blk, 0, st>>>(F, f0, pl->halves, pl->order_off, work,
                                                    reinterpret_cast<double2 *>(out), ew);
            BF_CUDA(cudaGetLastError());
        }
        pl->launches += 2;
    }
    return 0;
}

int bf_half_apply(bfsht_plan *pl, int dir, int half, int k, const double *in, double *out,
                  double *work, cudaStream_t st) {
    const bf_half hf = pl->host_halves[half];
    const bf_half lay = pl->host_layout_fwd[half];
    // forward: columns in (x region), rows out (Yr: base lay.y, stride lay.x)
    // inverse: rows in (y region), columns out (x region)
    const int64_t in_base = dir == BFSHT_FORWARD ? hf.x : hf.y;
    const int64_t in_stride = 1;
    const int in_len = dir == BFSHT_FORWARD ? hf.ncols : pl->n;
    const int64_t out_base = dir == BFSHT_FORWARD ? lay.y : hf.x;
    const int64_t out_stride = dir == BFSHT_FORWARD ? lay.x : 1;
    const int out_len = dir == BFSHT_FORWARD ? pl->n : hf.ncols;
    const dim3 blk(kW, 16);
    for (int c0 = 0; c0 < k; c0 += kW) {
        half_load_kernel<<<(in_len + 15) / 16, blk, 0, st>>>(in_base, in_stride, in_len, k, c0, in,
                                                              work);
        BF_CUDA(cudaGetLastError());
        int rc = bf_alt_apply_wide(pl, dir, work, st);
        if (rc) return rc;
        half_store_kernel<<<(out_len + 15) / 16, blk, 0, st>>>(out_base, out_stride, out_len, k,
                                                                c0, work, out);
        BF_CUDA(cudaGetLastError());
        pl->launches += 2;
    }
    return 0;
}

// Batched SHT: B <= BF_WIDE_NRHS / BF_NRHS independent transforms share one
// pass of the 16-RHS engine over the payload; transform b owns doubles
// [4b, 4b + 4) of every wide arena entry, so packing, the DFT stage and
// unpacking are the single-transform kernels with entry width 16 and an
// offset.  Outputs are bitwise those of B single-transform calls.
int bf_sht_batch(bfsht_plan *pl, int dir, int B, const double *in, double *out,
                 const double *weights, double *work, cudaStream_t st) {
    const int n = pl->n;
    const int ew = BF_WIDE_NRHS;
    int rc = bf_dft_prepare(pl, 4LL * n - 1);
    if (rc) return rc;
    const int64_t L = pl->dft_L;
    const int64_t ncoef = 4LL * n * n, ngrid = 2LL * n * L;
    dim3 g1((n + 255) / 256, 2 * n);
    if (dir == BFSHT_FORWARD) {
        for (int b = 0; b < ew / BF_NRHS; ++b) {
            const double2 *src = b < B ? reinterpret_cast<const double2 *>(in) + b * ncoef : nullptr;
            coef_pack_kernel<<<g1, 256, 0, st>>>(n, pl->halves, src, work + BF_NRHS * b, ew);
            BF_CUDA(cudaGetLastError());
            pl->launches += 1;
        }
        rc = bf_alt_apply_wide(pl, BFSHT_FORWARD, work, st);
        if (rc) return rc;
        for (int b = 0; b < B; ++b) {
            rc = launch_synth(pl, pl->layout_fwd, work + BF_NRHS * b, 0, n, out + 2 * b * ngrid,
                              pl->info[10], 2 * pl->norders, ew, st);
            if (rc) return rc;
        }
    } else {
        for (int b = 0; b < B; ++b) {
            rc = launch_anal(pl, pl->layout_inv, work + BF_NRHS * b, 0, n, in + 2 * b * ngrid,
                             weights, pl->node_y, ew, st);
            if (rc) return rc;
        }
        rc = bf_alt_apply_wide(pl, BFSHT_INVERSE, work, st);
        if (rc) return rc;
        for (int b = 0; b < B; ++b) {
            coef_unpack_kernel<<<g1, 256, 0, st>>>(n, pl->halves, work + BF_NRHS * b,
                                                   reinterpret_cast<double2 *>(out) + b * ncoef, ew);
            BF_CUDA(cudaGetLastError());
            pl->launches += 1;
        }
    }
    return 0;
}

int bf_dft_rows(bfsht_plan *pl, int64_t L, int64_t rows, int dir, const double *in, double *out,
                cudaStream_t st) {
    int rc = bf_dft_prepare(pl, L);
    if (rc) return rc;
    const bool sm = dft_smem_bytes(pl->dft_Lb, 1) + pl->dft_gen <= 227 * 1024;
    int grid = (int)(rows < 4096 ? rows : 4096);
    if (!sm) grid = (int)std::min<int64_t>(grid, pl->dft_scratch_rows);
    if (grid <= 0) return 0;
    // kernels without the generic-radix code keep the smaller register
    // footprint (2 CTAs per SM) for the all-templated lengths
    auto kern = sm ? (pl->dft_gen ? dft_rows_kernel<true, true> : dft_rows_kernel<true, false>)
                   : (pl->dft_gen ? dft_rows_kernel<false, true> : dft_rows_kernel<false, false>);
    const int smem = sm ? dft_smem_bytes(pl->dft_Lb, 1) + pl->dft_gen : pl->dft_gen;
    rc = bf_ensure_smem((const void *)kern, smem);
    if (rc) return rc;
    kern<<<grid, kDftThreads, smem, st>>>(
        make_desc(pl), reinterpret_cast<const double2 *>(in), reinterpret_cast<double2 *>(out), rows,
        pl->dft_perm, reinterpret_cast<const double2 *>(pl->dft_w), dir == BFSHT_INVERSE, sm,
        reinterpret_cast<double2 *>(pl->dft_scratch), reinterpret_cast<const double2 *>(pl->dft_chirp), reinterpret_cast<const double2 *>(pl->dft_hhat));
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bf_synth_rows(bfsht_plan *pl, const bf_half *halves, const double *ybuf, int r_begin,
                  int r_count, double *grid, cudaStream_t st) {
    const int n = pl->n;
    int rc = bf_dft_prepare(pl, 4LL * n - 1);
    if (rc) return rc;
    if (r_count <= 0) return 0;
    return launch_synth(pl, halves, ybuf, r_begin, r_count, grid, 0, 0, BF_NRHS, st);
}

int bf_anal_rows(bfsht_plan *pl, const bf_half *halves, double *ubuf, int r_begin, int r_count,
                 const double *grid, const double *weights, cudaStream_t st) {
    const int n = pl->n;
    int rc = bf_dft_prepare(pl, 4LL * n - 1);
    if (rc) return rc;
    if (r_count <= 0) return 0;
    return launch_anal(pl, halves, ubuf, r_begin, r_count, grid, weights, nullptr, BF_NRHS, st);
}
