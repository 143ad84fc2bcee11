// Device-side entry evaluation for factor construction.
//
// The reference planner evaluates ALT matrix entries through its entry
// oracle: the normalized associated Legendre degree recurrence run per node
// from checkpointed states (pkg/src/bfsht/partition.py:91-169 over
// kernels/_recur_cy.pyx:18-67).  The host planner here tabulates each
// order-m parity half once with the same recurrence (csrc/recur.c); this
// file moves that tabulation onto the GPU.  One thread per node runs the
// degree chain with the shared step of recur.h (__dmul_rn / __dsub_rn, no
// FMA contraction, exact 2^-+1000 rescales), so every entry is bitwise the
// host table's, and the factors the planner builds from it keep the
// reference plan digests.  The table is written column-major (entry (r, j)
// at j * n + r): consecutive threads store consecutive addresses, and the
// planner only reads the table through copies, which are layout-blind
// (tests/test_planner.py passes on the transposed table too).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <mutex>
#include <map>

#include "engine.cuh"
#include "recur.h"

namespace {

__device__ __forceinline__ double emit_entry(double p, int e, double mag_min) {
    const double v = ldexp(p, e);   // exact: results below mag_min are flushed
    return fabs(v) < mag_min ? 0.0 : v;
}

__global__ void half_table_kernel(int64_t m, int64_t offset, int n, int64_t ncols,
                                  const double *__restrict__ x, const double *__restrict__ alpha,
                                  const double *__restrict__ beta,
                                  const double *__restrict__ mant0,
                                  const int32_t *__restrict__ exp0, double mag_min,
                                  double *__restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double xr = x[r];
    double pp = 0.0, pc = mant0[r];
    int e = exp0[r];
    const int64_t k_first = m + offset, k_last = m + offset + 2 * (ncols - 1);
    int64_t j = 0;
    if (k_first == m) out[(j++) * n + r] = emit_entry(pc, e, mag_min);
    for (int64_t k = m; k < k_last; ++k) {
        const int64_t s = k - m;
        bfr_step(xr, __ldg(alpha + s), __ldg(beta + s), &pp, &pc, &e);
        if (j < ncols && k + 1 == k_first + 2 * j) out[(j++) * n + r] = emit_entry(pc, e, mag_min);
    }
}

// per-device workspace, grown on demand (plan-time only)
struct Workspace {
    void *buf = nullptr;
    size_t bytes = 0;
    cudaStream_t st = nullptr;
};

}  // namespace

extern "C" int bfsht_half_table_device(int device, int64_t m, int64_t offset, int64_t n,
                                       int64_t ncols, const double *x, const double *alpha,
                                       const double *beta, const double *mant0,
                                       const int32_t *exp0, double mag_min, double *out) {
    if (n <= 0 || ncols <= 0) return 0;
    if (n > (1 << 30) || m < 0 || offset < 0 || offset > 1) {
        bfsht_set_error("bfsht_half_table_device: bad sizes");
        return -1;
    }
    static std::mutex mu;
    static std::map<int, Workspace> ws_by_dev;
    std::lock_guard<std::mutex> lock(mu);
    int prev = -1;
    BF_CUDA(cudaGetDevice(&prev));
    if (prev != device) BF_CUDA(cudaSetDevice(device));
    struct Restore {
        int d;
        ~Restore() {
            if (d >= 0) cudaSetDevice(d);
        }
    } restore{prev != device ? prev : -1};
    Workspace &ws = ws_by_dev[device];
    if (!ws.st) BF_CUDA(cudaStreamCreateWithFlags(&ws.st, cudaStreamNonBlocking));
    const int64_t nsteps = offset + 2 * (ncols - 1);   // alpha / beta entries used
    const size_t b_out = sizeof(double) * (size_t)(n * ncols);
    const size_t b_x = sizeof(double) * (size_t)n;
    const size_t b_ab = sizeof(double) * (size_t)(nsteps > 0 ? nsteps : 1);
    const size_t b_e = sizeof(int32_t) * (size_t)n;
    auto up = [](size_t v) { return (v + 255) / 256 * 256; };
    const size_t need = up(b_out) + 2 * up(b_x) + 2 * up(b_ab) + up(b_e);
    if (need > ws.bytes) {
        if (ws.buf) cudaFree(ws.buf);
        ws.buf = nullptr;
        ws.bytes = 0;
        BF_CUDA(cudaMalloc(&ws.buf, need));
        ws.bytes = need;
    }
    char *p = static_cast<char *>(ws.buf);
    double *d_out = reinterpret_cast<double *>(p);
    p += up(b_out);
    double *d_x = reinterpret_cast<double *>(p);
    p += up(b_x);
    double *d_m = reinterpret_cast<double *>(p);
    p += up(b_x);
    double *d_a = reinterpret_cast<double *>(p);
    p += up(b_ab);
    double *d_b = reinterpret_cast<double *>(p);
    p += up(b_ab);
    int32_t *d_e = reinterpret_cast<int32_t *>(p);
    BF_CUDA(cudaMemcpyAsync(d_x, x, b_x, cudaMemcpyHostToDevice, ws.st));
    BF_CUDA(cudaMemcpyAsync(d_m, mant0, b_x, cudaMemcpyHostToDevice, ws.st));
    BF_CUDA(cudaMemcpyAsync(d_e, exp0, b_e, cudaMemcpyHostToDevice, ws.st));
    if (nsteps > 0) {
        BF_CUDA(cudaMemcpyAsync(d_a, alpha, sizeof(double) * nsteps, cudaMemcpyHostToDevice, ws.st));
        BF_CUDA(cudaMemcpyAsync(d_b, beta, sizeof(double) * nsteps, cudaMemcpyHostToDevice, ws.st));
    }
    const int threads = 128;
    half_table_kernel<<<(int)((n + threads - 1) / threads), threads, 0, ws.st>>>(
        m, offset, (int)n, ncols, d_x, d_a, d_b, d_m, d_e, mag_min, d_out);
    BF_CUDA(cudaGetLastError());
    BF_CUDA(cudaMemcpyAsync(out, d_out, b_out, cudaMemcpyDeviceToHost, ws.st));
    BF_CUDA(cudaStreamSynchronize(ws.st));
    return 0;
}
