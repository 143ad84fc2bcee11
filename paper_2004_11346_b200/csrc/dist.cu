// Multi-GPU pieces of the SHT: order-sharded coefficient packing and the
// entry gather/scatter around the NCCL all-to-all that transposes node
// halves between the m-major ALT stage and the theta-major DFT stage.
//
// The reference is single-process (no distributed execution);
// the sharding follows its independence structure: each order's plan is
// used only by +m and -m (pkg/src/bfsht/sht.py:146,165), and each
// colatitude row's DFT needs every order (sht.py:148,161).
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.cuh"

int bf_synth_rows(bfsht_plan *pl, const bf_half *halves, const double *ybuf, int r_begin,
                  int r_count, double *grid, cudaStream_t st);
int bf_anal_rows(bfsht_plan *pl, const bf_half *halves, double *ubuf, int r_begin, int r_count,
                 const double *grid, const double *weights, cudaStream_t st);

namespace {

// Shard coefficient layout: for each plan order o (|m| = m_o) the +m vector
// (2N - m_o values, k ascending) at off[o], then the -m vector (m_o > 0).
__global__ void shard_pack_kernel(int n, const bf_half *__restrict__ halves,
                                  const int64_t *__restrict__ off,
                                  const double2 *__restrict__ c, double *__restrict__ arena) {
    const int o = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = halves[2 * o].m;
    const int64_t len = 2 * (int64_t)n - m;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        const int k = (par == 0 ? 1 : 0) + 2 * j;
        const double2 p = c[off[o] + k];
        const double2 q = m ? c[off[o] + len + k] : make_double2(0.0, 0.0);
        double *e = arena + ((int64_t)h.x + j) * BF_NRHS;
        *reinterpret_cast<double2 *>(e) = p;
        *reinterpret_cast<double2 *>(e + 2) = q;
    }
}

__global__ void shard_unpack_kernel(int n, const bf_half *__restrict__ halves,
                                    const int64_t *__restrict__ off,
                                    const double *__restrict__ arena, double2 *__restrict__ c) {
    const int o = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int m = halves[2 * o].m;
    const int64_t len = 2 * (int64_t)n - m;
    for (int par = 0; par < 2; ++par) {
        const bf_half h = halves[2 * o + par];
        if (j >= h.ncols) continue;
        const int k = (par == 0 ? 1 : 0) + 2 * j;
        const double *e = arena + ((int64_t)h.x + j) * BF_NRHS;
        c[off[o] + k] = *reinterpret_cast<const double2 *>(e);
        if (m) c[off[o] + len + k] = *reinterpret_cast<const double2 *>(e + 2);
    }
}

// out[i] = arena[idx[i]] (one 4-double entry per index)
__global__ void gather_entries_kernel(const double4 *__restrict__ arena,
                                      const int32_t *__restrict__ idx, int64_t count,
                                      double4 *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = arena[idx[i]];
}

__global__ void scatter_entries_kernel(double4 *__restrict__ arena,
                                       const int32_t *__restrict__ idx, int64_t count,
                                       const double4 *__restrict__ in) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = idx[i];
        if (t >= 0) arena[t] = in[i];   // -1: absent half, nothing to write
    }
}

int grid_for(int64_t count) {
    int64_t b = (count + 255) / 256;
    return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace

int bf_shard_pack(bfsht_plan *pl, const int64_t *off, const double *coeffs, cudaStream_t st) {
    if (pl->norders == 0) return 0;
    dim3 g((pl->n + 255) / 256, pl->norders);
    shard_pack_kernel<<<g, 256, 0, st>>>(pl->n, pl->halves, off,
                                         reinterpret_cast<const double2 *>(coeffs), pl->arena);
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bf_shard_unpack(bfsht_plan *pl, const int64_t *off, double *coeffs, cudaStream_t st) {
    if (pl->norders == 0) return 0;
    dim3 g((pl->n + 255) / 256, pl->norders);
    shard_unpack_kernel<<<g, 256, 0, st>>>(pl->n, pl->halves, off, pl->arena,
                                           reinterpret_cast<double2 *>(coeffs));
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

extern "C" {

int bfsht_shard_pack(bfsht_plan *pl, const int64_t *off, const double *coeffs, void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    return bf_shard_pack(pl, off, coeffs, (cudaStream_t)stream);
}

int bfsht_shard_unpack(bfsht_plan *pl, const int64_t *off, double *coeffs, void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    return bf_shard_unpack(pl, off, coeffs, (cudaStream_t)stream);
}

int bfsht_gather_entries(bfsht_plan *pl, const int32_t *idx, int64_t count, double *out,
                         void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    if (count <= 0) return 0;
    gather_entries_kernel<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const double4 *>(pl->arena), idx, count,
        reinterpret_cast<double4 *>(out));
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bfsht_scatter_entries(bfsht_plan *pl, const int32_t *idx, int64_t count, const double *in,
                          void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    if (count <= 0) return 0;
    scatter_entries_kernel<<<grid_for(count), 256, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<double4 *>(pl->arena), idx, count,
        reinterpret_cast<const double4 *>(in));
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bfsht_synth_rows(bfsht_plan *pl, const void *halves, const double *ybuf, int64_t r_begin,
                     int64_t r_count, double *grid, void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    return bf_synth_rows(pl, (const bf_half *)halves, ybuf, (int)r_begin, (int)r_count, grid,
                         (cudaStream_t)stream);
}

int bfsht_anal_rows(bfsht_plan *pl, const void *halves, double *ubuf, int64_t r_begin,
                    int64_t r_count, const double *grid, const double *weights, void *stream) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    return bf_anal_rows(pl, (const bf_half *)halves, ubuf, (int)r_begin, (int)r_count, grid,
                        weights, (cudaStream_t)stream);
}

int bfsht_reset_launches(bfsht_plan *pl) {
    DeviceGuard guard(pl);
    if (!pl) return -1;
    pl->launches = 0;
    return 0;
}

}  // extern "C"
