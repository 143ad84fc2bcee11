// extern "C" entry points of libbfsht_b200.so (declared in
// include/bfsht_b200.h).  Plain pointers and sizes; no torch types.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "bfsht_b200.h"
#include "engine.cuh"

static thread_local std::string g_err;

void bfsht_set_error(const std::string &msg) { g_err = msg; }

int bf_ensure_smem(const void *func, int bytes) {
    if (bytes <= 48 * 1024) return 0;
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> high;
    int dev = 0;
    BF_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    int &h = high[{dev, func}];
    if (bytes <= h) return 0;
    BF_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    h = bytes;
    return 0;
}

int bf_sht_forward(bfsht_plan *pl, const double *coeffs, double *grid, cudaStream_t st);
int bf_sht_inverse(bfsht_plan *pl, const double *grid, double *coeffs, const double *weights,
                   cudaStream_t st);
int bf_alt_orders(bfsht_plan *pl, int dir, const double *in, double *out, const double *weights,
                  cudaStream_t st);
int bf_dft_rows(bfsht_plan *pl, int64_t L, int64_t rows, int dir, const double *in, double *out,
                cudaStream_t st);

namespace {

int finish_plan(bfsht_plan *pl, const bf_half *host_halves, const int64_t *sf,
                const int64_t *si, const bf_op *host_ops, const bf_task *host_tasks) {
    const int64_t nh = pl->info[6];
    pl->stages[0].assign(sf, sf + pl->info[7] + 1);
    pl->stages[1].assign(si, si + pl->info[8] + 1);
    pl->norders = (int32_t)(nh / 2);
    pl->n = (int32_t)pl->info[14];
    pl->orders.resize(pl->norders);
    std::vector<int64_t> off(pl->norders + 1, 0);
    for (int o = 0; o < pl->norders; ++o) {
        pl->orders[o] = host_halves[2 * o].m;
        off[o + 1] = off[o] + 2 * (int64_t)pl->n - pl->orders[o];
    }
    BF_CUDA(cudaMalloc(&pl->order_off, sizeof(int64_t) * (pl->norders + 1)));
    pl->owned.push_back(pl->order_off);
    BF_CUDA(cudaMemcpy(pl->order_off, off.data(), sizeof(int64_t) * (pl->norders + 1),
                       cudaMemcpyHostToDevice));
    // DFT-stage addressing of node halves (see engine.cuh)
    {
        std::vector<bf_half> lf(nh), li(nh);
        const int32_t stride = 2 * pl->norders;
        for (int64_t h = 0; h < nh; ++h) {
            lf[h] = li[h] = host_halves[h];
            lf[h].x = stride;
            lf[h].y = (int32_t)pl->info[10] + (int32_t)h;
            li[h].x = 1;
        }
        pl->host_halves.assign(host_halves, host_halves + nh);
        std::vector<int> ny(nh ? nh : 1, -1);
        for (int64_t h = 0; h < nh; ++h) ny[h] = host_halves[h].ncols > 0 ? host_halves[h].y : -1;
        BF_CUDA(cudaMalloc(&pl->node_y, sizeof(int) * ny.size()));
        pl->owned.push_back(pl->node_y);
        BF_CUDA(cudaMemcpy(pl->node_y, ny.data(), sizeof(int) * ny.size(), cudaMemcpyHostToDevice));
        pl->host_layout_fwd = lf;
        BF_CUDA(cudaMalloc(&pl->layout_fwd, sizeof(bf_half) * (nh ? nh : 1)));
        pl->owned.push_back(pl->layout_fwd);
        BF_CUDA(cudaMalloc(&pl->layout_inv, sizeof(bf_half) * (nh ? nh : 1)));
        pl->owned.push_back(pl->layout_inv);
        if (nh) {
            BF_CUDA(cudaMemcpy(pl->layout_fwd, lf.data(), sizeof(bf_half) * nh,
                               cudaMemcpyHostToDevice));
            BF_CUDA(cudaMemcpy(pl->layout_inv, li.data(), sizeof(bf_half) * nh,
                               cudaMemcpyHostToDevice));
        }
    }
    pl->ncounters = (int)std::max(pl->info[7], pl->info[8]) + 1;
    BF_CUDA(cudaMalloc(&pl->counters, sizeof(int) * pl->ncounters));
    pl->owned.push_back(pl->counters);
    int dev = 0;
    BF_CUDA(cudaGetDevice(&dev));
    pl->device = dev;
    BF_CUDA(cudaDeviceGetAttribute(&pl->sm_count, cudaDevAttrMultiProcessorCount, dev));
    return bf_chain_build(pl, host_ops, host_tasks);
}

}  // namespace

extern "C" {

const char *bfsht_last_error(void) { return g_err.c_str(); }

int bfsht_plan_upload(const bfsht_packed *p, bfsht_plan **out) {
    if (!p || !out) {
        g_err = "null argument";
        return -1;
    }
    auto *pl = new bfsht_plan();
    if (bfsht_packed_info(p, pl->info)) {
        delete pl;
        g_err = "bad packed plan";
        return -1;
    }
    const void *arr[12];
    bfsht_packed_arrays(p, arr);
    // device copies of arrays 0..5 and 8..9 (stage bounds stay on the host)
    const int which[8] = {0, 1, 2, 3, 4, 5, 8, 9};
    const size_t sz[8] = {(size_t)pl->info[0] * 8, (size_t)pl->info[1] * sizeof(bf_op),
                          (size_t)pl->info[2] * 4, (size_t)pl->info[3] * BF_SLOTS,
                          (size_t)pl->info[4] * sizeof(bf_task),
                          (size_t)pl->info[6] * sizeof(bf_half),
                          (size_t)pl->info[20] * 8, (size_t)pl->info[21] * 8};
    void *dev[8];
    for (int i = 0; i < 8; ++i) {
        dev[i] = nullptr;
        if (cudaMalloc(&dev[i], sz[i] ? sz[i] : 16) != cudaSuccess ||
            (sz[i] && cudaMemcpy(dev[i], arr[which[i]], sz[i], cudaMemcpyHostToDevice) != cudaSuccess)) {
            g_err = "device allocation/copy failed";
            for (int j = 0; j <= i; ++j) cudaFree(dev[j]);
            delete pl;
            return -2;
        }
        pl->owned.push_back(dev[i]);
    }
    void *arena = nullptr;
    if (cudaMalloc(&arena, (size_t)pl->info[5] * BF_NRHS * 8 + 16) != cudaSuccess) {
        g_err = "arena allocation failed";
        bfsht_plan_free(pl);
        return -2;
    }
    pl->owned.push_back(arena);
    // zeroed: absent halves' entries of the node array Yr are read as zeros
    if (cudaMemset(arena, 0, (size_t)pl->info[5] * BF_NRHS * 8 + 16) != cudaSuccess) {
        g_err = "arena clear failed";
        bfsht_plan_free(pl);
        return -2;
    }
    pl->tiles = (const double *)dev[0];
    pl->ops = (const bf_op *)dev[1];
    pl->idx = (const int32_t *)dev[2];
    pl->maps = (const int8_t *)dev[3];
    pl->tasks = (const bf_task *)dev[4];
    pl->halves = (const bf_half *)dev[5];
    pl->rec = (const double *)dev[6];
    pl->xpos = (const double *)dev[7];
    pl->arena = (double *)arena;
    int rc = finish_plan(pl, (const bf_half *)arr[5], (const int64_t *)arr[6],
                         (const int64_t *)arr[7], (const bf_op *)arr[1], (const bf_task *)arr[4]);
    if (rc) {
        bfsht_plan_free(pl);
        return rc;
    }
    *out = pl;
    return 0;
}

int bfsht_plan_wrap(const int64_t info[BFSHT_INFO_LEN], const void *const host[8],
                    void *const dev[12], bfsht_plan **out) {
    if (!info || !host || !dev || !out) {
        g_err = "null argument";
        return -1;
    }
    auto *pl = new bfsht_plan();
    std::memcpy(pl->info, info, sizeof(pl->info));
    pl->tiles = (const double *)dev[0];
    pl->ops = (const bf_op *)dev[1];
    pl->idx = (const int32_t *)dev[2];
    pl->maps = (const int8_t *)dev[3];
    pl->tasks = (const bf_task *)dev[4];
    pl->halves = (const bf_half *)dev[5];
    pl->arena = (double *)dev[6];
    pl->rec = (const double *)dev[7];
    pl->xpos = (const double *)dev[8];
    if (info[18] > 0 && (!pl->rec || !pl->xpos)) {
        delete pl;
        g_err = "plan has regenerated tiles but no coefficient table / nodes";
        return -1;
    }
    int rc = finish_plan(pl, (const bf_half *)host[5], (const int64_t *)host[6],
                         (const int64_t *)host[7], (const bf_op *)host[1],
                         (const bf_task *)host[4]);
    if (rc) {
        bfsht_plan_free(pl);
        return rc;
    }
    *out = pl;
    return 0;
}

void bfsht_plan_free(bfsht_plan *pl) {
    if (!pl) return;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != pl->device) cudaSetDevice(pl->device);
    for (void *p : pl->owned) cudaFree(p);
    for (void *p : {(void *)pl->dft_w, (void *)pl->dft_perm, (void *)pl->dft_tw,
                    (void *)pl->dft_scratch, (void *)pl->dft_chirp, (void *)pl->dft_hhat})
        if (p) cudaFree(p);
    if (cur != pl->device) cudaSetDevice(cur);
    delete pl;
}

double *bfsht_plan_arena(bfsht_plan *pl) { return pl ? pl->arena : nullptr; }

int64_t bfsht_plan_launches(bfsht_plan *pl) { return pl ? pl->launches : -1; }

int bfsht_alt_apply(bfsht_plan *pl, int dir, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan or direction";
        return -1;
    }

    return bf_alt_apply(pl, dir, (cudaStream_t)stream);
}

int bfsht_alt_stage(bfsht_plan *pl, int dir, int stage, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan or direction";
        return -1;
    }
    const std::vector<int64_t> &b = pl->stages[dir];
    if (stage < 0 || stage + 1 >= (int)b.size()) {
        g_err = "stage out of range";
        return -1;
    }
    return bf_run_stage(pl, dir, stage, (cudaStream_t)stream);
}

int bfsht_plan_chain_info(bfsht_plan *pl, int dir, int stage, int64_t out[3]) {
    if (!pl || !out || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan, direction or output";
        return -1;
    }
    out[0] = out[1] = out[2] = 0;
    if (stage < 0 || stage + 1 >= (int)pl->stages[dir].size()) {
        g_err = "stage out of range";
        return -1;
    }
    if (stage < (int)pl->chain[dir].size()) {
        out[0] = pl->chain[dir][stage].nb;
        out[1] = pl->chain[dir][stage].nrec;
        out[2] = pl->chain[dir][stage].nfold;
    }
    return 0;
}

int bfsht_alt_orders(bfsht_plan *pl, int dir, const double *in, double *out,
                     const double *weights, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan or direction";
        return -1;
    }
    if (dir == BFSHT_INVERSE && !weights) {
        g_err = "inverse ALT needs quadrature weights";
        return -1;
    }

    return bf_alt_orders(pl, dir, in, out, weights, (cudaStream_t)stream);
}

int bfsht_alt_fields(bfsht_plan *pl, int dir, int nfields, const double *in, double *out,
                     const double *weights, double *work, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan or direction";
        return -1;
    }
    if (nfields < 0 || (nfields > 0 && (!in || !out || !work))) {
        g_err = "bad field count or null buffer";
        return -1;
    }
    if (dir == BFSHT_INVERSE && !weights) {
        g_err = "inverse ALT needs quadrature weights";
        return -1;
    }
    return bf_alt_fields(pl, dir, nfields, in, out, weights, work, (cudaStream_t)stream);
}

int bfsht_half_apply(bfsht_plan *pl, int dir, int half, int k, const double *in, double *out,
                     double *work, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan or direction";
        return -1;
    }
    if (half < 0 || half >= (int)pl->host_halves.size() || pl->host_halves[half].ncols <= 0) {
        g_err = "half out of range or absent";
        return -1;
    }
    if (k < 0 || (k > 0 && (!in || !out || !work))) {
        g_err = "bad column count or null buffer";
        return -1;
    }
    if (k == 0) return 0;
    return bf_half_apply(pl, dir, half, k, in, out, work, (cudaStream_t)stream);
}

static int check_sht(bfsht_plan *pl) {
    if (!pl) {
        g_err = "null plan";
        return -1;
    }
    if (pl->norders != 2 * pl->n) {
        g_err = "SHT needs plans for every order m = 0..2N-1";
        return -1;
    }
    for (int o = 0; o < pl->norders; ++o)
        if (pl->orders[o] != o) {
            g_err = "SHT plans must be ordered by m";
            return -1;
        }
    return 0;
}

int bfsht_alt_apply_wide(bfsht_plan *pl, int dir, double *work, void *stream) {
    DeviceGuard guard(pl);
    if (!pl || !work || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad plan, direction or work arena";
        return -1;
    }
    return bf_alt_apply_wide(pl, dir, work, (cudaStream_t)stream);
}

int bfsht_sht_batch(bfsht_plan *pl, int dir, int batch, const double *in, double *out,
                    const double *weights, double *work, void *stream) {
    DeviceGuard guard(pl);
    int rc = check_sht(pl);
    if (rc) return rc;
    if (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE) {
        g_err = "bad direction";
        return -1;
    }
    if (batch < 1 || batch > BFSHT_WIDE_NRHS / 4 || !in || !out || !work) {
        g_err = "batch must be 1..4 with device buffers and a wide work arena";
        return -1;
    }
    if (dir == BFSHT_INVERSE && !weights) {
        g_err = "inverse SHT needs quadrature weights";
        return -1;
    }
    return bf_sht_batch(pl, dir, batch, in, out, weights, work, (cudaStream_t)stream);
}

int bfsht_sht_forward(bfsht_plan *pl, const double *coeffs, double *grid, void *stream) {
    DeviceGuard guard(pl);
    if (check_sht(pl)) return -1;

    return bf_sht_forward(pl, coeffs, grid, (cudaStream_t)stream);
}

int bfsht_sht_inverse(bfsht_plan *pl, const double *grid, double *coeffs,
                      const double *weights, void *stream) {
    DeviceGuard guard(pl);
    if (check_sht(pl)) return -1;
    if (!weights) {
        g_err = "inverse SHT needs quadrature weights";
        return -1;
    }

    return bf_sht_inverse(pl, grid, coeffs, weights, (cudaStream_t)stream);
}

int bfsht_dft_rows(int64_t L, int64_t rows, int dir, const double *in, double *out,
                   void *stream) {
    if (L < 1 || rows < 0 || (dir != BFSHT_FORWARD && dir != BFSHT_INVERSE)) {
        g_err = "bad DFT arguments";
        return -1;
    }
    // DFT tables live in a per-(thread, device) context plan that keeps the
    // tables of the last length used (re-prepared, old tables freed, when
    // the length changes); it is freed with the thread
    struct Ctx {
        std::map<int, bfsht_plan *> by_dev;
        ~Ctx() {
            for (auto &kv : by_dev) bfsht_plan_free(kv.second);
        }
    };
    static thread_local Ctx ctx;
    int dev = 0;
    BF_CUDA(cudaGetDevice(&dev));
    bfsht_plan *&pl = ctx.by_dev[dev];
    if (!pl) {
        pl = new bfsht_plan();
        pl->device = dev;
        BF_CUDA(cudaDeviceGetAttribute(&pl->sm_count, cudaDevAttrMultiProcessorCount, dev));
    }
    return bf_dft_rows(pl, L, rows, dir, in, out, (cudaStream_t)stream);
}

}  // extern "C"
