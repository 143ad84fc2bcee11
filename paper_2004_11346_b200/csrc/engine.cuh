// Device-side plan handle and launch helpers shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "bfsht_b200.h"
#include "format.h"

struct bfsht_plan {
    int64_t info[BFSHT_INFO_LEN];
    const double *tiles = nullptr;
    const bf_op *ops = nullptr;
    const int32_t *idx = nullptr;
    const int8_t *maps = nullptr;
    const bf_task *tasks = nullptr;
    const bf_half *halves = nullptr;
    const double *rec = nullptr;      // recurrence coefficients (regenerated tiles)
    const double *xpos = nullptr;     // positive nodes (regenerated tiles)
    // node-half addressing for the DFT stage: entry (order o, parity p, row r)
    // at layout[2o+p].y + r * layout[2o+p].x (fwd: row-major Yr; inv: halves)
    bf_half *layout_fwd = nullptr;
    bf_half *layout_inv = nullptr;
    std::vector<bf_half> host_halves, host_layout_fwd;   // host copies
    int *node_y = nullptr;            // device: node-half base per half, -1 absent
    double *arena = nullptr;
    std::vector<int64_t> stages[2];   // task bounds per stage (host)
    int32_t n = 0;                    // half size N
    int32_t norders = 0;
    std::vector<int32_t> orders;      // m of each plan (host)
    // owned device allocations (upload path) and scratch
    std::vector<void *> owned;
    int *counters = nullptr;          // one per stage launch (device)
    int ncounters = 0;
    // per-order API scratch
    int64_t *order_off = nullptr;     // device, 2*norders+2 offsets
    // DFT tables (built lazily for L = 4N-1)
    int64_t dft_L = 0;                // transform length
    int64_t dft_Lb = 0;               // row buffer length (L, or Bluestein M)
    bool dft_blue = false;            // Bluestein rows
    double *dft_chirp = nullptr;      // Bluestein: L complex exp(-i pi j^2/L)
    double *dft_hhat = nullptr;       // Bluestein: M complex FFT_M(conj chirp)/M
    double *dft_w = nullptr;          // pass twiddle table (L complex) + radix roots
    int32_t *dft_perm = nullptr;      // digit-reversal positions
    double *dft_tw = nullptr;         // L complex: exp(i m phi0) per bin
    std::vector<int32_t> dft_radix;
    int dft_gen = 0;                  // generic-radix staging bytes (dynamic smem tail)
    double *dft_scratch = nullptr;    // global fallback buffer
    int64_t dft_scratch_rows = 0;
    int64_t launches = 0;
    int sm_count = 148;
    int device = 0;                   // CUDA device the plan lives on
    // chain schedule (engine.cu, bf_chain_build): the stages made of small
    // butterfly / low-rank-core tasks re-encoded as 32-byte records in
    // cost-balanced bundles for alt_chain_kernel; nb == 0: the stage runs
    // on alt_stage_kernel
    struct ChainStage {
        int64_t b0 = 0;               // first entry of the stage in chain_bund
        int nb = 0;                   // bundles
        int64_t nrec = 0, nfold = 0;  // records, index adds folded into tile ops
    };
    std::vector<ChainStage> chain[2];
    void *chain_rec[2] = {nullptr, nullptr};        // device, per direction: bf_crec records
    int32_t *chain_bund[2] = {nullptr, nullptr};    // device: bundle bounds (record indices)
};

void bfsht_set_error(const std::string &msg);

// Raise the dynamic shared-memory limit of kernel `func` on the CURRENT
// device to at least `bytes` before a launch.  The attribute is per kernel
// and per device context, so a per-(device, kernel) high-water mark is
// kept: the limit only ever grows, and a launch never runs against a limit
// another plan (or another device) set lower.  Thread-safe.
int bf_ensure_smem(const void *func, int bytes);

// Every entry point that takes a plan runs on the plan's device and leaves
// the caller's current device as it found it.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const bfsht_plan *pl) {
        if (!pl) return;
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != pl->device) {
            prev = cur;
            cudaSetDevice(pl->device);
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

#define BF_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) {                                               \
            bfsht_set_error(std::string(#call) + ": " + cudaGetErrorString(_e)); \
            return -2;                                                         \
        }                                                                      \
    } while (0)

// engine.cu
int bf_run_stage(bfsht_plan *pl, int dir, int stage, cudaStream_t s);
// Build the chain schedule from host copies of the plan's ops and tasks
// (called once when the plan is created; without it every stage runs on
// alt_stage_kernel).
int bf_chain_build(bfsht_plan *pl, const bf_op *ops, const bf_task *tasks);
int bf_alt_apply(bfsht_plan *pl, int dir, cudaStream_t s);
int bf_alt_apply_wide(bfsht_plan *pl, int dir, double *arena, cudaStream_t s);
int bf_alt_apply_group(bfsht_plan *pl, int dir, double *arena, cudaStream_t s);
int bf_alt_fields(bfsht_plan *pl, int dir, int F, const double *in, double *out,
                  const double *weights, double *work, cudaStream_t st);
int bf_sht_batch(bfsht_plan *pl, int dir, int B, const double *in, double *out,
                 const double *weights, double *work, cudaStream_t st);
int bf_half_apply(bfsht_plan *pl, int dir, int half, int k, const double *in, double *out,
                  double *work, cudaStream_t st);
// sht.cu
int bf_dft_prepare(bfsht_plan *pl, int64_t L);
