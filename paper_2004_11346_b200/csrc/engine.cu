// ALT apply engine: persistent warp-task kernel over the packed tile store.
//
// Replaces the reference's per-order Python block loop
// (pkg/src/bfsht/alt.py:197-222) with its per-payload BLAS/scipy calls
// (butterfly.py:275-292, lowrank.py:196-202, alt.py:207,221) by one launch
// per dependency stage, covering every order of the plan at once.
//
// Execution model (sm_100a):
//  * grid = one CTA per SM, 8 warps per CTA; every warp is an independent
//    worker that claims tasks from a global counter (tasks are pre-sorted by
//    cost, so this is longest-first list scheduling).
//  * a task accumulates <= 32 output entries x 4 RHS in registers (lane =
//    output entry) over its ops, then stores them once: no atomics, fixed
//    summation order, bitwise-reproducible results.
//  * each warp owns a 3-slot shared-memory ring.  Lane 0 streams the next
//    ops' tiles (and contiguous input vectors) with 1-D TMA bulk copies
//    (cp.async.bulk ... mbarrier::complete_tx), all lanes gather indexed
//    input entries with cp.async into the same slot, and the slot's
//    mbarrier completes when both have landed.  Payload bytes are read from
//    HBM exactly once per direction; all reuse (4 RHS per value) is from
//    shared memory, conflict-free thanks to the rotated tile layout.
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.cuh"

namespace {

constexpr int kWarps = 8;
constexpr int kStages = 3;
constexpr int kTileDoubles = BF_T * BF_T;
constexpr int kVecDoubles = BF_T * BF_NRHS;

struct alignas(128) WarpRing {
    double tile[kStages][kTileDoubles];
    double vec[kStages][kVecDoubles];
    unsigned long long full[kStages];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}

__device__ __forceinline__ void cp_async_arrive(unsigned long long *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct StageArgs {
    const double *tiles;
    const bf_op *ops;
    const int32_t *idx;
    const int8_t *maps;
    const bf_task *tasks;
    double *arena;
    int64_t t0, ntasks;
    int *counter;
};

// Issue the loads of one op into ring slot `s` (whole warp).
__device__ __forceinline__ void issue_op(const StageArgs &a, WarpRing &ring, int s,
                                         const bf_op &op, int lane) {
    const double *arena = a.arena;
    uint32_t bytes = 0;
    int nvec = 0;
    bool gather = (op.flags & BF_OPF_GATHER) != 0;
    if (op.kind == BF_OP_ADD) {
        // entries for lanes [off, off+R)
        int j = lane - op.off;
        if (j >= 0 && j < op.R) {
            int src = gather ? __ldg(a.idx + op.in + j) : op.in + j;
            if (src >= 0) {
                const double *g = arena + (int64_t)src * BF_NRHS;
                cp_async16(&ring.vec[s][lane * BF_NRHS], g);
                cp_async16(&ring.vec[s][lane * BF_NRHS + 2], g + 2);
            }
        }
    } else {
        nvec = (op.kind == BF_OP_TILE_N) ? op.C : op.R;
        bytes = (((uint32_t)op.R * op.C * 8u) + 15u) & ~15u;
        if (gather) {
            if (lane < nvec) {
                int src = __ldg(a.idx + op.in + lane);
                const double *g = arena + (int64_t)src * BF_NRHS;
                cp_async16(&ring.vec[s][lane * BF_NRHS], g);
                cp_async16(&ring.vec[s][lane * BF_NRHS + 2], g + 2);
            }
        } else {
            bytes += (uint32_t)nvec * BF_NRHS * 8u;
        }
    }
    cp_async_arrive(&ring.full[s]);
    if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_tx(&ring.full[s], bytes);
        if (op.kind != BF_OP_ADD) {
            uint32_t tb = (((uint32_t)op.R * op.C * 8u) + 15u) & ~15u;
            bulk_g2s(ring.tile[s], a.tiles + op.tile, tb, &ring.full[s]);
            if (!gather)
                bulk_g2s(ring.vec[s], arena + (int64_t)op.in * BF_NRHS,
                         (uint32_t)nvec * BF_NRHS * 8u, &ring.full[s]);
        }
    }
}

__device__ __forceinline__ bf_op load_op(const bf_op *p) {
    // 24-byte record, 8-byte aligned: three 8-byte loads
    bf_op o;
    const int2 *q = reinterpret_cast<const int2 *>(p);
    int2 *d = reinterpret_cast<int2 *>(&o);
    d[0] = __ldg(q);
    d[1] = __ldg(q + 1);
    d[2] = __ldg(q + 2);
    return o;
}

__global__ void __launch_bounds__(kWarps * 32, 1) alt_stage_kernel(StageArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpRing &ring = reinterpret_cast<WarpRing *>(smem_raw)[warp];
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&ring.full[s], 33);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t seq_issue = 0, seq_use = 0;

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(a.counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= a.ntasks) break;
        const bf_task task = a.tasks[a.t0 + t];
        const bf_op *ops = a.ops + task.op_begin;
        const int nops = task.op_count;
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;

        int issued = 0;
        for (; issued < nops && issued < kStages; ++issued) {
            bf_op op = load_op(ops + issued);
            issue_op(a, ring, seq_issue % kStages, op, lane);
            ++seq_issue;
        }
        for (int i = 0; i < nops; ++i) {
            const int s = seq_use % kStages;
            mbar_wait(&ring.full[s], (seq_use / kStages) & 1u);
            ++seq_use;
            const bf_op op = load_op(ops + i);
            const double *T = ring.tile[s];
            const double *V = ring.vec[s];
            if (op.kind == BF_OP_ADD) {
                int j = lane - op.off;
                if (j >= 0 && j < op.R) {
                    int src = (op.flags & BF_OPF_GATHER) ? __ldg(a.idx + op.in + j) : 0;
                    if (src >= 0) {
                        double2 v01 = *reinterpret_cast<const double2 *>(V + lane * 4);
                        double2 v23 = *reinterpret_cast<const double2 *>(V + lane * 4 + 2);
                        acc0 += v01.x; acc1 += v01.y; acc2 += v23.x; acc3 += v23.y;
                    }
                }
            } else {
                const int R = op.R, C = op.C;
                double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
                if (op.kind == BF_OP_TILE_N) {
                    if (lane < R) {
                        int j = lane;
                        for (int c = 0; c < C; ++c) {
                            const double x = T[c * R + j];
                            const double2 v01 = *reinterpret_cast<const double2 *>(V + c * 4);
                            const double2 v23 = *reinterpret_cast<const double2 *>(V + c * 4 + 2);
                            p0 = fma(x, v01.x, p0); p1 = fma(x, v01.y, p1);
                            p2 = fma(x, v23.x, p2); p3 = fma(x, v23.y, p3);
                            j = (j + 1 == R) ? 0 : j + 1;
                        }
                    }
                } else {
                    if (lane < C) {
                        int j = lane % R;
                        const double *col = T + lane * R;
                        for (int r = 0; r < R; ++r) {
                            const double x = col[j];
                            const double2 v01 = *reinterpret_cast<const double2 *>(V + r * 4);
                            const double2 v23 = *reinterpret_cast<const double2 *>(V + r * 4 + 2);
                            p0 = fma(x, v01.x, p0); p1 = fma(x, v01.y, p1);
                            p2 = fma(x, v23.x, p2); p3 = fma(x, v23.y, p3);
                            j = (j + 1 == R) ? 0 : j + 1;
                        }
                    }
                }
                const int width = (op.kind == BF_OP_TILE_N) ? R : C;
                int src;
                if (op.flags & BF_OPF_LANEMAP)
                    src = __ldg(a.maps + (int64_t)op.aux * BF_T + lane);
                else
                    src = lane - op.off;
                const bool ok = src >= 0 && src < width;
                const int sl = ok ? src : 0;
                p0 = __shfl_sync(0xffffffffu, p0, sl);
                p1 = __shfl_sync(0xffffffffu, p1, sl);
                p2 = __shfl_sync(0xffffffffu, p2, sl);
                p3 = __shfl_sync(0xffffffffu, p3, sl);
                if (ok) { acc0 += p0; acc1 += p1; acc2 += p2; acc3 += p3; }
            }
            __syncwarp();
            if (issued < nops) {
                bf_op nop = load_op(ops + issued);
                issue_op(a, ring, seq_issue % kStages, nop, lane);
                ++seq_issue;
                ++issued;
            }
        }
        if (lane < task.nout) {
            double *o = a.arena + ((int64_t)task.out + lane) * BF_NRHS;
            *reinterpret_cast<double2 *>(o) = make_double2(acc0, acc1);
            *reinterpret_cast<double2 *>(o + 2) = make_double2(acc2, acc3);
        }
    }
}

}  // namespace

static bool g_attr_set = false;

int bf_run_stage(bfsht_plan *pl, int64_t t0, int64_t t1, int *counter, cudaStream_t st) {
    if (t1 <= t0) return 0;
    const size_t smem = sizeof(WarpRing) * kWarps;
    if (!g_attr_set) {
        BF_CUDA(cudaFuncSetAttribute(alt_stage_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        g_attr_set = true;
    }
    StageArgs a;
    a.tiles = pl->tiles;
    a.ops = pl->ops;
    a.idx = pl->idx;
    a.maps = pl->maps;
    a.tasks = pl->tasks;
    a.arena = pl->arena;
    a.t0 = t0;
    a.ntasks = t1 - t0;
    a.counter = counter;
    BF_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    int64_t want = (a.ntasks + kWarps - 1) / kWarps;
    int grid = (int)(want < pl->sm_count ? want : pl->sm_count);
    alt_stage_kernel<<<grid, kWarps * 32, smem, st>>>(a);
    BF_CUDA(cudaGetLastError());
    pl->launches += 1;
    return 0;
}

int bf_alt_apply(bfsht_plan *pl, int dir, cudaStream_t st) {
    const std::vector<int64_t> &b = pl->stages[dir];
    const int nst = (int)b.size() - 1;
    if (pl->ncounters < nst) {
        bfsht_set_error("plan counters not allocated");
        return -3;
    }
    for (int s = 0; s < nst; ++s) {
        int rc = bf_run_stage(pl, b[s], b[s + 1], pl->counters + s, st);
        if (rc) return rc;
    }
    return 0;
}
