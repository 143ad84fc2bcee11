// ALT apply engine: persistent warp-task kernel over the packed tile store.
//
// Replaces the reference's per-order Python block loop
// (pkg/src/bfsht/alt.py:197-222) with its per-payload BLAS/scipy calls
// (butterfly.py:275-292, lowrank.py:196-202, alt.py:207,221) by one launch
// per dependency stage, covering every order of the plan at once.
//
// Execution model (sm_100a):
//  * grid = one CTA per SM, 12 warps per CTA; every warp is an independent
//    worker that walks the stage's task list (pre-sorted by cost) as one
//    flat op stream, claiming tasks from a global counter two tasks ahead.
//    (Measured: 12 warps x 2 slots beats 8 x 3 by ~20% — the consumer is
//    latency-bound per warp, so warps matter more than ring depth; a
//    variable-size byte ring with up to 6 small ops in flight was slower.)
//  * a task accumulates <= 64 output entries x 4 RHS in registers, then
//    stores them once: no atomics, fixed summation order, bitwise-
//    reproducible results.
//  * each warp owns a 2-slot shared-memory ring.  Lane 0 streams tiles (and
//    contiguous input vectors) with 1-D TMA bulk copies
//    (cp.async.bulk ... mbarrier::complete_tx), all lanes gather indexed
//    input entries with cp.async into the same slot, and the slot's
//    mbarrier completes when both have landed.  Op descriptors and gather
//    indices are prefetched one step ahead so no dependent global load sits
//    between a consumed op and the next issue.
//  * tile products run on the fp64 tensor cores: mma.sync.m8n8k4.f64 with
//    the 4 RHS in the n dimension (n = 8, half used).  A 32x32 tile costs 32
//    DMMA + 40 fragment loads instead of ~650 scalar instructions, which is
//    what keeps the kernel on the HBM roofline rather than issue-bound.
//    Payload bytes are read from HBM exactly once per direction.
//
// Kernels in this file: alt_stage_kernel (the model above; final dense /
// group stages, and every stage of a plan without a chain schedule),
// alt_chain_kernel (the butterfly-chain and low-rank-core stages from the
// plan's chain schedule: 32-byte records, bundles, folded index adds — same
// ring, same sums), alt_group_kernel (batched fields, 4 warps share a ring).
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.cuh"
#include "recur.h"

namespace {

#ifndef BF_WARPS
#define BF_WARPS 12
#endif
#ifndef BF_STAGES
#define BF_STAGES 2
#endif
constexpr int kWarps = BF_WARPS;       // SHT path (4 RHS per entry)
constexpr int kStages = BF_STAGES;
constexpr int kTileDoubles = BF_T * BF_T;

// Entry width NR (real RHS per arena entry): 4 for the SHT (re/im of +m and
// -m), 16 for batched fields.  Lane (g = lane/4, q = lane%4) owns RHS
// 8*grp + 2q, +1 of each 8-wide DMMA n-group grp; at NR = 4 only lanes
// q < 2 carry data and the B fragment's columns 4..7 are padding.
template <int NR>
struct Width {
    static constexpr int G = NR >= 8 ? NR / 8 : 1;      // n-groups
    static constexpr int QACT = NR >= 8 ? 4 : NR / 2;   // lanes q < QACT own RHS
    static constexpr int GACT = NR >= 8 ? 8 : NR;       // valid B columns
    static constexpr int WARPS = NR == 4 ? kWarps : (kStages == 2 ? 8 : (kStages == 3 ? 5 : 4));  // register / shared-memory bound
};

template <int NR>
struct alignas(128) WarpRing {
    double tile[kStages][kTileDoubles];
    double vec[kStages][BF_T * NR];
    int8_t map[kStages][BF_SLOTS];  // lane map of the slot's op (prefetched)
    double zero[16];                // stands in for blocks past a tile edge
    bf_op meta[kStages];            // op descriptor of the slot's op
    int4 tmeta[kStages];            // task out, nout|stride<<8, last-op-of-task
    unsigned long long full[kStages];
};
static_assert(sizeof(WarpRing<4>) * kWarps <= 227 * 1024, "SHT ring exceeds shared memory");
static_assert(sizeof(WarpRing<16>) * Width<16>::WARPS <= 227 * 1024,
              "batched ring exceeds shared memory");

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

// Programmatic dependent launch (the ALT stages of one direction are chained
// with cudaLaunchAttributeProgrammaticStreamSerialization): a stage's CTAs may
// start as the previous stage's CTAs retire, run their prologue (ring setup,
// first claims, first record / task loads — all plan data the previous stage
// does not write) and wait here before they touch the vector arena.  Without
// the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D(8x8) += A(8x4) * B(4x8), fp64 tensor core.  Lane l holds A[l/4][l%4],
// B[l%4][l/4], D[l/4][2(l%4)], D[l/4][2(l%4)+1].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
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
    const double *rec;     // recurrence coefficients (regenerated tiles)
    const double *xpos;    // positive nodes
    double mag_min;
};

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

// One op in flight through the per-warp pipeline (uniform across lanes).
struct Rec {
    bf_op op;
    int out, nout, last, valid;
};

// Walks the global task list as one flat op stream, one op per call.  Tasks
// are claimed two ahead: the atomicAdd result of the claim after next sits
// unread in lane 0 (raw) for a whole task, the next task's record is already
// loaded, so neither the atomic nor the record load stalls the warp.
struct Cursor {
    int base, n, i, out, nout;   // current task
    int nt;                      // next task id (uniform)
    bf_task ntask;               // its record (valid when nt < ntasks)
    int raw;                     // lane 0: claimed id of the task after next
};

// One claim by lane 0, as inline PTX: with atomicAdd() the compiler applies
// its warp-aggregation pattern (vote, popc, atomic, shuffle) and the shuffle
// reads the atomic's result at once — ncu showed the warp stalled there for
// the whole L2 round trip (6-9% of the chain stages' samples).  This way
// the result stays in flight until the next bcast() reads it.
__device__ __forceinline__ int claim_counter(int *counter, int lane) {
    int v = 0;
    if (lane == 0)
        asm volatile("atom.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(counter) : "memory");
    return v;
}

__device__ __forceinline__ int claim_raw(const StageArgs &a, int lane) {
    return claim_counter(a.counter, lane);
}

__device__ __forceinline__ int bcast(int raw) { return __shfl_sync(0xffffffffu, raw, 0); }

__device__ __forceinline__ bf_task load_task(const StageArgs &a, int t) {
    const int4 v = __ldg(reinterpret_cast<const int4 *>(a.tasks + a.t0 + t));
    bf_task k;
    k.op_begin = v.x;
    k.op_count = v.y;
    k.out = v.z;
    k.nout = v.w;
    return k;
}

__device__ __forceinline__ Rec advance(const StageArgs &a, Cursor &c, int lane) {
    Rec r;
    r.valid = 0;
    if (c.i >= c.n) {
        if (c.nt >= a.ntasks) return r;
        c.base = c.ntask.op_begin;
        c.n = c.ntask.op_count;
        c.out = c.ntask.out;
        c.nout = c.ntask.nout;
        c.i = 0;
        c.nt = bcast(c.raw);
        if (c.nt < a.ntasks) {
            c.ntask = load_task(a, c.nt);
            c.raw = claim_raw(a, lane);
        }
    }
    r.op = load_op(a.ops + c.base + c.i);
    r.out = c.out;
    r.nout = c.nout;
    r.last = (c.i == c.n - 1);
    r.valid = 1;
    ++c.i;
    return r;
}

// gather source of this lane for op r (-1: none); loaded one step early
__device__ __forceinline__ int gather_src(const StageArgs &a, const Rec &r, int lane) {
    if (!r.valid || !(r.op.flags & BF_OPF_GATHER)) return -1;
    if (r.op.kind == BF_OP_ADD) return lane < r.op.R ? __ldg(a.idx + r.op.in + lane) : -1;
    const int nvec = (r.op.kind == BF_OP_TILE_N) ? r.op.C : r.op.R;
    return lane < nvec ? __ldg(a.idx + r.op.in + lane) : -1;
}

__device__ __forceinline__ uint32_t tile_bytes(const bf_op &op) {
    return (op.flags & BF_OPF_REGEN) ? (uint32_t)bf_seed_doubles(op.R, op.C) * 8u
                                     : (uint32_t)bf_tile_doubles(op.R, op.C) * 8u;
}

// Where a tile's bytes land in its ring slot: at the start, stored values
// and regeneration seed blocks alike (the seeds are read into registers
// before any value is written).  A regenerated tile's step coefficients are
// staged separately (regen_coef).
__device__ __forceinline__ uint32_t tile_dst(const bf_op &) { return 0u; }

// Ring-slot position (doubles) of column c's four step coefficients
// (alpha, beta of its two steps) for a regenerated tile with C4 column
// blocks, chosen so that no value is written there before the coefficient
// has been read and no seed is staged there: with <= 7 column blocks the
// free tail of the slot (values end below 7 x 8 x 16 = 896 doubles); with 8,
// column blocks 3 and 7 of row blocks 2-7 — the blocks the two chains write
// last (seeds occupy row blocks 0-1).
__device__ __forceinline__ int regen_coef(int c, int C4) {
    if (C4 < BF_T / 4) return 896 + 4 * c;
    const int k = c >> 2;
    return (2 + (k >> 1)) * 128 + ((k & 1) ? 7 : 3) * 16 + 4 * (c & 3);
}

// |v| as its IEEE bit pattern, built from the two 32-bit halves so that the
// compiler keeps it on the integer pipe (a 64-bit mask becomes a DADD |v|)
__device__ __forceinline__ long long abits(double v) {
    const unsigned hi = (unsigned)__double2hiint(v) & 0x7fffffffu;
    const unsigned lo = (unsigned)__double2loint(v);
    return (long long)(((unsigned long long)hi << 32) | lo);
}

// One recurrence step without the range test (recur.h bfr_step's
// arithmetic: three roundings, one subtraction, no FMA).
__device__ __forceinline__ void rec_step(double x, double a, double b, double &pp, double &pc) {
    const double t1 = __dmul_rn(x, pc);
    const double t2 = __dmul_rn(a, t1);
    const double t3 = __dmul_rn(b, pp);
    const double pn = __dsub_rn(t2, t3);
    pp = pc;
    pc = pn;
}

// bfr_step's range test and exact 2^-+1000 rescale, on IEEE bit patterns
// (|p| > 2^500 <=> abits(p) > 0x5F3..., |p| < 2^-500 <=> abits(p) < 0x20B...),
// branch-free: the scale factor is 1.0 (exact, no change) when in range.
__device__ __forceinline__ void rec_rescale(double &pp, double &pc, int &e) {
    const long long ua = abits(pc), ub = abits(pp);
    const long long mx = ua > ub ? ua : ub;
    const bool big = mx > 0x5F30000000000000LL;
    const bool small = mx < 0x20B0000000000000LL && mx > 0;
    const double f = big ? 0x1p-1000 : (small ? 0x1p1000 : 1.0);
    pc = __dmul_rn(pc, f);
    pp = __dmul_rn(pp, f);
    e += big ? 1000 : (small ? -1000 : 0);
}

// One block step of K chains (chain h covers columns [16h, ...)): emit
// column block j of each chain, advance each by its 4 columns, range-test.
// Emission with e fixed for the block, as one 64-bit compare: for a value
// that survives the flush (|p| 2^e >= mag_min, hence normal), its bits are
// abits(p) + (e << 52), so "keep" is abits(p) >= mag_bits - (e << 52); a
// kept value is that exponent shift of p (exact).  e <= -1700 can only give
// flushed values (|p| < 2^560).  p = 0 is never kept.
template <int K>
__device__ __forceinline__ void regen_block(const double *T, int C, int C4, int j, double x,
                                            double (&pp)[K], double (&pc)[K], int (&e)[K],
                                            long long mag_bits, double (&v)[K][4]) {
    const int cend0 = C < BF_SEED_SPLIT ? C : BF_SEED_SPLIT;
#pragma unroll
    for (int h = 0; h < K; ++h) {
        // this block's coefficients, 4 columns x (alpha, beta) x 2 steps,
        // contiguous in the slot (regen_coef), loaded before the chain work
        double2 cf[8];
        const double2 *base =
            reinterpret_cast<const double2 *>(T + regen_coef(h * BF_SEED_SPLIT + 4 * j, C4));
#pragma unroll
        for (int t = 0; t < 8; ++t) cf[t] = base[t];
        const long long e52 = (long long)e[h] << 52;
        const long long thr = e[h] <= -1700 ? 0x7fffffffffffffffLL : mag_bits - e52;
        const int cend = h == 0 ? cend0 : C;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = h * BF_SEED_SPLIT + 4 * j + i;
            const long long b = __double_as_longlong(pc[h]);
            v[h][i] = (c < cend && abits(pc[h]) >= thr) ? __longlong_as_double(b + e52) : 0.0;
            if (c + 1 < cend) {
                rec_step(x, cf[2 * i].x, cf[2 * i].y, pp[h], pc[h]);
                rec_step(x, cf[2 * i + 1].x, cf[2 * i + 1].y, pp[h], pc[h]);
            }
        }
        rec_rescale(pp[h], pc[h], e[h]);
    }
}

template <int K>
__device__ __forceinline__ void regen_chains(const double *sb, const double *__restrict__ xpos,
                                             long long mag_bits, int R, int C, double *T,
                                             int lane) {
    const int C4 = (C + 3) >> 2, R4 = (R + 3) >> 2;
    const int r_a = __double2loint(sb[0]);
    double pp[K], pc[K], x = 0.0;
    int e[K];
#pragma unroll
    for (int h = 0; h < K; ++h) {
        pp[h] = pc[h] = 0.0;
        e[h] = 0;
        if (lane < R) {
            pp[h] = sb[2 + 3 * (h * R + lane)];
            pc[h] = sb[3 + 3 * (h * R + lane)];
            e[h] = (int)sb[4 + 3 * (h * R + lane)];
        }
    }
    if (lane < R) x = __ldg(xpos + r_a + lane);
    __syncwarp();   // seeds read: their slot region may now be overwritten
    double *row = T + (lane >> 2) * C4 * 16 + (lane & 3) * 4;
    const int nj = K == 1 ? C4 : BF_SEED_SPLIT / 4;
#pragma unroll 1
    for (int j = 0; j < nj; ++j) {
        double v[K][4];
        regen_block<K>(T, C, C4, j, x, pp, pc, e, mag_bits, v);
        __syncwarp();   // every lane has read this block's coefficients
        if (lane < R4 * 4) {
#pragma unroll
            for (int h = 0; h < K; ++h) {
                const int cb = h * (BF_SEED_SPLIT / 4) + j;
                if (cb < C4) {
                    double2 *d = reinterpret_cast<double2 *>(row + cb * 16);
                    d[0] = make_double2(v[h][0], v[h][1]);
                    d[1] = make_double2(v[h][2], v[h][3]);
                }
            }
        }
    }
    __syncwarp();
}

// Regenerate a dense turning tile in place from its seed block:
// lane r re-runs row r's degree recurrence as the planner did (recur.h;
// pkg/src/bfsht/kernels/_recur_cy.pyx:45-66), two steps per column
// (degrees of one parity), emitting ldexp(p, e) flushed below MAG_MIN —
// the stored values bit for bit (tests/test_regen_pack.py,
// tests/test_gpu_regen.py).
//
// Cost shape.  The step is a chain of three dependent fp64 operations, so
// one recurrence per lane is latency-bound (measured ~2500 warp
// instructions and ~15 k cycles per tile in the first version): tiles
// wider than 16 columns carry a second seed (the state at column 16), and
// every lane runs the two column halves as two independent chains.  The
// reference tests the (mantissa, 2^e) range after every step; here it is
// tested once per 4 columns (8 steps), branch-free.  The rescale multiplies
// by an exact power of two; a step grows |p| by at most alpha |x| + beta
// < 2^7 and shrinks the larger of |p_k|, |p_k-1| by at most ~2, so between
// tests the mantissas stay inside [2^-510, 2^556] (a nonzero difference of
// two rounded products there is above 2^-560): every intermediate is the
// reference's value times 2^(1000 j), and every emitted ldexp(p, e) is the
// same number.  The step coefficients were staged into the slot at issue
// time (cp.async, regen_coef) and are read as warp-uniform shared loads.
// Padding rows / columns come out as zeros.
// Emission of one column (e fixed for the block), as regen_block.
__device__ __forceinline__ double regen_emit(double pc, long long thr, long long e52) {
    return abits(pc) >= thr ? __longlong_as_double(__double_as_longlong(pc) + e52) : 0.0;
}

// Full 32 x 32 tile (the common case: turning blocks cut on the absolute
// 32-grid): the same operation sequence as regen_chains<2> — chain h covers
// columns 16h .. 16h+15, emit, two steps after every column but the chain's
// last, range test after every 4 columns — as straight-line code: no
// per-column edge tests, the two chains interleaved step by step for ILP,
// and each block's 16 coefficient pairs loaded before its chain work.
__device__ __forceinline__ void regen_full(const double *__restrict__ xpos, long long mag_bits,
                                           double *T, int lane) {
    constexpr int C4 = 8, R = 32;
    const int r_a = __double2loint(T[0]);
    double pp0 = T[2 + 3 * lane], pc0 = T[3 + 3 * lane];
    int e0 = (int)T[4 + 3 * lane];
    double pp1 = T[2 + 3 * (R + lane)], pc1 = T[3 + 3 * (R + lane)];
    int e1 = (int)T[4 + 3 * (R + lane)];
    const double x = __ldg(xpos + r_a + lane);
    __syncwarp();   // seeds read: their slot region may now be overwritten
    double *row = T + (lane >> 2) * C4 * 16 + (lane & 3) * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        double2 c0[8], c1[8];
        const double2 *b0 = reinterpret_cast<const double2 *>(T + regen_coef(4 * j, C4));
        const double2 *b1 = reinterpret_cast<const double2 *>(T + regen_coef(16 + 4 * j, C4));
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            c0[t] = b0[t];
            c1[t] = b1[t];
        }
        const long long e52a = (long long)e0 << 52, e52b = (long long)e1 << 52;
        const long long tha = e0 <= -1700 ? 0x7fffffffffffffffLL : mag_bits - e52a;
        const long long thb = e1 <= -1700 ? 0x7fffffffffffffffLL : mag_bits - e52b;
        double v0[4], v1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v0[i] = regen_emit(pc0, tha, e52a);
            v1[i] = regen_emit(pc1, thb, e52b);
            if (j < 3 || i < 3) {
                rec_step(x, c0[2 * i].x, c0[2 * i].y, pp0, pc0);
                rec_step(x, c1[2 * i].x, c1[2 * i].y, pp1, pc1);
                rec_step(x, c0[2 * i + 1].x, c0[2 * i + 1].y, pp0, pc0);
                rec_step(x, c1[2 * i + 1].x, c1[2 * i + 1].y, pp1, pc1);
            }
        }
        rec_rescale(pp0, pc0, e0);
        rec_rescale(pp1, pc1, e1);
        __syncwarp();   // every lane has read this block's coefficients
        double2 *d0 = reinterpret_cast<double2 *>(row + j * 16);
        double2 *d1 = reinterpret_cast<double2 *>(row + (4 + j) * 16);
        d0[0] = make_double2(v0[0], v0[1]);
        d0[1] = make_double2(v0[2], v0[3]);
        d1[0] = make_double2(v1[0], v1[1]);
        d1[1] = make_double2(v1[2], v1[3]);
    }
    __syncwarp();
}

__device__ __noinline__ void regen_tile(const double *__restrict__ xpos, long long mag_bits, int R,
                                        int C, double *T, int lane) {
    if (R == BF_T && C == BF_T) {
        regen_full(xpos, mag_bits, T, lane);
        return;
    }
    if (bf_seed_chains(C) == 2)
        regen_chains<2>(T, xpos, mag_bits, R, C, T, lane);
    else
        regen_chains<1>(T, xpos, mag_bits, R, C, T, lane);
}

// Issue the loads of one op into ring slot s (whole warp).
template <int NR>
__device__ __forceinline__ void issue(const StageArgs &a, WarpRing<NR> &ring, int s, const Rec &r,
                                      int gsrc, int lane) {
    const bf_op &op = r.op;
    const double *arena = a.arena;
    const bool gather = (op.flags & BF_OPF_GATHER) != 0;
    if (lane == 0) {
        ring.meta[s] = op;
        ring.tmeta[s] = make_int4(r.out, r.nout, r.last, 0);
    }
    uint32_t bytes = 0;
    int nvec = 0;
    int src = -1;
    if (op.kind == BF_OP_ADD) {
        // lane j < R fetches entry j (added into slot off + j by the consumer)
        if (lane < op.R) src = gather ? gsrc : op.in + lane;
    } else {
        nvec = (op.kind == BF_OP_TILE_N) ? op.C : op.R;
        bytes = tile_bytes(op);
        if (gather)
            src = gsrc;
        else
            bytes += (uint32_t)nvec * NR * 8u;
    }
    if (src >= 0 && (gather || op.kind == BF_OP_ADD)) {
        const double *gp = arena + (int64_t)src * NR;
#pragma unroll
        for (int k = 0; k < NR; k += 2) cp_async16(&ring.vec[s][lane * NR + k], gp + k);
    } else if (op.kind == BF_OP_ADD) {
        // lanes without a source add zeros (keeps index loads off the consumer)
#pragma unroll
        for (int k = 0; k < NR; k += 2)
            *reinterpret_cast<double2 *>(&ring.vec[s][lane * NR + k]) = make_double2(0.0, 0.0);
    }
    if ((op.flags & BF_OPF_LANEMAP) && lane < BF_SLOTS / 16)
        cp_async16(&ring.map[s][lane * 16], a.maps + (int64_t)op.aux * BF_SLOTS + lane * 16);
    if ((op.flags & BF_OPF_REGEN) && lane + 1 < op.C) {
        // lane c: column c's 4 step coefficients (32 B) from the rec table
        double *d = ring.tile[s] + regen_coef(lane, (op.C + 3) >> 2);
        const double *g = a.rec + (int64_t)op.aux + 4 * lane;
        cp_async16(d, g);
        cp_async16(d + 2, g + 2);
    }
    cp_async_arrive(&ring.full[s]);
    if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_tx(&ring.full[s], bytes);
        if (op.kind != BF_OP_ADD) {
            bulk_g2s(ring.tile[s] + tile_dst(op), a.tiles + op.tile, tile_bytes(op), &ring.full[s]);
            if (!gather)
                bulk_g2s(ring.vec[s], arena + (int64_t)op.in * NR, (uint32_t)nvec * NR * 8u,
                         &ring.full[s]);
        }
    }
}

// B fragment of n-group grp at k block ks: lane holds V[k = 4ks + q][rhs =
// 8grp + g] (columns past the entry width are the n-padding)
template <int VS>
__device__ __forceinline__ double bfrag(const double *Vb, int ks, int grp, bool bl) {
    return bl ? Vb[ks * 4 * VS + grp * 8] : 0.0;
}

// Tile product of one op into fragments e: e[grp][mt][0..1] = result row
// 8mt + lane/4, RHS 8grp + 2(lane%4), +1.  V: input entries VS doubles
// apart (the warp's NR-wide slice of a wider entry when VS > NR).
template <int NR, int VS = NR>
__device__ __forceinline__ void tile_product(const bf_op &op, const double *T, const double *V,
                                             const double *Z, int lane,
                                             double e[Width<NR>::G][4][2]) {
    constexpr int G = Width<NR>::G;
    const int g = lane >> 2, q = lane & 3, hi = lane >> 4;
    const int R4 = (op.R + 3) >> 2, C4 = (op.C + 3) >> 2;
#pragma unroll
    for (int gr = 0; gr < G; ++gr)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) e[gr][mt][0] = e[gr][mt][1] = 0.0;
    const bool bl = g < Width<NR>::GACT;
    const double *Vb = V + q * VS + (NR >= 8 ? g : (g & (NR - 1)));
    if (op.R == BF_T && op.C == BF_T) {
        // full tile: straight-line, all fragment offsets are immediates
        if (op.kind == BF_OP_TILE_N) {
            const double *Ta = T + hi * (8 * 16) + (lane & 15);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                double av[4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) av[mt] = Ta[(mt * 16 + ks) * 16];
#pragma unroll
                for (int gr = 0; gr < G; ++gr) {
                    const double b = bfrag<VS>(Vb, ks, gr, bl);
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma(e[gr][mt][0], e[gr][mt][1], av[mt], b);
                }
            }
        } else {
            const double *Ta = T + hi * 16 + q * 4 + (g & 3);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                double av[4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) av[mt] = Ta[(ks * 8 + 2 * mt) * 16];
#pragma unroll
                for (int gr = 0; gr < G; ++gr) {
                    const double b = bfrag<VS>(Vb, ks, gr, bl);
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) dmma(e[gr][mt][0], e[gr][mt][1], av[mt], b);
                }
            }
        }
        return;
    }
    // partial tile: per-lane fragment pointers walk the k blocks; block rows
    // (N) / block columns (T) past the tile edge read a zero block instead,
    // so the k loop carries no predicates
    const double *p[4];
    int st[4];
    int K, MT;
    if (op.kind == BF_OP_TILE_N) {
        // y = A x: result rows = tile rows, k over tile column blocks
        K = C4;
        MT = (op.R + 7) >> 3;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int br = 2 * mt + hi;
            const bool ok = br < R4;
            p[mt] = (ok ? T + br * C4 * 16 : Z) + (lane & 15);
            st[mt] = ok ? 16 : 0;
        }
    } else {
        // x = A^T y: result rows = tile columns, k over tile row blocks
        K = R4;
        MT = (op.C + 7) >> 3;
        const int inblk = q * 4 + (g & 3);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int bc = 2 * mt + hi;
            const bool ok = bc < C4;
            p[mt] = (ok ? T + bc * 16 : Z) + inblk;
            st[mt] = ok ? C4 * 16 : 0;
        }
    }
#define BF_PARTIAL(NMT)                                                        \
    for (int ks = 0; ks < K; ++ks) {                                           \
        double av[NMT];                                                        \
        _Pragma("unroll") for (int mt = 0; mt < NMT; ++mt) {                   \
            av[mt] = *p[mt];                                                   \
            p[mt] += st[mt];                                                   \
        }                                                                      \
        _Pragma("unroll") for (int gr = 0; gr < G; ++gr) {                     \
            const double b = bfrag<VS>(Vb, ks, gr, bl);                        \
            _Pragma("unroll") for (int mt = 0; mt < NMT; ++mt)                 \
                dmma(e[gr][mt][0], e[gr][mt][1], av[mt], b);                   \
        }                                                                      \
    }
    switch (MT) {
        case 4: BF_PARTIAL(4) break;
        case 3: BF_PARTIAL(3) break;
        case 2: BF_PARTIAL(2) break;
        default: BF_PARTIAL(1) break;
    }
#undef BF_PARTIAL
}

// result m-tiles 0..3 of an op onto accumulator m-tiles SH..SH+3
template <int G, int SH>
__device__ __forceinline__ void place_tiles(double acc[G][8][2], const double e[G][4][2]) {
#pragma unroll
    for (int gr = 0; gr < G; ++gr)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
            if (SH + mt < 8) {
                acc[gr][SH + mt][0] += e[gr][mt][0];
                acc[gr][SH + mt][1] += e[gr][mt][1];
            }
}

template <int NR>
__global__ void __launch_bounds__(Width<NR>::WARPS * 32, 1) alt_stage_kernel(StageArgs a) {
    constexpr int G = Width<NR>::G, QACT = Width<NR>::QACT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpRing<NR> &ring = reinterpret_cast<WarpRing<NR> *>(smem_raw)[warp];
    {
        // zero the ring once: padded tile columns multiply stale vector
        // entries, which must therefore be finite
        double2 *z = reinterpret_cast<double2 *>(&ring);
        const int n2 = (int)(offsetof(WarpRing<NR>, meta) / sizeof(double2));
        for (int i = lane; i < n2; i += 32) z[i] = make_double2(0.0, 0.0);
    }
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&ring.full[s], 33);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int g = lane >> 2, q = lane & 3;

    Cursor cur;
    cur.n = cur.i = 0;
    cur.base = cur.out = cur.nout = 0;
    cur.nt = bcast(claim_raw(a, lane));
    cur.raw = 0;
    if (cur.nt < a.ntasks) {
        cur.ntask = load_task(a, cur.nt);
        cur.raw = claim_raw(a, lane);
    }

    Rec q0 = advance(a, cur, lane);
    int g0 = gather_src(a, q0, lane);
    Rec q1 = advance(a, cur, lane);
    uint32_t seq_issue = 0, seq_use = 0;
    auto issue_next = [&]() {
        issue<NR>(a, ring, seq_issue % kStages, q0, g0, lane);
        ++seq_issue;
        q0 = q1;
        g0 = gather_src(a, q0, lane);
        q1 = advance(a, cur, lane);
    };
    pdl_launch_dependents();
    pdl_wait();
    while (q0.valid && seq_issue - seq_use < kStages) issue_next();

    // task accumulator: acc[grp][j] = slot 8j + lane/4, RHS 8grp + 2(lane%4)
    // .. +1, 64 slots (dense group tasks use the first 32)
    double acc[G][8][2];
#pragma unroll
    for (int gr = 0; gr < G; ++gr)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[gr][j][0] = acc[gr][j][1] = 0.0;

    while (seq_use < seq_issue) {
        const int s = seq_use % kStages;
        mbar_wait(&ring.full[s], (seq_use / kStages) & 1u);
        ++seq_use;
        const bf_op op = ring.meta[s];
        const int4 tm = ring.tmeta[s];
        const double *V = ring.vec[s];
        if (op.kind == BF_OP_ADD) {
            // entry j of the op (vec row j) adds into slot off + j
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = 8 * j + g - op.off;
                if (q < QACT && jj >= 0 && jj < op.R) {
#pragma unroll
                    for (int gr = 0; gr < G; ++gr) {
                        const double2 v =
                            *reinterpret_cast<const double2 *>(V + jj * NR + gr * 8 + 2 * q);
                        acc[gr][j][0] += v.x;
                        acc[gr][j][1] += v.y;
                    }
                }
            }
        } else {
            if (op.flags & BF_OPF_REGEN)
                regen_tile(a.xpos, __double_as_longlong(a.mag_min), op.R, op.C, ring.tile[s], lane);
            double e[G][4][2];
            tile_product<NR>(op, ring.tile[s], V, ring.zero, lane, e);
            const bool lanemap = (op.flags & BF_OPF_LANEMAP) != 0;
            if (!lanemap && (op.off & 7) == 0) {
                // result m-tile mt lands on slot m-tile mt + off/8
                // (one case per shift keeps acc and e in registers)
                switch (op.off >> 3) {
                    case 0: place_tiles<G, 0>(acc, e); break;
                    case 1: place_tiles<G, 1>(acc, e); break;
                    case 2: place_tiles<G, 2>(acc, e); break;
                    case 3: place_tiles<G, 3>(acc, e); break;
                    case 4: place_tiles<G, 4>(acc, e); break;
                    case 5: place_tiles<G, 5>(acc, e); break;
                    case 6: place_tiles<G, 6>(acc, e); break;
                    default: place_tiles<G, 7>(acc, e); break;
                }
            } else {
                // general placement through the warp's scratch rows
                // the slot's input vector is dead once the product is formed:
                // it doubles as the staging area for the placement
                double *S = ring.vec[s];
                __syncwarp();
                const int width = (op.kind == BF_OP_TILE_N) ? op.R : op.C;
                const int MT = (width + 7) >> 3;
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
                    if (mt < MT && q < QACT) {
#pragma unroll
                        for (int gr = 0; gr < G; ++gr)
                            *reinterpret_cast<double2 *>(S + (8 * mt + g) * NR + gr * 8 + 2 * q) =
                                make_double2(e[gr][mt][0], e[gr][mt][1]);
                    }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int sl = 8 * j + g;
                    const int src = lanemap ? (int)ring.map[s][sl]
                                            : sl - op.off;
                    if (q < QACT && src >= 0 && src < width) {
#pragma unroll
                        for (int gr = 0; gr < G; ++gr) {
                            const double2 v =
                                *reinterpret_cast<const double2 *>(S + src * NR + gr * 8 + 2 * q);
                            acc[gr][j][0] += v.x;
                            acc[gr][j][1] += v.y;
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (tm.z) {
            const int nout = tm.y & 0xff;
            const int stride = (tm.y >> 8) ? (tm.y >> 8) : 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int sl = 8 * j + g;
                if (q < QACT && sl < nout) {
                    double *o = a.arena + ((int64_t)tm.x + (int64_t)sl * stride) * NR + 2 * q;
#pragma unroll
                    for (int gr = 0; gr < G; ++gr)
                        *reinterpret_cast<double2 *>(o + gr * 8) =
                            make_double2(acc[gr][j][0], acc[gr][j][1]);
                }
#pragma unroll
                for (int gr = 0; gr < G; ++gr) acc[gr][j][0] = acc[gr][j][1] = 0.0;
            }
        }
        __syncwarp();
        while (q0.valid && seq_issue - seq_use < kStages) issue_next();
    }
}

// ------------------------------------------------------------ chain engine
// The butterfly-chain and low-rank-core stages are made of small tasks (3-9
// ops, tiles of 2-6 KB, 32-byte gathers, 20-35% index adds).  On
// alt_stage_kernel they ran at under half of the HBM roofline, and ncu put
// that on instruction issue, not on memory: ~600 warp instructions per op
// (task claims, cursor and record bookkeeping ~60% of them) with warps
// stalled on fixed-latency dependencies and on the record / claim loads.
// alt_chain_kernel runs the same ops, in the same per-task order (results
// are bitwise those of alt_stage_kernel), from a schedule built once per
// plan (bf_chain_build):
//  * one 32-byte record per op carrying everything the warp needs (tile,
//    input, lane map, shape, the task's output range on its last op), read
//    as two 16-byte loads two ops ahead — no task records, no cursor;
//  * tasks pre-grouped into cost-balanced bundles (LPT) that a warp claims
//    with one atomic per bundle instead of one per task;
//  * an index add that follows a tile op is folded into that op's record:
//    its gathered entries land in the free tail of the tile slot and are
//    added right after the tile product, so it costs no ring slot, no
//    barrier wait and no op of its own.
struct ChainArgs {
    const double *tiles;
    const int4 *rec;         // bf_crec records as two int4 each
    const int32_t *bund;     // the stage's bundle bounds (nb + 1 record indices)
    const int32_t *idx;
    const int8_t *maps;
    double *arena;
    int nb;
    int *counter;
};

struct alignas(128) ChainRing {
    double tile[kStages][kTileDoubles];
    double vec[kStages][BF_T * BF_NRHS];
    int8_t map[kStages][BF_SLOTS];
    double zero[16];
    int4 meta[kStages][2];
    unsigned long long full[kStages];
};
static_assert(sizeof(ChainRing) * kWarps <= 227 * 1024, "chain ring exceeds shared memory");
static_assert(sizeof(bf_crec) == 32, "chain record is two int4");
static_assert(BF_FOLD_AT + BF_T * BF_NRHS <= kTileDoubles, "folded add past the tile slot");

// a: tile, in, aux, kind | R << 8 | C << 16 | off << 24
// b: flags | addR << 8 | addoff << 16, add_in, out, nout
struct CRec {
    int4 a, b;
};

__device__ __forceinline__ CRec load_crec(const ChainArgs &a, int i) {
    CRec r;
    const int4 *p = a.rec + 2 * (int64_t)i;
    r.a = __ldg(p);
    r.b = __ldg(p + 1);
    return r;
}

struct CStream {
    int pos, end;       // records of the current bundle
    int npos, nend;     // the next bundle (claimed, bounds loaded)
    int raw;            // lane 0: id of the bundle after next
};

__device__ __forceinline__ int chain_claim(const ChainArgs &a, int lane) {
    return claim_counter(a.counter, lane);
}

// index of the next record of this warp's stream, -1 at the end
__device__ __forceinline__ int chain_next(const ChainArgs &a, CStream &c, int lane) {
    if (c.pos >= c.end) {
        if (c.npos >= c.nend) return -1;
        c.pos = c.npos;
        c.end = c.nend;
        const int nb = bcast(c.raw);
        if (nb < a.nb) {
            c.npos = __ldg(a.bund + nb);
            c.nend = __ldg(a.bund + nb + 1);
            c.raw = chain_claim(a, lane);
        } else {
            c.npos = c.nend = 0;
        }
    }
    return c.pos++;
}

// gather sources of this lane for record r (-1: none), loaded one op early
__device__ __forceinline__ int chain_gsrc(const ChainArgs &a, const CRec &r, int lane) {
    const uint32_t w = (uint32_t)r.a.w;
    if (!(r.b.x & BF_OPF_GATHER)) return -1;
    const int kind = w & 0xff, R = (w >> 8) & 0xff, C = (w >> 16) & 0xff;
    const int nvec = kind == BF_OP_TILE_N ? C : R;
    return lane < nvec ? __ldg(a.idx + r.a.y + lane) : -1;
}

// sources of the folded index add: entries lane and lane + 32 (a fold holds
// up to 64 entries: two back-to-back adds of one scatter task)
__device__ __forceinline__ int2 chain_gadd(const ChainArgs &a, const CRec &r, int lane) {
    int2 v = make_int2(-1, -1);
    if (!(r.b.x & BF_CF_ADD)) return v;
    const int addR = ((uint32_t)r.b.x >> 8) & 0xff;
    if (lane < addR) v.x = __ldg(a.idx + r.b.y + lane);
    if (lane + 32 < addR) v.y = __ldg(a.idx + r.b.y + lane + 32);
    return v;
}

// where a fold's entries land in the tile slot: the last 1 KB, or the last
// 2 KB when it holds more than 32 entries
__device__ __forceinline__ int fold_at(int addR) {
    return addR > BF_T ? BF_FOLD_AT - BF_T * BF_NRHS : BF_FOLD_AT;
}

__device__ __forceinline__ void chain_issue(const ChainArgs &a, ChainRing &ring, int s,
                                            const CRec &r, int gsrc, int2 gadd, int lane) {
    const uint32_t w = (uint32_t)r.a.w, f = (uint32_t)r.b.x;
    const int kind = w & 0xff, R = (w >> 8) & 0xff, C = (w >> 16) & 0xff;
    const bool gather = (f & BF_OPF_GATHER) != 0;
    if (lane == 0) {
        ring.meta[s][0] = r.a;
        ring.meta[s][1] = r.b;
    }
    const int nvec = kind == BF_OP_TILE_N ? C : R;
    const uint32_t tb = kind == BF_OP_ADD ? 0u : (uint32_t)(((R + 3) >> 2) * ((C + 3) >> 2)) * 128u;
    if (gather) {
        double *d = &ring.vec[s][lane * BF_NRHS];
        if (gsrc >= 0) {
            const double *gp = a.arena + (int64_t)gsrc * BF_NRHS;
            cp_async16(d, gp);
            cp_async16(d + 2, gp + 2);
        } else if (kind == BF_OP_ADD) {
            // lanes without a source add zeros
            *reinterpret_cast<double2 *>(d) = make_double2(0.0, 0.0);
            *reinterpret_cast<double2 *>(d + 2) = make_double2(0.0, 0.0);
        }
    }
    if (f & BF_CF_ADD) {
        const int addR = (f >> 8) & 0xff;
        double *d = ring.tile[s] + fold_at(addR) + lane * BF_NRHS;
        if (gadd.x >= 0) {
            const double *gp = a.arena + (int64_t)gadd.x * BF_NRHS;
            cp_async16(d, gp);
            cp_async16(d + 2, gp + 2);
        } else {
            *reinterpret_cast<double2 *>(d) = make_double2(0.0, 0.0);
            *reinterpret_cast<double2 *>(d + 2) = make_double2(0.0, 0.0);
        }
        if (addR > BF_T) {
            d += BF_T * BF_NRHS;
            if (gadd.y >= 0) {
                const double *gp = a.arena + (int64_t)gadd.y * BF_NRHS;
                cp_async16(d, gp);
                cp_async16(d + 2, gp + 2);
            } else {
                *reinterpret_cast<double2 *>(d) = make_double2(0.0, 0.0);
                *reinterpret_cast<double2 *>(d + 2) = make_double2(0.0, 0.0);
            }
        }
    }
    cp_async_arrive(&ring.full[s]);
    if (lane == 0) {
        const bool lanemap = (f & BF_OPF_LANEMAP) != 0;
        const uint32_t vb = gather ? 0u : (uint32_t)nvec * (BF_NRHS * 8u);
        fence_proxy_async();
        mbar_arrive_tx(&ring.full[s], tb + vb + (lanemap ? (uint32_t)BF_SLOTS : 0u));
        if (tb) bulk_g2s(ring.tile[s], a.tiles + (int64_t)(uint32_t)r.a.x * 16, tb, &ring.full[s]);
        if (vb) bulk_g2s(ring.vec[s], a.arena + (int64_t)r.a.y * BF_NRHS, vb, &ring.full[s]);
        if (lanemap)
            bulk_g2s(ring.map[s], a.maps + (int64_t)r.a.z * BF_SLOTS, BF_SLOTS, &ring.full[s]);
    }
}

__global__ void __launch_bounds__(kWarps * 32, 1) alt_chain_kernel(ChainArgs a) {
    constexpr int NR = BF_NRHS, QACT = Width<NR>::QACT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    ChainRing &ring = reinterpret_cast<ChainRing *>(smem_raw)[warp];
    {
        double2 *z = reinterpret_cast<double2 *>(&ring);
        const int n2 = (int)(offsetof(ChainRing, meta) / sizeof(double2));
        for (int i = lane; i < n2; i += 32) z[i] = make_double2(0.0, 0.0);
    }
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&ring.full[s], 33);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int g = lane >> 2, q = lane & 3;

    CStream cs;
    cs.pos = cs.end = cs.npos = cs.nend = 0;
    cs.raw = 0;
    {
        const int first = bcast(chain_claim(a, lane));
        if (first < a.nb) {
            cs.npos = __ldg(a.bund + first);
            cs.nend = __ldg(a.bund + first + 1);
            cs.raw = chain_claim(a, lane);
        }
    }
    CRec r0, r1;
    r0.a = r0.b = r1.a = r1.b = make_int4(0, 0, 0, 0);
    int i0 = chain_next(a, cs, lane);
    if (i0 >= 0) r0 = load_crec(a, i0);
    int g0 = i0 >= 0 ? chain_gsrc(a, r0, lane) : -1;
    int2 ga0 = i0 >= 0 ? chain_gadd(a, r0, lane) : make_int2(-1, -1);
    int i1 = i0 >= 0 ? chain_next(a, cs, lane) : -1;
    if (i1 >= 0) r1 = load_crec(a, i1);
    uint32_t seq_issue = 0, seq_use = 0;
    auto issue_next = [&]() {
        chain_issue(a, ring, seq_issue % kStages, r0, g0, ga0, lane);
        ++seq_issue;
        r0 = r1;
        i0 = i1;
        if (i0 >= 0) {
            g0 = chain_gsrc(a, r0, lane);
            ga0 = chain_gadd(a, r0, lane);
            i1 = chain_next(a, cs, lane);
            if (i1 >= 0) r1 = load_crec(a, i1);
        }
    };
    pdl_launch_dependents();
    pdl_wait();
    while (i0 >= 0 && seq_issue - seq_use < kStages) issue_next();

    double acc[1][8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[0][j][0] = acc[0][j][1] = 0.0;

    while (seq_use < seq_issue) {
        const int s = seq_use % kStages;
        mbar_wait(&ring.full[s], (seq_use / kStages) & 1u);
        ++seq_use;
        const int4 ma = ring.meta[s][0], mb = ring.meta[s][1];
        const uint32_t w = (uint32_t)ma.w, f = (uint32_t)mb.x;
        bf_op op;
        op.kind = (uint8_t)(w & 0xff);
        op.R = (uint8_t)((w >> 8) & 0xff);
        op.C = (uint8_t)((w >> 16) & 0xff);
        op.off = (uint8_t)(w >> 24);
        const double *V = ring.vec[s];
        if (op.kind == BF_OP_ADD) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = 8 * j + g - op.off;
                if (q < QACT && jj >= 0 && jj < op.R) {
                    const double2 v = *reinterpret_cast<const double2 *>(V + jj * NR + 2 * q);
                    acc[0][j][0] += v.x;
                    acc[0][j][1] += v.y;
                }
            }
        } else {
            double e[1][4][2];
            tile_product<NR>(op, ring.tile[s], V, ring.zero, lane, e);
            const bool lanemap = (f & BF_OPF_LANEMAP) != 0;
            if (!lanemap && (op.off & 7) == 0) {
                switch (op.off >> 3) {
                    case 0: place_tiles<1, 0>(acc, e); break;
                    case 1: place_tiles<1, 1>(acc, e); break;
                    case 2: place_tiles<1, 2>(acc, e); break;
                    case 3: place_tiles<1, 3>(acc, e); break;
                    case 4: place_tiles<1, 4>(acc, e); break;
                    case 5: place_tiles<1, 5>(acc, e); break;
                    case 6: place_tiles<1, 6>(acc, e); break;
                    default: place_tiles<1, 7>(acc, e); break;
                }
            } else {
                // general placement through the slot's (now dead) input vector
                double *S = ring.vec[s];
                __syncwarp();
                const int width = (op.kind == BF_OP_TILE_N) ? op.R : op.C;
                const int MT = (width + 7) >> 3;
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
                    if (mt < MT && q < QACT)
                        *reinterpret_cast<double2 *>(S + (8 * mt + g) * NR + 2 * q) =
                            make_double2(e[0][mt][0], e[0][mt][1]);
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int sl = 8 * j + g;
                    const int src = lanemap ? (int)ring.map[s][sl] : sl - op.off;
                    if (q < QACT && src >= 0 && src < width) {
                        const double2 v = *reinterpret_cast<const double2 *>(S + src * NR + 2 * q);
                        acc[0][j][0] += v.x;
                        acc[0][j][1] += v.y;
                    }
                }
                __syncwarp();
            }
            if (f & BF_CF_ADD) {
                // folded index add: entry jj adds into slot addoff + jj
                const int addR = (f >> 8) & 0xff, addoff = (f >> 16) & 0xff;
                const double *A = ring.tile[s] + fold_at(addR);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int jj = 8 * j + g - addoff;
                    if (q < QACT && jj >= 0 && jj < addR) {
                        const double2 v = *reinterpret_cast<const double2 *>(A + jj * NR + 2 * q);
                        acc[0][j][0] += v.x;
                        acc[0][j][1] += v.y;
                    }
                }
            }
        }
        if (f & BF_CF_LAST) {
            const int nout = mb.w & 0xff;
            const int stride = (mb.w >> 8) ? (mb.w >> 8) : 1;
            double *o = a.arena + ((int64_t)mb.z + (int64_t)g * stride) * NR + 2 * q;
            const int64_t step = (int64_t)stride * (8 * NR);
            const int lim = q < QACT ? nout - g : 0;   // slot 8j + g < nout
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (8 * j < lim)
                    *reinterpret_cast<double2 *>(o) = make_double2(acc[0][j][0], acc[0][j][1]);
                o += step;
                acc[0][j][0] = acc[0][j][1] = 0.0;
            }
        }
        __syncwarp();
        while (i0 >= 0 && seq_issue - seq_use < kStages) issue_next();
    }
}

// ------------------------------------------------------------ group engine
// Batched fields with many fields per payload pass (BASELINE config 4, the
// "real dense contraction" of north_star (2)).  The warp engine above gives
// each warp its own op stream, so a staged tile meets only the 16 RHS of
// one wide entry (8 complex fields) and 64 fields stream the payload 8
// times at 4 flop/B — below the fp64 ridge.  Here kGW warps form a group
// that walks ONE op stream through ONE ring: warp w of the group computes
// RHS [16w, 16w + 16) of every 64-wide arena entry (fields 8w .. 8w+7 of a
// 32-field pass), so each tile fetched from HBM feeds kGW x 16 RHS and 64
// fields need 2 payload passes.  Warp 0 of the group is also the producer:
// it claims tasks, issues the tile and the 512-byte input entries as TMA
// bulk copies (per-lane bulk copies for gathered inputs) into a free slot,
// and publishes the op record in the slot; a slot is refilled only after
// all kGW warps have released it (empty mbarrier, kGW arrivals).  Per-warp
// accumulation, summation order and stores are those of the warp engine,
// so results are bitwise those of the 16-wide path.  Plans with
// regenerated tiles use the 16-wide path (regen is a per-warp step).
// 3 groups x 2 slots (12 warps at 168 registers, ~130 B of spills) measured
// 2284 fields/s on C4 against 2080 for 2 groups x 3 slots (8 warps at 230
// registers) and 2076 for 2 x 2: warps matter, ring depth does not
#ifndef BF_GROUPS
#define BF_GROUPS 3
#endif
#ifndef BF_GSLOTS
#define BF_GSLOTS 2
#endif
constexpr int kGW = 4;                  // warps per group
constexpr int kGroups = BF_GROUPS;      // groups per CTA (register-bound)
constexpr int kGS = BF_GSLOTS;          // ring slots per group
constexpr int kGNR = kGW * 16;          // doubles per arena entry (BFSHT_FIELDS_NRHS)
constexpr uint8_t kOpStop = 0xff;       // end-of-stream record

struct alignas(128) GroupRing {
    double tile[kGS][kTileDoubles];
    double vec[kGS][BF_T * kGNR];
    int8_t map[kGS][BF_SLOTS];
    double zero[16];
    bf_op meta[kGS];
    int4 tmeta[kGS];
    unsigned long long full[kGS], empty[kGS];
};
struct alignas(128) GroupScratch {
    double s[BF_T * 16];                // per-warp placement staging
};
constexpr size_t kGroupSmem = sizeof(GroupRing) * kGroups + sizeof(GroupScratch) * kGroups * kGW;
static_assert(kGroupSmem <= 227 * 1024, "group ring exceeds shared memory");

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Producer side of one op into slot s (whole producer warp).
__device__ __forceinline__ void group_issue(const StageArgs &a, GroupRing &ring, int s,
                                            const Rec &r, int gsrc, int lane) {
    const bf_op &op = r.op;
    const bool gather = (op.flags & BF_OPF_GATHER) != 0;
    const bool lanemap = (op.flags & BF_OPF_LANEMAP) != 0;
    constexpr uint32_t kEntry = kGNR * 8u;
    int nvec;
    uint32_t bytes = 0;
    if (op.kind == BF_OP_ADD) {
        nvec = op.R;
    } else {
        nvec = (op.kind == BF_OP_TILE_N) ? op.C : op.R;
        bytes += (uint32_t)bf_tile_doubles(op.R, op.C) * 8u;
    }
    int nsrc = 0;   // gathered entries present (sources < 0 are skipped)
    if (gather) {
        const unsigned has = __ballot_sync(0xffffffffu, lane < nvec && gsrc >= 0);
        nsrc = __popc(has);
    }
    bytes += gather ? (uint32_t)nsrc * kEntry : (uint32_t)nvec * kEntry;
    if (lanemap) bytes += BF_SLOTS;
    if (gather && lane < nvec && gsrc < 0) {
        // absent source (index-add lanes without a skeleton entry): zeros,
        // written before the arrive that publishes the slot
        double *d = ring.vec[s] + lane * kGNR;
        for (int k = 0; k < kGNR; k += 2)
            *reinterpret_cast<double2 *>(d + k) = make_double2(0.0, 0.0);
    }
    __syncwarp();
    if (lane == 0) {
        ring.meta[s] = op;
        ring.tmeta[s] = make_int4(r.out, r.nout, r.last, 0);
        mbar_arrive_tx(&ring.full[s], bytes);
    }
    // the slot was last read through the generic proxy; order those reads
    // before this thread's bulk (async-proxy) writes into it
    fence_proxy_async();
    __syncwarp();
    if (op.kind != BF_OP_ADD && lane == 0)
        bulk_g2s(ring.tile[s], a.tiles + op.tile, (uint32_t)bf_tile_doubles(op.R, op.C) * 8u,
                 &ring.full[s]);
    if (gather) {
        if (lane < nvec && gsrc >= 0)
            bulk_g2s(ring.vec[s] + lane * kGNR, a.arena + (int64_t)gsrc * kGNR, kEntry,
                     &ring.full[s]);
    } else if (lane == 1 && nvec > 0) {
        bulk_g2s(ring.vec[s], a.arena + (int64_t)op.in * kGNR, (uint32_t)nvec * kEntry,
                 &ring.full[s]);
    }
    if (lanemap && lane == 2)
        bulk_g2s(ring.map[s], a.maps + (int64_t)op.aux * BF_SLOTS, BF_SLOTS, &ring.full[s]);
}

__global__ void __launch_bounds__(kGroups * kGW * 32, 1) alt_group_kernel(StageArgs a) {
    constexpr int NR = 16, G = 2, QACT = 4;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = warp / kGW, wg = warp % kGW;
    GroupRing &ring = reinterpret_cast<GroupRing *>(smem_raw)[gid];
    double *S = reinterpret_cast<GroupScratch *>(smem_raw + sizeof(GroupRing) * kGroups)[warp].s;
    {
        // zero the rings once (padded tile columns multiply stale entries,
        // which must be finite) and init the barriers
        double2 *z = reinterpret_cast<double2 *>(smem_raw);
        for (int i = threadIdx.x; i < (int)(kGroupSmem / sizeof(double2)); i += blockDim.x)
            z[i] = make_double2(0.0, 0.0);
        __syncthreads();
        if (wg == 0 && lane == 0) {
            for (int s = 0; s < kGS; ++s) {
                mbar_init(&ring.full[s], 1);
                mbar_init(&ring.empty[s], kGW);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    const int g = lane >> 2, q = lane & 3;
    const bool producer = wg == 0;

    Cursor cur;
    Rec q0, q1;
    int g0 = -1;
    uint32_t seq_issue = 0, seq_use = 0;
    bool stopped = false;
    if (producer) {
        cur.n = cur.i = 0;
        cur.base = cur.out = cur.nout = 0;
        cur.nt = bcast(claim_raw(a, lane));
        cur.raw = 0;
        if (cur.nt < a.ntasks) {
            cur.ntask = load_task(a, cur.nt);
            cur.raw = claim_raw(a, lane);
        }
        q0 = advance(a, cur, lane);
        g0 = gather_src(a, q0, lane);
        q1 = advance(a, cur, lane);
    }
    // producer: fill free slots; the stream ends with one stop record
    auto produce = [&]() {
        while (!stopped && seq_issue - seq_use < kGS) {
            const int s = seq_issue % kGS;
            if (seq_issue >= kGS) mbar_wait(&ring.empty[s], ((seq_issue / kGS) - 1) & 1u);
            if (q0.valid) {
                group_issue(a, ring, s, q0, g0, lane);
                q0 = q1;
                g0 = gather_src(a, q0, lane);
                q1 = advance(a, cur, lane);
            } else {
                if (lane == 0) {
                    ring.meta[s].kind = kOpStop;
                    mbar_arrive_tx(&ring.full[s], 0);
                }
                stopped = true;
            }
            ++seq_issue;
            __syncwarp();
        }
    };
    if (producer) produce();

    double acc[G][8][2];
#pragma unroll
    for (int gr = 0; gr < G; ++gr)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[gr][j][0] = acc[gr][j][1] = 0.0;

    for (;;) {
        const int s = seq_use % kGS;
        mbar_wait(&ring.full[s], (seq_use / kGS) & 1u);
        ++seq_use;
        const bf_op op = ring.meta[s];
        if (op.kind == kOpStop) break;
        const int4 tm = ring.tmeta[s];
        const double *V = ring.vec[s] + wg * 16;
        if (op.kind == BF_OP_ADD) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = 8 * j + g - op.off;
                if (q < QACT && jj >= 0 && jj < op.R) {
#pragma unroll
                    for (int gr = 0; gr < G; ++gr) {
                        const double2 v =
                            *reinterpret_cast<const double2 *>(V + jj * kGNR + gr * 8 + 2 * q);
                        acc[gr][j][0] += v.x;
                        acc[gr][j][1] += v.y;
                    }
                }
            }
        } else {
            double e[G][4][2];
            tile_product<NR, kGNR>(op, ring.tile[s], V, ring.zero, lane, e);
            const bool lanemap = (op.flags & BF_OPF_LANEMAP) != 0;
            if (!lanemap && (op.off & 7) == 0) {
                switch (op.off >> 3) {
                    case 0: place_tiles<G, 0>(acc, e); break;
                    case 1: place_tiles<G, 1>(acc, e); break;
                    case 2: place_tiles<G, 2>(acc, e); break;
                    case 3: place_tiles<G, 3>(acc, e); break;
                    case 4: place_tiles<G, 4>(acc, e); break;
                    case 5: place_tiles<G, 5>(acc, e); break;
                    case 6: place_tiles<G, 6>(acc, e); break;
                    default: place_tiles<G, 7>(acc, e); break;
                }
            } else {
                const int width = (op.kind == BF_OP_TILE_N) ? op.R : op.C;
                const int MT = (width + 7) >> 3;
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
                    if (mt < MT && q < QACT) {
#pragma unroll
                        for (int gr = 0; gr < G; ++gr)
                            *reinterpret_cast<double2 *>(S + (8 * mt + g) * NR + gr * 8 + 2 * q) =
                                make_double2(e[gr][mt][0], e[gr][mt][1]);
                    }
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int sl = 8 * j + g;
                    const int src = lanemap ? (int)ring.map[s][sl] : sl - op.off;
                    if (q < QACT && src >= 0 && src < width) {
#pragma unroll
                        for (int gr = 0; gr < G; ++gr) {
                            const double2 v =
                                *reinterpret_cast<const double2 *>(S + src * NR + gr * 8 + 2 * q);
                            acc[gr][j][0] += v.x;
                            acc[gr][j][1] += v.y;
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (tm.z) {
            const int nout = tm.y & 0xff;
            const int stride = (tm.y >> 8) ? (tm.y >> 8) : 1;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int sl = 8 * j + g;
                if (q < QACT && sl < nout) {
                    double *o = a.arena + ((int64_t)tm.x + (int64_t)sl * stride) * kGNR + wg * 16 +
                                2 * q;
#pragma unroll
                    for (int gr = 0; gr < G; ++gr)
                        *reinterpret_cast<double2 *>(o + gr * 8) =
                            make_double2(acc[gr][j][0], acc[gr][j][1]);
                }
#pragma unroll
                for (int gr = 0; gr < G; ++gr) acc[gr][j][0] = acc[gr][j][1] = 0.0;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ring.empty[s]);
        if (producer) produce();
    }
}

}  // namespace

// All stages of one direction over a 64-wide arena (group engine).
int bf_alt_apply_group(bfsht_plan *pl, int dir, double *arena, cudaStream_t st) {
    const std::vector<int64_t> &b = pl->stages[dir];
    const int nst = (int)b.size() - 1;
    if (pl->ncounters < nst) {
        bfsht_set_error("plan counters not allocated");
        return -3;
    }
    int rc = bf_ensure_smem((const void *)alt_group_kernel, (int)kGroupSmem);
    if (rc) return rc;
    BF_CUDA(cudaMemsetAsync(pl->counters, 0, sizeof(int) * nst, st));
    for (int s = 0; s < nst; ++s) {
        if (b[s + 1] <= b[s]) continue;
        StageArgs a;
        a.tiles = pl->tiles;
        a.ops = pl->ops;
        a.idx = pl->idx;
        a.maps = pl->maps;
        a.tasks = pl->tasks;
        a.arena = arena;
        a.t0 = b[s];
        a.ntasks = b[s + 1] - b[s];
        a.counter = pl->counters + s;
        a.rec = pl->rec;
        a.xpos = pl->xpos;
        std::memcpy(&a.mag_min, &pl->info[22], sizeof(double));
        const int64_t want = (a.ntasks + kGroups - 1) / kGroups;
        const int grid = (int)(want < pl->sm_count ? want : pl->sm_count);
        alt_group_kernel<<<grid, kGroups * kGW * 32, kGroupSmem, st>>>(a);
        BF_CUDA(cudaGetLastError());
        pl->launches += 1;
    }
    return 0;
}

// reset: zero the stage's task counter first (single-stage calls); the
// whole-direction paths zero every stage counter with one memset instead
// One ALT kernel launch; pdl = programmatic dependent launch on the previous
// kernel in the stream (an ALT stage of the same direction).
static cudaError_t launch_alt(const void *kern, int grid, int block, size_t smem, cudaStream_t st,
                              void *args_struct, bool pdl) {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    void *args[1] = {args_struct};
    return cudaLaunchKernelExC(&cfg, kern, args);
}

static bool pdl_enabled() {
    static const int on = [] {
        const char *v = std::getenv("BFSHT_PDL");
        return (v && *v) ? std::atoi(v) : 1;
    }();
    return on != 0;
}

template <int NR>
static int launch_stage(bfsht_plan *pl, int64_t t0, int64_t t1, int *counter, double *arena,
                        cudaStream_t st, int max_ctas, bool reset, bool pdl = false) {
    constexpr int W = Width<NR>::WARPS;
    const size_t smem = sizeof(WarpRing<NR>) * W;
    int rc = bf_ensure_smem((const void *)alt_stage_kernel<NR>, (int)smem);
    if (rc) return rc;
    StageArgs a;
    a.tiles = pl->tiles;
    a.ops = pl->ops;
    a.idx = pl->idx;
    a.maps = pl->maps;
    a.tasks = pl->tasks;
    a.arena = arena;
    a.t0 = t0;
    a.ntasks = t1 - t0;
    a.counter = counter;
    a.rec = pl->rec;
    a.xpos = pl->xpos;
    std::memcpy(&a.mag_min, &pl->info[22], sizeof(double));
    if (reset) BF_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    int64_t want = (a.ntasks + W - 1) / W;
    const int cap = (max_ctas > 0 && max_ctas < pl->sm_count) ? max_ctas : pl->sm_count;
    int grid = (int)(want < cap ? want : cap);
    BF_CUDA(launch_alt((const void *)alt_stage_kernel<NR>, grid, W * 32, smem, st, &a, pdl));
    pl->launches += 1;
    return 0;
}

// ---------------------------------------------------------- chain schedule
static int env_int(const char *name, int dflt) {
    const char *v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

// The schedule itself is built on the host by bfsht_chain_schedule
// (packer.cpp); this uploads it.  Environment knobs, read when a plan is
// created: BFSHT_CHAIN = 0 every stage on alt_stage_kernel, 1 (default)
// stages holding gather / lane-map ops (the butterfly chain; stage 0 also
// carries the low-rank cores) on alt_chain_kernel, 2 every stage without
// regenerated tiles; BFSHT_CHAIN_BUNDLES = bundles per warp (default 8);
// BFSHT_CHAIN_CFIX = fixed cost of an op in byte equivalents for the bundle
// balance (default 3072).
int bf_chain_build(bfsht_plan *pl, const bf_op *ops, const bf_task *tasks) {
    const int mode = env_int("BFSHT_CHAIN", 1);
    if (!ops || !tasks || mode <= 0) return 0;
    const int per_warp = std::max(1, env_int("BFSHT_CHAIN_BUNDLES", 8));
    const int cfix = std::max(0, env_int("BFSHT_CHAIN_CFIX", 3072));
    for (int d = 0; d < 2; ++d) {
        const std::vector<int64_t> &b = pl->stages[d];
        const int nst = (int)b.size() - 1;
        pl->chain[d].assign(nst > 0 ? nst : 0, bfsht_plan::ChainStage());
        if (nst <= 0) continue;
        bfsht_chain_sched *sc = nullptr;
        if (bfsht_chain_schedule(ops, tasks, b.data(), nst, pl->sm_count * kWarps, mode, per_warp,
                                 cfix, &sc)) {
            bfsht_set_error(std::string("chain schedule: ") + bfsht_host_last_error());
            return -3;
        }
        const void *recs = nullptr;
        const int32_t *bund = nullptr;
        const int64_t *st = nullptr;
        int64_t nrec = 0, nbund = 0;
        bfsht_chain_sched_arrays(sc, &recs, &nrec, &bund, &nbund, &st);
        if (nrec > 0) {
            void *dr = nullptr, *db = nullptr;
            if (cudaMalloc(&dr, (size_t)nrec * sizeof(bf_crec)) != cudaSuccess ||
                cudaMalloc(&db, (size_t)nbund * sizeof(int32_t)) != cudaSuccess ||
                cudaMemcpy(dr, recs, (size_t)nrec * sizeof(bf_crec), cudaMemcpyHostToDevice) !=
                    cudaSuccess ||
                cudaMemcpy(db, bund, (size_t)nbund * sizeof(int32_t), cudaMemcpyHostToDevice) !=
                    cudaSuccess) {
                if (dr) cudaFree(dr);
                if (db) cudaFree(db);
                bfsht_chain_sched_free(sc);
                bfsht_set_error("chain schedule upload failed");
                return -2;
            }
            pl->owned.push_back(dr);
            pl->owned.push_back(db);
            pl->chain_rec[d] = dr;
            pl->chain_bund[d] = (int32_t *)db;
            for (int s = 0; s < nst; ++s) {
                pl->chain[d][s].b0 = st[4 * s];
                pl->chain[d][s].nb = (int)st[4 * s + 1];
                pl->chain[d][s].nrec = st[4 * s + 2];
                pl->chain[d][s].nfold = st[4 * s + 3];
            }
        }
        bfsht_chain_sched_free(sc);
    }
    return 0;
}

static int launch_chain(bfsht_plan *pl, int dir, int s, int *counter, cudaStream_t st,
                        bool reset, bool pdl = false) {
    const bfsht_plan::ChainStage &c = pl->chain[dir][s];
    const size_t smem = sizeof(ChainRing) * kWarps;
    int rc = bf_ensure_smem((const void *)alt_chain_kernel, (int)smem);
    if (rc) return rc;
    ChainArgs a;
    a.tiles = pl->tiles;
    a.rec = (const int4 *)pl->chain_rec[dir];
    a.bund = pl->chain_bund[dir] + c.b0;
    a.idx = pl->idx;
    a.maps = pl->maps;
    a.arena = pl->arena;
    a.nb = c.nb;
    a.counter = counter;
    if (reset) BF_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), st));
    const int64_t want = ((int64_t)c.nb + kWarps - 1) / kWarps;
    const int grid = (int)(want < pl->sm_count ? want : pl->sm_count);
    BF_CUDA(launch_alt((const void *)alt_chain_kernel, grid, kWarps * 32, smem, st, &a, pdl));
    pl->launches += 1;
    return 0;
}

static bool is_chain_stage(const bfsht_plan *pl, int dir, int s) {
    return s < (int)pl->chain[dir].size() && pl->chain[dir][s].nb > 0;
}

int bf_run_stage(bfsht_plan *pl, int dir, int stage, cudaStream_t st) {
    const std::vector<int64_t> &b = pl->stages[dir];
    if (b[stage + 1] <= b[stage]) return 0;
    if (is_chain_stage(pl, dir, stage))
        return launch_chain(pl, dir, stage, pl->counters + stage, st, true);
    return launch_stage<BF_NRHS>(pl, b[stage], b[stage + 1], pl->counters + stage, pl->arena, st,
                                 0, true);
}

// All stages of one direction over a wide (16 RHS per entry) arena.
int bf_alt_apply_wide(bfsht_plan *pl, int dir, double *arena, cudaStream_t st) {
    const std::vector<int64_t> &b = pl->stages[dir];
    const int nst = (int)b.size() - 1;
    if (pl->ncounters < nst) {
        bfsht_set_error("plan counters not allocated");
        return -3;
    }
    BF_CUDA(cudaMemsetAsync(pl->counters, 0, sizeof(int) * nst, st));
    for (int s = 0; s < nst; ++s) {
        if (b[s + 1] <= b[s]) continue;
        int rc =
            launch_stage<BF_WIDE_NRHS>(pl, b[s], b[s + 1], pl->counters + s, arena, st, 0, false);
        if (rc) return rc;
    }
    return 0;
}

int bf_alt_apply(bfsht_plan *pl, int dir, cudaStream_t st) {
    const std::vector<int64_t> &b = pl->stages[dir];
    const int nst = (int)b.size() - 1;
    if (pl->ncounters < nst) {
        bfsht_set_error("plan counters not allocated");
        return -3;
    }
    BF_CUDA(cudaMemsetAsync(pl->counters, 0, sizeof(int) * nst, st));
    bool first = true;
    for (int s = 0; s < nst; ++s) {
        if (b[s + 1] <= b[s]) continue;
        // every stage after the first follows an ALT kernel in the stream
        const bool pdl = !first && pdl_enabled();
        int rc = is_chain_stage(pl, dir, s)
                     ? launch_chain(pl, dir, s, pl->counters + s, st, false, pdl)
                     : launch_stage<BF_NRHS>(pl, b[s], b[s + 1], pl->counters + s, pl->arena, st,
                                             0, false, pdl);
        if (rc) return rc;
        first = false;
    }
    return 0;
}
