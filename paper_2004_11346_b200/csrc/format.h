/*
 * Device plan format shared by the host packer (packer.cpp) and the CUDA
 * apply engine (engine.cu).  Plain C so it can sit under the C ABI.
 *
 * Every payload value of a plan (dense turning blocks, low-rank u*diag(s)
 * and v, butterfly ID interpolation blocks and middle skeleton blocks)
 * lives in one fp64 "tile store" as R x C tiles (R, C <= 32), each tile
 * contiguous and 128-byte aligned, stored as 4x4 blocks (zero padded to
 * multiples of 4): block (r/4, c/4) at ((r/4)*C4 + c/4)*16, element
 * (r%4)*4 + c%4 inside it.  Every fp64 tensor-core fragment load
 * (mma.m8n8k4.f64) then touches one 128-byte block per half-warp, for the
 * A operand of both tile products:
 *   N-mode  y += A x     (apply)
 *   T-mode  x += A^T y   (apply transpose)
 * so one stored copy serves the forward ALT (A x) and the inverse ALT
 * (A^T y) — the reference's "one plan serves both directions"
 * (pkg/src/bfsht/alt.py:1-9).
 *
 * All vectors (coefficient halves, node halves, butterfly intermediates,
 * low-rank cores, butterfly block outputs) live in one "vector arena" of
 * NRHS-double entries addressed by int32 entry index; NRHS = 4 carries
 * (Re, Im) of +m and -m, which share one plan (pkg/src/bfsht/sht.py:146).
 *
 * A task produces <= 32 consecutive arena entries as a fixed-order sum of
 * ops, so results are deterministic run to run (no atomics).  Tasks are
 * grouped in stages; a stage only reads entries written by earlier stages.
 */
#ifndef BFSHT_FORMAT_H
#define BFSHT_FORMAT_H
#include <stdint.h>

#define BF_T 32          /* max tile edge; dense group tasks write <= 32 entries */
#define BF_SLOTS 64      /* max outputs per task (butterfly scatter tasks) */
#define BF_NRHS 4        /* doubles per arena entry (SHT path) */
#define BF_WIDE_NRHS 16  /* doubles per entry of the batched-fields arena */

enum bf_op_kind {
    BF_OP_TILE_N = 0,    /* lanes = tile rows, inputs = C entries  */
    BF_OP_TILE_T = 1,    /* lanes = tile cols, inputs = R entries  */
    BF_OP_ADD = 2        /* lanes [off, off+R) += arena[src]       */
};

enum bf_op_flags {
    BF_OPF_GATHER = 1,   /* inputs through idx[in + i], else in + i (idx < 0: none) */
    BF_OPF_LANEMAP = 2,  /* outputs through maps[aux*32 + slot] (tile lane or -1) */
    BF_OPF_REGEN = 4     /* `tile` is a seed block: regenerate the values (f1) */
};

/* Seed block of a regenerated dense tile (R rows, C <= 32 columns):
 *   double[0]: int32 first row r_a (index into x_pos), int32 unused
 *   double[1]: int64 offset (doubles) in the coefficient table of the step
 *              leaving the tile's first degree: alpha at [+0], beta at [+1],
 *              next step at [+2], [+3], ...
 *   double[2 + 3r .. 4 + 3r]: row r's p_prev, p_cur and exponent e (exact,
 *              as a double) at the tile's first degree (column 0)
 *   when C > 16, double[2 + 3R + 3r .. 4 + 3R + 3r]: the same state at
 *              column 16 (the engine runs the two column halves as two
 *              independent recurrence chains per row)
 * padded to a multiple of 16 doubles (128 B). */
#define BF_SEED_SPLIT 16
static inline
#ifdef __CUDACC__
__host__ __device__
#endif
int bf_seed_chains(int C) { return C > BF_SEED_SPLIT ? 2 : 1; }

static inline
#ifdef __CUDACC__
__host__ __device__
#endif
int64_t bf_seed_doubles(int R, int C) {
    return ((int64_t)(2 + 3 * R * bf_seed_chains(C)) + 15) / 16 * 16;
}

typedef struct {
    int64_t tile;        /* element offset of the tile in the tile store  */
    int32_t in;          /* arena entry (contiguous) or idx offset (gather) */
    int32_t aux;         /* lane-map index when BF_OPF_LANEMAP; recurrence-
                            table offset of the tile's first step when
                            BF_OPF_REGEN                                  */
    uint8_t kind, R, C, off;
    uint8_t flags, pad0;
    uint16_t pad1;
} bf_op;                 /* 24 bytes */

typedef struct {
    int32_t op_begin;
    int32_t op_count;
    int32_t out;         /* first arena entry written */
    int32_t nout;        /* entries written (<= 32) */
} bf_task;               /* 16 bytes */

/* Chain record: one op of a chain stage (small butterfly gather / scatter
 * and low-rank-core tasks), re-encoded at plan-upload time from bf_op /
 * bf_task for alt_chain_kernel (engine.cu).  Records of a task are
 * consecutive; tasks are grouped in cost-balanced bundles that warps
 * claim.  An index add that directly follows a tile op of its task rides
 * on that op's record ("folded": BF_CF_ADD, add_in / addR / addoff), when
 * the tile leaves the last BF_T entries of its ring slot free; a second add
 * that continues the first (next sources, next slots) extends the fold to
 * up to 2 BF_T entries when the tile leaves twice that free. */
enum bf_crec_flags {
    BF_CF_LAST = 8,      /* last op of its task: store the outputs */
    BF_CF_ADD = 16       /* folded index add (gathered through idx[add_in + j]) */
};
#define BF_FOLD_AT 896   /* doubles: where the folded add's entries land in the tile slot */

typedef struct {
    uint32_t tile;       /* tile offset in 16-double (128-byte) units */
    int32_t in;          /* as bf_op.in */
    int32_t aux;         /* lane-map index */
    uint8_t kind, R, C, off;
    uint8_t flags, addR, addoff, pad;
    int32_t add_in;      /* idx offset of the folded add's sources */
    int32_t out;         /* task: first arena entry written */
    int32_t nout;        /* task: entries written | stride << 8 */
} bf_crec;               /* 32 bytes */

/* per (order, parity) half: where its vectors live */
typedef struct {
    int32_t x;           /* coefficient half: ncols entries (fwd in, inv out) */
    int32_t y;           /* node half: n entries (fwd out, inv in)            */
    int32_t ncols;       /* 0 when this parity half is absent                 */
    int32_t m;
} bf_half;

#ifdef __CUDACC__
#define BF_HD __host__ __device__
#else
#define BF_HD
#endif

static inline BF_HD int64_t bf_tile_doubles(int R, int C) {
    return (int64_t)((R + 3) / 4) * ((C + 3) / 4) * 16;
}
static inline BF_HD int64_t bf_tile_index(int r, int c, int C4) {
    return ((int64_t)(r >> 2) * C4 + (c >> 2)) * 16 + (r & 3) * 4 + (c & 3);
}

#endif
