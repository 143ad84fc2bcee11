/*
 * bfsht-b200 C ABI.
 *
 * Drop-in boundary for the apply phase of the reference package `bfsht`
 * (arXiv 2004.11346).  The reference has no FFI; its boundary is the set of
 * Python apply functions, which paper_2004_11346_b200/api.py mirrors with the
 * same names, argument meaning and ValueError messages on top of this ABI:
 *
 *   reference (pkg/src/bfsht/…)                 replaced by
 *   ------------------------------------------  ---------------------------------
 *   alt.py:264  alt_forward(plan, coeffs)        bfsht_alt_apply(.., BFSHT_FORWARD)
 *   alt.py:275  alt_inverse(plan, column)        bfsht_alt_apply(.., BFSHT_INVERSE)
 *   alt.py:197  _apply_half  (+ butterfly.py:275
 *               idbf_apply, lowrank.py:196)      stages of bfsht_alt_apply
 *   alt.py:211  _apply_half_transpose (+ :285
 *               idbf_apply_transpose, :200)      stages of bfsht_alt_apply
 *   sht.py:137  sht_forward(plan, coeffs)         bfsht_sht_forward
 *   sht.py:151  sht_inverse(plan, grid_values)    bfsht_sht_inverse
 *   sht.py:148,161 np.fft.ifft/fft(axis=1)       bfsht_dft_rows
 *   alt.py:57 AltPlan / butterfly.py:66 payloads  bfsht_pack_plan (host) +
 *                                                bfsht_plan_upload (device)
 *
 * Conventions: plain pointers and sizes only; device pointers are raw CUDA
 * device addresses, `stream` is a cudaStream_t passed as void*.  Every call
 * returns 0 on success or a negative code, with a message retrievable from
 * bfsht_last_error() (thread-local).  Device buffers created by the library
 * are owned by the handle; pointers passed in are borrowed.
 */
#ifndef BFSHT_B200_H
#define BFSHT_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFSHT_FORWARD 0
#define BFSHT_INVERSE 1

/* ---------------------------------------------------------------- host side
 * Plan manifest: the reference payload layout, flattened.  One entry per
 * retained block of every AltPlan half (pkg/src/bfsht/alt.py:57-73,
 * partition.py:189-204).  kind: 0 butterfly (butterfly.py:66-80, COO
 * factors, factors[0] applied first), 1 low-rank u diag(s) v^T
 * (lowrank.py:184-202), 2 dense h x w row-major (alt.py:183-187). */
typedef struct {
    int32_t order;              /* index into bfsht_manifest.m            */
    int32_t parity;             /* 0 odd, 1 even                          */
    int32_t kind;
    int32_t r0, r1, c0, c1;     /* Block.trim                             */
    int32_t rank;               /* low-rank r                             */
    const double *a, *b, *c;    /* dense: a; low-rank: u, s, v            */
    int32_t nfac, levels, middle;
    const int64_t *fshape;      /* 2*nfac                                 */
    const int64_t *fnnz;        /* nfac                                   */
    const int64_t *const *frows;
    const int64_t *const *fcols;
    const double *const *fvals;
} bfsht_block;

typedef struct {
    int32_t n;                  /* transform half-size N (2N nodes)       */
    int32_t norders;
    const int32_t *m;           /* order of each plan                     */
    const int32_t *ncols;       /* 2*norders: (odd, even) columns, 0=absent */
    int64_t nblocks;
    const bfsht_block *blocks;
    /* On-GPU regeneration of dense turning tiles.  A
     * fraction regen in [0, 1] of the full-height (32-row) tiles of kind-2
     * blocks is stored as recurrence seeds (per row: p_prev, p_cur, 2^e at
     * the tile's first degree, and at column 16 for tiles wider than 16;
     * format.h bf_seed_doubles) instead of values; the engine re-runs the
     * reference recurrence (kernels/_recur_cy.pyx:18-67) bit for bit.
     * Needs the nodes and start values below; regen = 0 ignores them. */
    double regen;
    const double *x_pos;        /* n positive nodes, ascending (AltMatrixSpec.x_pos) */
    const double *mant0;        /* norders x n: start mantissas (common.py:65-77) */
    const int32_t *exp0;        /* norders x n: start exponents                */
    double mag_min;             /* flush threshold of emitted values (MAG_MIN)  */
} bfsht_manifest;

typedef struct bfsht_packed bfsht_packed;   /* opaque host-side packed plan */

/* Pack a manifest into the device format (tiles + task lists).  Threads:
 * 0 = all host cores.  Returns 0 / negative. */
int bfsht_pack_plan(const bfsht_manifest *man, int threads,
                    bfsht_packed **out);
/* Sizes and host pointers of the packed arrays (for upload / inspection).
 * info[]: 0 tile doubles, 1 ops, 2 idx, 3 lane maps, 4 tasks,
 * 5 arena entries, 6 halves, 7 stages fwd, 8 stages inv,
 * 9 payload values (sum of stored reference values), 10 arena entry of the
 * row-major forward node array Yr[r][order][parity], 11 butterfly blocks, 12 low-rank blocks, 13 dense blocks,
 * 14 half-size N, 15 number of order plans, 16/17 index of the free
 * (dependency-free dense) stage of the forward/inverse direction,
 * 18 regenerated tiles, 19 reference values they replace (not stored),
 * 20 doubles of the recurrence-coefficient table, 21 doubles of x_pos,
 * 22 bit pattern of mag_min (double); 16, 17 and 23 are reserved (-1, -1,
 * 0) */
#define BFSHT_INFO_LEN 24
int bfsht_packed_info(const bfsht_packed *p, int64_t info[BFSHT_INFO_LEN]);
/* arrays: 0 tiles, 1 ops, 2 idx, 3 maps, 4 tasks, 5 halves, 6/7 stage
 * bounds fwd/inv, 8 recurrence coefficients (alpha, beta pairs), 9 x_pos,
 * 10, 11 reserved (NULL) */
int bfsht_packed_arrays(const bfsht_packed *p, const void *arrays[12]);
/* alpha_s, beta_s (s = 0 .. k_max-m-1) of the degree recurrence
 * (kernels/common.py:37-53), interleaved; for tests of the seed path. */
int bfsht_rec_coeffs(int64_t m, int64_t k_max, double *out);
/* Regenerate one seeded tile on the host with the reference step sequence
 * (range test after every step), chain by chain from the seed block's
 * states — the test oracle of the device generation: seed block at `seed`,
 * R x C tile in the 4x4-block layout into out (bf_tile_doubles(R, C)
 * doubles). */
int bfsht_regen_tile_host(const double *seed, int R, int C, const double *rec,
                          const double *x_pos, double mag_min, double *out);
void bfsht_packed_free(bfsht_packed *p);

/* Chain schedule (host side of the chain kernel, csrc/engine.cu): the
 * stages of one direction that are made of small tasks — the butterfly
 * factors' gather / scatter tasks (butterfly.py:275-292) and the low-rank
 * cores (lowrank.py:196-202) — re-encoded as one 32-byte record per op
 * (csrc/format.h bf_crec; an index add folded into the tile op it follows)
 * in cost-balanced bundles of whole tasks.  ops / tasks = arrays 1 and 4
 * of bfsht_packed_arrays, bounds = one direction's stage bounds (nstages +
 * 1), warps = worker warps of the device (SMs x 12); mode 1 = stages that
 * hold gather / lane-map ops, 2 = every stage without regenerated tiles,
 * 0 = none; per_warp = bundles per warp, cfix = fixed cost of an op in byte
 * equivalents.  bfsht_plan_upload / bfsht_plan_wrap call this themselves;
 * it is exported for tests and tools. */
typedef struct bfsht_chain_sched bfsht_chain_sched;
int bfsht_chain_schedule(const void *ops, const void *tasks, const int64_t *bounds, int nstages,
                         int warps, int mode, int per_warp, int cfix, bfsht_chain_sched **out);
/* recs: bf_crec records (nrecs), bund: bundle bounds (record indices; a
 * stage with nb bundles owns nb + 1 consecutive entries), stage: 4 int64
 * per stage = first bund entry, bundles (0: not a chain stage), records,
 * folded index adds. */
int bfsht_chain_sched_arrays(const bfsht_chain_sched *sc, const void **recs, int64_t *nrecs,
                             const int32_t **bund, int64_t *nbund, const int64_t **stage);
void bfsht_chain_sched_free(bfsht_chain_sched *sc);

const char *bfsht_last_error(void);
/* message of the last failed host-side call (packer, chain schedule) */
const char *bfsht_host_last_error(void);

/* ------------------------------------------------------------- device side */
typedef struct bfsht_plan bfsht_plan;       /* opaque device plan */

/* Upload a packed plan (arrays as returned by bfsht_packed_arrays) to the
 * current device.  A plan remembers its device: every call below that takes
 * a plan runs on that device and restores the caller's current device. */
int bfsht_plan_upload(const bfsht_packed *p, bfsht_plan **out);
/* Device arrays already resident (e.g. allocated through torch), borrowed:
 * dev[0..5] = tiles, ops, idx, maps, tasks, halves (bfsht_packed_arrays
 * order), dev[6] = vector arena (info[5] x 4 doubles), dev[7] = recurrence
 * coefficients, dev[8] = x_pos (both only read by regenerated tiles, may
 * be NULL when info[18] == 0), dev[9..11] reserved (NULL); host[5..7] =
 * host copies of halves and the two stage-bound arrays; host[1] and
 * host[4] = host copies of ops and tasks (optional, both or neither: with
 * them the butterfly-chain stages get their bundle schedule and run on the
 * chain kernel; without them every stage runs on the stage kernel — same
 * results, bit for bit). */
int bfsht_plan_wrap(const int64_t info[BFSHT_INFO_LEN], const void *const host[8],
                    void *const dev[12], bfsht_plan **out);
void bfsht_plan_free(bfsht_plan *pl);
/* Device pointer to the vector arena (info[5] entries x 4 doubles). */
double *bfsht_plan_arena(bfsht_plan *pl);

/* Run every ALT stage of one direction over the arena (inputs already in
 * the arena: coefficient halves for FORWARD, node halves for INVERSE). */
int bfsht_alt_apply(bfsht_plan *pl, int dir, void *stream);
/* One stage of one direction (stages run in order; for profiling). */
int bfsht_alt_stage(bfsht_plan *pl, int dir, int stage, void *stream);
/* Chain schedule of one stage: out[0] = bundles (0: the stage runs on the
 * stage kernel), out[1] = op records, out[2] = index adds folded into the
 * preceding tile op's record. */
int bfsht_plan_chain_info(bfsht_plan *pl, int dir, int stage, int64_t out[3]);

/* Per-order ALT boundary (alt_forward / alt_inverse for one or more plans):
 * in/out are device complex128 buffers laid out plan after plan, lengths
 * 2N-m (coefficients) and 2N (node values); weights = 2N quadrature
 * weights (device) for the inverse fold (alt.py:239-253). */
int bfsht_alt_orders(bfsht_plan *pl, int dir, const double *in, double *out,
                     const double *weights, void *stream);

/* Doubles per entry of the wide work arena used by the batched calls below:
 * `work` must hold info[5] (arena entries) x BFSHT_WIDE_NRHS doubles, zeroed
 * once before first use. */
#define BFSHT_WIDE_NRHS 16

/* Doubles per arena entry of bfsht_alt_fields' work buffer: info[5] x
 * BFSHT_FIELDS_NRHS doubles, zeroed once before first use. */
#define BFSHT_FIELDS_NRHS 64

/* Batched fields (SURVEY 8(b) "API extension", config 4): alt_forward /
 * alt_inverse on (2N-m, F) / (2N, F) complex128 arrays per plan (alt.py:
 * 264-282 applied column by column; the reference supports 2-D right-hand
 * sides only at idbf_apply, butterfly.py:275-292).  in/out are field-minor
 * (row-major L x F) and laid out plan after plan.  The payload is streamed
 * once per 32 fields (group engine: 4 warps share each staged tile), or
 * once per 8 fields when F <= 8 or the plan regenerates tiles. */
int bfsht_alt_fields(bfsht_plan *pl, int dir, int nfields, const double *in, double *out,
                     const double *weights, double *work, void *stream);

/* Batched SHT: `batch` (1..4) independent transforms in one pass of the
 * 16-RHS engine over the payload (each stored value read once for all of
 * them; transform b owns doubles [4b, 4b+4) of every wide entry).  FORWARD:
 * in = batch x 4N^2 coefficients (ShtCoeffs.pack() order each), out = batch
 * x 2N x (4N-1) grids; INVERSE the reverse (weights required).  Outputs are
 * bitwise those of `batch` bfsht_sht_forward / _inverse calls. */
int bfsht_sht_batch(bfsht_plan *pl, int dir, int batch, const double *in, double *out,
                    const double *weights, double *work, void *stream);
/* All ALT stages of one direction over a wide (BFSHT_WIDE_NRHS) arena with
 * inputs already in place (profiling / timing of the batched paths). */
int bfsht_alt_apply_wide(bfsht_plan *pl, int dir, double *work, void *stream);

/* Raw half apply: the matrix of one (order, parity) half — for a plan built
 * from a single ButterflyFactorization, exactly idbf_apply (FORWARD, K x) /
 * idbf_apply_transpose (INVERSE, K^T y) (butterfly.py:275-292).  in/out are
 * device real row-major (len x k) arrays; complex data is passed as
 * interleaved re/im columns. */
int bfsht_half_apply(bfsht_plan *pl, int dir, int half, int k, const double *in, double *out,
                     double *work, void *stream);

/* Full SHT on device buffers.  coeffs: flat m-major complex128, m from
 * -(2N-1) to 2N-1 (ShtCoeffs.pack(), sht.py:68-81); grid: 2N x (4N-1)
 * complex128 row-major, rows node-ascending.  The plan must hold orders
 * 0..2N-1 in order. */
int bfsht_sht_forward(bfsht_plan *pl, const double *coeffs, double *grid,
                      void *stream);
int bfsht_sht_inverse(bfsht_plan *pl, const double *grid, double *coeffs,
                      const double *weights, void *stream);

/* Batched length-L complex DFT of `rows` contiguous rows, unnormalized,
 * sign -1 (dir FORWARD, numpy fft) or +1 (INVERSE, L*ifft). */
int bfsht_dft_rows(int64_t L, int64_t rows, int dir, const double *in,
                   double *out, void *stream);

/* Factor construction: one parity half of the order-m ALT
 * matrix tabulated on GPU `device` — the entry evaluation of the reference
 * planner's oracle (pkg/src/bfsht/partition.py:91-169 over
 * kernels/_recur_cy.pyx:18-67), replacing the host table of
 * bfsht_legendre_half_table (libbfsht_host) bit for bit.  HOST pointers:
 * x, mant0, exp0 (n nodes), alpha, beta (offset + 2 (ncols-1) steps), out
 * (n * ncols doubles, written COLUMN-major: entry (r, j) at j * n + r). */
int bfsht_half_table_device(int device, int64_t m, int64_t offset, int64_t n, int64_t ncols,
                            const double *x, const double *alpha, const double *beta,
                            const double *mant0, const int32_t *exp0, double mag_min,
                            double *out);

/* Kernel launches issued on this plan since creation or the last reset. */
int64_t bfsht_plan_launches(bfsht_plan *pl);
int bfsht_reset_launches(bfsht_plan *pl);

/* ----------------------------------------- multi-GPU (order-sharded) SHT
 * A rank's plan holds its share of the orders.  Coefficient shard layout:
 * per plan order o, the +m vector at off[o] (2N-m values, k ascending) and,
 * for m > 0, the -m vector right after it.  Node-half entries are moved
 * between ranks with gather/scatter (4 doubles per entry, index lists into
 * the arena) around an NCCL all-to-all; the DFT stage then works on the
 * rank's row pairs r in [r_begin, r_begin + r_count): `halves` (device,
 * bf_half per (order, parity) for ALL 2N orders) locates each order's
 * entries in `ybuf` at .y + (r - r_begin); the local grid holds rows
 * n-r_begin-r_count .. n-r_begin-1 then n+r_begin .. n+r_begin+r_count-1. */
int bfsht_shard_pack(bfsht_plan *pl, const int64_t *off, const double *coeffs,
                     void *stream);
int bfsht_shard_unpack(bfsht_plan *pl, const int64_t *off, double *coeffs,
                       void *stream);
int bfsht_gather_entries(bfsht_plan *pl, const int32_t *idx, int64_t count,
                         double *out, void *stream);
int bfsht_scatter_entries(bfsht_plan *pl, const int32_t *idx, int64_t count,
                          const double *in, void *stream);
int bfsht_synth_rows(bfsht_plan *pl, const void *halves, const double *ybuf,
                     int64_t r_begin, int64_t r_count, double *grid,
                     void *stream);
int bfsht_anal_rows(bfsht_plan *pl, const void *halves, double *ubuf,
                    int64_t r_begin, int64_t r_count, const double *grid,
                    const double *weights, void *stream);

/* ------------------------------------------------ NCCL communicator + the
 * exchange (SURVEY 8(b) "bfsht_comm_init + bfsht_alltoall_transpose").
 * NCCL is loaded at run time (libnccl.so.2; the copy already in the process
 * if there is one).  One rank per GPU; call on the rank's current device. */
typedef struct bfsht_comm bfsht_comm;
#define BFSHT_COMM_ID_BYTES 128        /* = NCCL_UNIQUE_ID_BYTES */
/* Rank 0 creates the id (ncclGetUniqueId) and ships it to the other ranks
 * out of band (MPI, a TCP store, torch.distributed, ...). */
int bfsht_comm_unique_id(void *id);
int bfsht_comm_init(const void *id, int rank, int nranks, bfsht_comm **out);
void bfsht_comm_free(bfsht_comm *c);
/* Grouped ncclSend / ncclRecv: peer q gets send_counts[q] entries of
 * entry_doubles fp64 each (peers' runs back to back in send), and
 * recv_counts[q] entries from peer q land back to back in recv. */
int bfsht_alltoall_transpose(bfsht_comm *c, const double *send, const int64_t *send_counts,
                             double *recv, const int64_t *recv_counts, int64_t entry_doubles,
                             void *stream);

/* Host-only (no GPU needed): the orders of `rank` under the greedy LPT
 * split of m = 0..2N-1 on the cost 2N-m (orders: capacity 2N, may be NULL
 * to count), and the exchange layout of that rank: recv_layout = 4N
 * bf_half-like records {x, y, ncols, m} (entry (m, parity, r) of the
 * theta-major receive buffer at y + (r - r0) * x), send / recv entry counts
 * per peer (row pairs split contiguously: peer q owns [qN/P, (q+1)N/P)). */
int bfsht_shard_orders(int n, int nranks, int rank, int32_t *orders, int32_t *count);
int bfsht_exchange_layout(int n, int nranks, int rank, void *recv_layout, int64_t *send_counts,
                          int64_t *recv_counts);

/* The whole order-sharded SHT of one rank.  `pl` must hold exactly the
 * orders bfsht_shard_orders gives this rank (ascending); coefficients are
 * the shard layout (bfsht_shard_pack); the grid is this rank's 2*rc rows
 * (rows n-r0-rc .. n-r0-1, then n+r0 .. n+r0+rc-1).  Forward = shard pack,
 * ALT, all-to-all of the node halves (sent straight from the row-major Yr
 * array), fused synthesis/DFT of the rank's row pairs; inverse the reverse.
 * info: 0 r0, 1 rc, 2 shard coefficient count, 3 receive-buffer entries. */
typedef struct bfsht_sharded bfsht_sharded;
int bfsht_sharded_create(bfsht_plan *pl, bfsht_comm *comm, bfsht_sharded **out);
int64_t bfsht_sharded_info(const bfsht_sharded *s, int64_t info[4]);
int bfsht_sharded_forward(bfsht_sharded *s, const double *coeffs, double *grid, void *stream);
int bfsht_sharded_inverse(bfsht_sharded *s, const double *grid, double *coeffs,
                          const double *weights, void *stream);
void bfsht_sharded_free(bfsht_sharded *s);

#ifdef __cplusplus
}
#endif
#endif
