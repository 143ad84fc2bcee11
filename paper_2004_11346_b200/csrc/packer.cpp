// Host packer: reference-layout plan payloads -> device tile store + tasks.
//
// Input is the reference payload layout (pkg/src/bfsht/alt.py:57-73,
// butterfly.py:45-80, lowrank.py:184-202) flattened into a bfsht_manifest.
// Output is the format of format.h.  Nothing is approximated: every stored
// reference value lands in exactly one tile (plus explicit zeros where a
// dense block or ID tile has structural zeros), and the per-task op order
// fixes the summation order.
//
// Block kinds and how they become tasks (forward / inverse):
//  * dense turning block P: tiles cut on the absolute 32-row / 32-column
//    grid of its half matrix; N-mode ops in the row-group task of the node
//    half (forward, alt.py:207) and T-mode ops in the column-group task of
//    the coefficient half (inverse, alt.py:221).
//  * low-rank u diag(s) v^T (lowrank.py:196-202): s folded into u; a stage-0
//    task forms t = v^T x (fwd) or t = (u s)^T y (inv), the group tasks add
//    (u s) t or v t.
//  * butterfly chain (butterfly.py:275-292): every factor is put in its
//    "ID orientation" G (G = F for the V factors and the middle, G = F^T for
//    the U factors, whose COO is the transpose of a column ID,
//    butterfly.py:153-157).  G's rows are split into segments of rows that
//    share column support (one segment = one interpolative decomposition);
//    in a segment, columns holding a single exact 1.0 are identity
//    ("skeleton") entries and become index adds, the rest form a dense
//    interpolation block.  Applying G is a gather task per 32 segment rows
//    (N-mode tiles); applying G^T is a scatter task per 32 output columns
//    of the segment's column range (T-mode tiles through a lane map), with
//    all segments sharing a range summed in one task.  The same tiles serve
//    both, so a factor is stored once.  Depth-0 chains are dense blocks.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "bfsht_b200.h"
#include "format.h"
#include "recur.h"

static thread_local std::string g_err;

extern "C" const char *bfsht_host_last_error(void) { return g_err.c_str(); }

struct bfsht_packed {
    std::unique_ptr<double[]> tiles;
    int64_t n_tiles = 0;
    std::vector<bf_op> ops;
    std::vector<int32_t> idx;
    std::vector<int8_t> maps;
    std::vector<bf_task> tasks;
    std::vector<bf_half> halves;
    std::vector<int64_t> stage_bounds[2];
    int64_t arena = 0;
    int64_t payload_values = 0;
    int64_t n_bf = 0, n_lr = 0, n_dn = 0;
    int64_t n = 0, norders = 0;
    int32_t yr = 0;   // row-major forward node array Yr[r][order][parity]
    // regenerated dense tiles (f1)
    int64_t n_regen = 0, regen_values = 0;
    std::vector<double> rec;            // per order: (alpha, beta) for s = 0 .. 2N-m-1
    std::vector<double> xpos;
    double mag_min = 0.0;
    // dataflow schedule (one launch per direction): claim order per
    // direction (fwd then inv) and per task stage | (dep stage + 1) << 8
    std::vector<int32_t> flow;
    std::vector<int32_t> tinfo;
};

namespace {

struct TileJob {
    int64_t dst;
    int R, C;
    const double *src;
    int64_t rs, cs;  // element (r, c) = src[r*rs + c*cs]
};

struct SeedJob {
    int64_t dst;      // seed block offset in the tile store
    int h;            // half index (2 * order + parity)
    int r_a, R;       // rows
    int64_t c_a;      // first half column
    int C;            // columns
};

struct TaskBuild {
    int32_t out, nout;
    std::vector<bf_op> ops;
    double cost = 0.0;
};

// One interpolative decomposition (segment of G rows).
struct Segment {
    int64_t row0, rows;          // G rows [row0, row0+rows)
    std::vector<int64_t> dcols;  // dense columns, ascending
    std::vector<double> t;       // rows x dcols.size(), row-major
    std::vector<std::pair<int64_t, int64_t>> units;  // (row, col)
    int64_t cmin = -1, cmax = -1;
    int range = -1;
};

struct FactorSegs {
    int64_t nrows = 0, ncols = 0;              // G shape
    std::vector<Segment> segs;
    std::vector<std::pair<int64_t, int64_t>> ranges;  // [a, b) covering [0, ncols)
    std::vector<int> range_has_segs;
};

std::vector<std::pair<int64_t, int64_t>> cuts(int64_t a, int64_t b) {
    // [a, b) cut at absolute multiples of BF_T
    std::vector<std::pair<int64_t, int64_t>> out;
    int64_t x = a;
    while (x < b) {
        int64_t nx = std::min<int64_t>(b, (x / BF_T + 1) * BF_T);
        out.push_back({x, nx});
        x = nx;
    }
    return out;
}

// Split G (given as COO in G orientation) into ID segments.
void segment_factor(int64_t nr, int64_t nc, int64_t nnz, const int64_t *gr,
                    const int64_t *gc, const double *gv, FactorSegs &fs) {
    fs.nrows = nr;
    fs.ncols = nc;
    // CSR by row, columns ascending within a row
    std::vector<int64_t> rowptr(nr + 1, 0);
    for (int64_t e = 0; e < nnz; ++e) {
        if (gr[e] < 0 || gr[e] >= nr || gc[e] < 0 || gc[e] >= nc)
            throw std::runtime_error("factor triplet index out of range");
        rowptr[gr[e] + 1]++;
    }
    for (int64_t r = 0; r < nr; ++r) rowptr[r + 1] += rowptr[r];
    std::vector<int64_t> ccol(nnz);
    std::vector<double> cval(nnz);
    {
        std::vector<int64_t> fill(rowptr.begin(), rowptr.end() - 1);
        for (int64_t e = 0; e < nnz; ++e) {
            int64_t p = fill[gr[e]]++;
            ccol[p] = gc[e];
            cval[p] = gv[e];
        }
        std::vector<std::pair<int64_t, double>> tmp;
        for (int64_t r = 0; r < nr; ++r) {
            int64_t b = rowptr[r], e = rowptr[r + 1];
            if (e - b < 2) continue;
            tmp.clear();
            for (int64_t p = b; p < e; ++p) tmp.push_back({ccol[p], cval[p]});
            std::sort(tmp.begin(), tmp.end(),
                      [](auto &x, auto &y) { return x.first < y.first; });
            for (int64_t p = b; p < e; ++p) {
                ccol[p] = tmp[p - b].first;
                cval[p] = tmp[p - b].second;
            }
        }
    }
    // greedy segmentation on shared support
    std::vector<int64_t> stamp(nc, -1);
    std::vector<std::pair<int64_t, int64_t>> bounds;
    int64_t cur = -1, start = 0;
    bool cur_dense = false;
    for (int64_t r = 0; r < nr; ++r) {
        int64_t b = rowptr[r], e = rowptr[r + 1];
        bool unit_row = (e - b == 1 && cval[b] == 1.0);
        bool fresh;
        if (cur < 0) {
            fresh = true;
        } else if (e == b) {
            fresh = false;
        } else {
            int64_t overlap = 0;
            for (int64_t p = b; p < e; ++p) overlap += (stamp[ccol[p]] == cur);
            fresh = overlap == 0 && !(unit_row && !cur_dense);
        }
        if (fresh) {
            if (cur >= 0) bounds.push_back({start, r});
            cur = (int64_t)bounds.size();
            start = r;
            cur_dense = false;
        }
        for (int64_t p = b; p < e; ++p) stamp[ccol[p]] = cur;
        if (e > b && !unit_row) cur_dense = true;
    }
    if (nr > 0) bounds.push_back({start, nr});

    std::vector<int32_t> cnt(nc, 0);
    std::vector<double> lastv(nc, 0.0);
    std::vector<int64_t> lastr(nc, -1), pos(nc, -1);
    for (auto &bd : bounds) {
        Segment s;
        s.row0 = bd.first;
        s.rows = bd.second - bd.first;
        std::vector<int64_t> touched;
        for (int64_t r = bd.first; r < bd.second; ++r)
            for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) {
                int64_t c = ccol[p];
                if (cnt[c] == 0) touched.push_back(c);
                cnt[c]++;
                lastv[c] = cval[p];
                lastr[c] = r;
            }
        std::sort(touched.begin(), touched.end());
        for (int64_t c : touched) {
            if (cnt[c] == 1 && lastv[c] == 1.0)
                s.units.push_back({lastr[c], c});
            else
                s.dcols.push_back(c);
        }
        if (!touched.empty()) {
            s.cmin = touched.front();
            s.cmax = touched.back();
        }
        for (size_t j = 0; j < s.dcols.size(); ++j) pos[s.dcols[j]] = (int64_t)j;
        const int64_t nd = (int64_t)s.dcols.size();
        s.t.assign((size_t)(s.rows * nd), 0.0);
        for (int64_t r = bd.first; r < bd.second; ++r)
            for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) {
                int64_t c = ccol[p];
                if (!(cnt[c] == 1 && lastv[c] == 1.0))
                    s.t[(size_t)((r - bd.first) * nd + pos[c])] = cval[p];
            }
        for (int64_t c : touched) {
            cnt[c] = 0;
            pos[c] = -1;
        }
        fs.segs.push_back(std::move(s));
    }
    // column ranges: merged support intervals, gaps filled, covering [0, nc)
    std::vector<std::pair<int64_t, int64_t>> iv;
    for (auto &s : fs.segs)
        if (s.cmin >= 0) iv.push_back({s.cmin, s.cmax + 1});
    std::sort(iv.begin(), iv.end());
    std::vector<std::pair<int64_t, int64_t>> merged;
    for (auto &x : iv) {
        if (!merged.empty() && x.first < merged.back().second)
            merged.back().second = std::max(merged.back().second, x.second);
        else
            merged.push_back(x);
    }
    int64_t at = 0;
    for (auto &x : merged) {
        if (x.first > at) {
            fs.ranges.push_back({at, x.first});
            fs.range_has_segs.push_back(0);
        }
        fs.ranges.push_back(x);
        fs.range_has_segs.push_back(1);
        at = x.second;
    }
    if (at < nc) {
        fs.ranges.push_back({at, nc});
        fs.range_has_segs.push_back(0);
    }
    for (auto &s : fs.segs) {
        if (s.cmin < 0) continue;
        auto it = std::upper_bound(
            fs.ranges.begin(), fs.ranges.end(), std::make_pair(s.cmin, INT64_MAX));
        s.range = (int)(it - fs.ranges.begin()) - 1;
    }
}

struct Packer {
    static constexpr int kMaxTaskOps = 48;   // longer group tasks are split
    bfsht_packed &P;
    const bfsht_manifest &M;
    std::vector<TileJob> jobs;
    std::vector<SeedJob> seeds;
    std::vector<int64_t> rec_base;      // per order: offset of its table in P.rec
    int64_t regen_candidates = 0;
    std::vector<std::unique_ptr<std::vector<double>>> keep;  // temp sources
    // tasks by direction and stage
    std::vector<std::vector<TaskBuild>> stages[2];
    // per half: group ops (fwd row groups over Y, inv col groups over X)
    std::vector<std::vector<std::vector<bf_op>>> fwd_groups, inv_groups;  // dense tiles
    std::vector<std::vector<std::vector<bf_op>>> fwd_other, inv_other;    // low-rank, butterfly

    Packer(bfsht_packed &p, const bfsht_manifest &m) : P(p), M(m) {}

    int32_t alloc_entries(int64_t n) {
        int64_t at = P.arena;
        P.arena += n;
        if (P.arena > INT32_MAX) throw std::runtime_error("vector arena exceeds int32");
        return (int32_t)at;
    }
    int64_t alloc_tile(int R, int C, const double *src, int64_t rs, int64_t cs) {
        int64_t at = P.n_tiles;
        P.n_tiles += bf_tile_doubles(R, C);
        jobs.push_back({at, R, C, src, rs, cs});
        return at;
    }
    std::vector<TaskBuild> &stage(int dir, int s) {
        if ((int)stages[dir].size() <= s) stages[dir].resize(s + 1);
        return stages[dir][s];
    }
    static bf_op mk(int kind, int64_t tile, int32_t in, int R, int C, int off,
                    int flags = 0, int32_t aux = 0) {
        bf_op o;
        std::memset(&o, 0, sizeof(o));
        o.tile = tile;
        o.in = in;
        o.aux = aux;
        o.kind = (uint8_t)kind;
        o.R = (uint8_t)R;
        o.C = (uint8_t)C;
        o.off = (uint8_t)off;
        o.flags = (uint8_t)flags;
        return o;
    }
    static double op_cost(const bf_op &o) {
        if (o.kind == BF_OP_ADD) return 32.0 * o.R;
        return 8.0 * o.R * o.C + 32.0 * (o.kind == BF_OP_TILE_N ? o.C : o.R);
    }
    int32_t push_idx(const std::vector<int32_t> &v) {
        int64_t at = (int64_t)P.idx.size();
        P.idx.insert(P.idx.end(), v.begin(), v.end());
        if ((int64_t)P.idx.size() > INT32_MAX) throw std::runtime_error("idx exceeds int32");
        return (int32_t)at;
    }
    int32_t push_map(const int8_t *m) {
        int64_t at = (int64_t)P.maps.size() / BF_SLOTS;
        P.maps.insert(P.maps.end(), m, m + BF_SLOTS);
        return (int32_t)at;
    }
    void add_task(int dir, int s, int32_t out, int32_t nout, std::vector<bf_op> &&ops) {
        TaskBuild t;
        t.out = out;
        t.nout = nout;
        // the engine consumes tasks as op streams: an empty task carries
        // one no-op add so it still emits its (zero) outputs
        if (ops.empty()) ops.push_back(mk(BF_OP_ADD, 0, 0, 0, 0, 0));
        for (auto &o : ops) t.cost += op_cost(o);
        t.ops = std::move(ops);
        stage(dir, s).push_back(std::move(t));
    }

    // ---------------------------------------------------------- dense
    // Regeneration choice for one tile of a turning block: full-height
    // tiles only (one recurrence chain per lane covers 32 rows), spread
    // evenly over the candidates in packing order.
    // debugging knob: BFSHT_REGEN_COLS=full|partial restricts regeneration
    // to full-width (32-column) or narrower tiles
    static bool regen_cols_ok(int C) {
        static const char *v = std::getenv("BFSHT_REGEN_COLS");
        if (!v || !*v) return true;
        return std::strcmp(v, "full") == 0 ? C == BF_T : C < BF_T;
    }

    bool want_regen(int R) {
        if (M.regen <= 0.0 || R != BF_T) return false;
        const double f = M.regen >= 1.0 ? 1.0 : M.regen;
        const int64_t k = regen_candidates++;
        return (int64_t)((double)(k + 1) * f) > (int64_t)((double)k * f);
    }

    void dense(int h_idx, const double *a, int64_t lda, int64_t r0, int64_t r1,
               int64_t c0, int64_t c1, bool turning = false) {
        const bf_half &hf = P.halves[h_idx];
        for (auto rr : cuts(r0, r1))
            for (auto cc : cuts(c0, c1)) {
                int R = (int)(rr.second - rr.first), C = (int)(cc.second - cc.first);
                int flags = 0;
                int32_t aux = 0;
                int64_t t;
                if (turning && regen_cols_ok(C) && want_regen(R)) {
                    t = P.n_tiles;
                    P.n_tiles += bf_seed_doubles(R, C);
                    seeds.push_back({t, h_idx, (int)rr.first, R, cc.first, C});
                    flags = BF_OPF_REGEN;
                    P.n_regen++;
                    P.regen_values += (int64_t)R * C;
                    // the engine stages the tile's step coefficients from
                    // the rec table at issue time: their offset rides in aux
                    const int o = h_idx / 2;
                    const int64_t k_a = M.m[o] + (h_idx % 2 == 0 ? 1 : 0) + 2 * cc.first;
                    const int64_t rb = rec_base[o] + 2 * (k_a - M.m[o]);
                    if (rb > INT32_MAX) throw std::runtime_error("recurrence table exceeds int32 offsets");
                    aux = (int32_t)rb;
                } else {
                    t = alloc_tile(R, C, a + (rr.first - r0) * lda + (cc.first - c0), lda, 1);
                }
                int g = (int)(rr.first / BF_T), gc = (int)(cc.first / BF_T);
                fwd_groups[h_idx][g].push_back(mk(BF_OP_TILE_N, t, hf.x + (int32_t)cc.first, R, C,
                                                  (int)(rr.first - (int64_t)g * BF_T), flags, aux));
                inv_groups[h_idx][gc].push_back(mk(BF_OP_TILE_T, t, hf.y + (int32_t)rr.first, R, C,
                                                   (int)(cc.first - (int64_t)gc * BF_T), flags, aux));
            }
    }

    // Recurrence-coefficient tables and per-row seeds of the regenerated
    // tiles: the states (p_prev, p_cur, e) at each tile's first degree,
    // from the reference start values by the same no-FMA step the table
    // was built with, so the regenerated values are the stored ones.
    void build_rec() {
        const int64_t n2 = 2 * (int64_t)M.n;
        rec_base.assign(M.norders + 1, 0);
        for (int o = 0; o < M.norders; ++o) rec_base[o + 1] = rec_base[o] + 2 * (n2 - M.m[o]);
        P.rec.assign((size_t)rec_base[M.norders], 0.0);
        for (int o = 0; o < M.norders; ++o)
            for (int64_t s = 0; s < n2 - M.m[o]; ++s)
                bfr_coeffs(M.m[o], M.m[o] + s, &P.rec[rec_base[o] + 2 * s],
                           &P.rec[rec_base[o] + 2 * s + 1]);
        P.xpos.assign(M.x_pos, M.x_pos + M.n);
        P.mag_min = M.mag_min;
    }

    void fill_seeds(int threads) {
        if (seeds.empty()) return;
        if (!M.x_pos || !M.mant0 || !M.exp0) throw std::runtime_error("regen needs x_pos and start values");
        // per half and 32-row band: every seed job, by first degree
        std::map<std::pair<int, int>, std::vector<size_t>> bands;
        for (size_t i = 0; i < seeds.size(); ++i) bands[{seeds[i].h, seeds[i].r_a}].push_back(i);
        std::vector<std::pair<std::pair<int, int>, std::vector<size_t>>> work(bands.begin(), bands.end());
        double *T = P.tiles.get();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
        for (int64_t wi = 0; wi < (int64_t)work.size(); ++wi) {
            const int h = work[wi].first.first, r_a = work[wi].first.second;
            std::vector<size_t> js = work[wi].second;
            const int o = h / 2, par = h % 2;
            const int64_t m = M.m[o], offset = par == 0 ? 1 : 0;
            std::sort(js.begin(), js.end(), [&](size_t x, size_t y) { return seeds[x].c_a < seeds[y].c_a; });
            const double *rec = P.rec.data() + rec_base[o];
            int R = 0;
            for (size_t j : js) {
                const SeedJob &sj = seeds[j];
                R = std::max(R, sj.R);
                double *sb = T + sj.dst;
                std::memset(sb, 0, sizeof(double) * bf_seed_doubles(sj.R, sj.C));
                const int64_t k_a = m + offset + 2 * sj.c_a;
                int32_t hdr[2] = {sj.r_a, 0};
                std::memcpy(sb, hdr, sizeof(hdr));
                const int64_t rb = rec_base[o] + 2 * (k_a - m);
                std::memcpy(sb + 1, &rb, sizeof(rb));
            }
            for (int r = 0; r < R; ++r) {
                const int row = r_a + r;
                const double xr = M.x_pos[row];
                double pp = 0.0, pc = M.mant0[(int64_t)o * M.n + row];
                int e = M.exp0[(int64_t)o * M.n + row];
                int64_t k = m;
                for (size_t j : js) {
                    const SeedJob &sj = seeds[j];
                    // chain starts: column 0, and column 16 when split
                    for (int ch = 0; ch < bf_seed_chains(sj.C); ++ch) {
                        const int64_t k_a = m + offset + 2 * (sj.c_a + ch * BF_SEED_SPLIT);
                        for (; k < k_a; ++k)
                            bfr_step(xr, rec[2 * (k - m)], rec[2 * (k - m) + 1], &pp, &pc, &e);
                        if (r < sj.R) {
                            double *sr = T + sj.dst + 2 + 3 * (ch * sj.R + r);
                            sr[0] = pp;
                            sr[1] = pc;
                            sr[2] = (double)e;
                        }
                    }
                }
            }
        }
    }

    // -------------------------------------------------------- low-rank
    void lowrank(int h_idx, const bfsht_block &b) {
        const bf_half &hf = P.halves[h_idx];
        const int64_t h = b.r1 - b.r0, w = b.c1 - b.c0, r = b.rank;
        if (r <= 0) return;
        auto us = std::make_unique<std::vector<double>>((size_t)(h * r));
        for (int64_t i = 0; i < h; ++i)
            for (int64_t k = 0; k < r; ++k) (*us)[i * r + k] = b.a[i * r + k] * b.b[k];
        const double *u = us->data();
        keep.push_back(std::move(us));
        const double *v = b.c;
        int32_t tf = alloc_entries(r), ti = alloc_entries(r);
        for (int64_t k0 = 0; k0 < r; k0 += BF_T) {
            int K = (int)std::min<int64_t>(BF_T, r - k0);
            std::vector<bf_op> f1, i1;
            for (auto cc : cuts(b.c0, b.c1)) {  // v tiles: rows = block columns
                int R = (int)(cc.second - cc.first);
                int64_t t = alloc_tile(R, K, v + (cc.first - b.c0) * r + k0, r, 1);
                f1.push_back(mk(BF_OP_TILE_T, t, hf.x + (int32_t)cc.first, R, K, 0));
                int gc = (int)(cc.first / BF_T);
                inv_other[h_idx][gc].push_back(mk(BF_OP_TILE_N, t, ti + (int32_t)k0, R, K,
                                                   (int)(cc.first - (int64_t)gc * BF_T)));
            }
            for (auto rr : cuts(b.r0, b.r1)) {  // u s tiles: rows = block rows
                int R = (int)(rr.second - rr.first);
                int64_t t = alloc_tile(R, K, u + (rr.first - b.r0) * r + k0, r, 1);
                i1.push_back(mk(BF_OP_TILE_T, t, hf.y + (int32_t)rr.first, R, K, 0));
                int g = (int)(rr.first / BF_T);
                fwd_other[h_idx][g].push_back(mk(BF_OP_TILE_N, t, tf + (int32_t)k0, R, K,
                                                  (int)(rr.first - (int64_t)g * BF_T)));
            }
            add_task(0, 0, tf + (int32_t)k0, K, std::move(f1));
            add_task(1, 0, ti + (int32_t)k0, K, std::move(i1));
        }
        (void)h;
        (void)w;
    }

    // ---------------------------------------------------- butterfly
    // gather tasks applying G: in_vec indexes G columns, out_vec G rows
    void gather_tasks(const FactorSegs &fs, std::vector<std::vector<int64_t>> &tile_of,
                      int dir, int st, int32_t in_vec, int32_t out_vec) {
        for (size_t si = 0; si < fs.segs.size(); ++si) {
            const Segment &s = fs.segs[si];
            const auto &runs = tile_runs(fs, s);
            for (int64_t p0 = 0, p = 0; p0 < s.rows; p0 += BF_T, ++p) {
                int R = (int)std::min<int64_t>(BF_T, s.rows - p0);
                std::vector<bf_op> ops;
                for (size_t q = 0; q < runs.size(); ++q) {
                    int C = (int)(runs[q].second - runs[q].first);
                    std::vector<int32_t> ix(C);
                    for (int c = 0; c < C; ++c)
                        ix[c] = in_vec + (int32_t)s.dcols[runs[q].first + c];
                    ops.push_back(mk(BF_OP_TILE_N, tile_of[si][p * runs.size() + q], push_idx(ix),
                                     R, C, 0, BF_OPF_GATHER));
                }
                // identity (skeleton) entries; a row may carry more than one
                std::vector<std::vector<int32_t>> lanes;
                for (auto &u : s.units) {
                    int64_t lr = u.first - s.row0 - p0;
                    if (lr < 0 || lr >= R) continue;
                    size_t k = 0;
                    while (k < lanes.size() && lanes[k][lr] >= 0) ++k;
                    if (k == lanes.size()) lanes.emplace_back(BF_T, -1);
                    lanes[k][lr] = in_vec + (int32_t)u.second;
                }
                for (auto &ln : lanes) {
                    ln.resize(R);
                    ops.push_back(mk(BF_OP_ADD, 0, push_idx(ln), R, 0, 0, BF_OPF_GATHER));
                }
                add_task(dir, st, out_vec + (int32_t)(s.row0 + p0), R, std::move(ops));
            }
        }
    }

    // column runs of a segment's dense columns: cut at the BF_SLOTS-position
    // chunks of its range (one scatter task each) and at BF_T columns
    std::vector<std::pair<int64_t, int64_t>> tile_runs(const FactorSegs &fs, const Segment &s) {
        std::vector<std::pair<int64_t, int64_t>> runs;
        if (s.dcols.empty()) return runs;
        const int64_t a = fs.ranges[s.range].first;
        int64_t b = 0;
        for (int64_t j = 1; j <= (int64_t)s.dcols.size(); ++j) {
            if (j == (int64_t)s.dcols.size() || j - b == BF_T ||
                (s.dcols[j] - a) / BF_SLOTS != (s.dcols[b] - a) / BF_SLOTS) {
                runs.push_back({b, j});
                b = j;
            }
        }
        return runs;
    }

    // scatter tasks applying G^T: in_vec indexes G rows, out_vec G columns
    void scatter_tasks(const FactorSegs &fs, std::vector<std::vector<int64_t>> &tile_of,
                       int dir, int st, int32_t in_vec, int32_t out_vec) {
        std::vector<std::vector<size_t>> by_range(fs.ranges.size());
        for (size_t si = 0; si < fs.segs.size(); ++si)
            if (fs.segs[si].range >= 0) by_range[fs.segs[si].range].push_back(si);
        for (size_t ri = 0; ri < fs.ranges.size(); ++ri) {
            const int64_t a = fs.ranges[ri].first, e = fs.ranges[ri].second;
            for (int64_t q0 = a; q0 < e; q0 += BF_SLOTS) {
                const int64_t qid = (q0 - a) / BF_SLOTS;
                int nout = (int)std::min<int64_t>(BF_SLOTS, e - q0);
                std::vector<bf_op> ops;
                for (size_t si : by_range[ri]) {
                    const Segment &s = fs.segs[si];
                    const auto runs = tile_runs(fs, s);
                    for (size_t q = 0; q < runs.size(); ++q) {
                        if ((s.dcols[runs[q].first] - a) / BF_SLOTS != qid) continue;
                        int C = (int)(runs[q].second - runs[q].first);
                        int8_t lm[BF_SLOTS];
                        std::memset(lm, -1, sizeof(lm));
                        for (int c = 0; c < C; ++c)
                            lm[s.dcols[runs[q].first + c] - q0] = (int8_t)c;
                        int32_t mi = push_map(lm);
                        for (int64_t p0 = 0, p = 0; p0 < s.rows; p0 += BF_T, ++p) {
                            int R = (int)std::min<int64_t>(BF_T, s.rows - p0);
                            ops.push_back(mk(BF_OP_TILE_T, tile_of[si][p * runs.size() + q],
                                             in_vec + (int32_t)(s.row0 + p0), R, C, 0,
                                             BF_OPF_LANEMAP, mi));
                        }
                    }
                    // identity entries: index adds of <= 32 lanes each
                    for (int h0 = 0; h0 < nout; h0 += BF_T) {
                        const int hn = std::min(BF_T, nout - h0);
                        std::vector<int32_t> ln(hn, -1);
                        bool any = false;
                        for (auto &u : s.units) {
                            if (u.second < q0 + h0 || u.second >= q0 + h0 + hn) continue;
                            ln[u.second - q0 - h0] = in_vec + (int32_t)u.first;
                            any = true;
                        }
                        if (any)
                            ops.push_back(mk(BF_OP_ADD, 0, push_idx(ln), hn, 0, h0, BF_OPF_GATHER));
                    }
                }
                add_task(dir, st, out_vec + (int32_t)q0, nout, std::move(ops));
            }
        }
    }

    void butterfly(int h_idx, const bfsht_block &b, std::vector<FactorSegs> &segs) {
        const bf_half &hf = P.halves[h_idx];
        const int L = b.nfac;
        const int64_t h = b.r1 - b.r0, w = b.c1 - b.c0;
        const int nv = 1 + b.levels - b.middle;
        // forward vectors z[0..L], inverse vectors zi[0..L]
        std::vector<int32_t> z(L + 1), zi(L + 1);
        z[0] = hf.x + b.c0;
        for (int i = 1; i < L; ++i) z[i] = alloc_entries(b.fshape[2 * (i - 1)]);
        z[L] = alloc_entries(h);
        zi[0] = hf.y + b.r0;
        for (int j = 1; j < L; ++j) zi[j] = alloc_entries(b.fshape[2 * (L - j) + 1]);
        zi[L] = alloc_entries(w);
        for (int i = 0; i < L; ++i) {
            FactorSegs &fs = segs[i];
            bool g_is_f = i <= nv;
            // tiles of every segment: row groups x column runs
            std::vector<std::vector<int64_t>> tile_of(fs.segs.size());
            for (size_t si = 0; si < fs.segs.size(); ++si) {
                const Segment &s = fs.segs[si];
                auto runs = tile_runs(fs, s);
                const int64_t nd = (int64_t)s.dcols.size();
                for (int64_t p0 = 0; p0 < s.rows; p0 += BF_T)
                    for (auto &rn : runs) {
                        int R = (int)std::min<int64_t>(BF_T, s.rows - p0);
                        int C = (int)(rn.second - rn.first);
                        tile_of[si].push_back(alloc_tile(R, C, s.t.data() + p0 * nd + rn.first, nd, 1));
                    }
            }
            if (g_is_f) {
                gather_tasks(fs, tile_of, 0, i, z[i], z[i + 1]);
                scatter_tasks(fs, tile_of, 1, L - 1 - i, zi[L - 1 - i], zi[L - i]);
            } else {
                scatter_tasks(fs, tile_of, 0, i, z[i], z[i + 1]);
                gather_tasks(fs, tile_of, 1, L - 1 - i, zi[L - 1 - i], zi[L - i]);
            }
        }
        // block outputs into the group tasks
        for (auto rr : cuts(b.r0, b.r1)) {
            int g = (int)(rr.first / BF_T);
            fwd_other[h_idx][g].push_back(mk(BF_OP_ADD, 0, z[L] + (int32_t)(rr.first - b.r0),
                                              (int)(rr.second - rr.first), 0,
                                              (int)(rr.first - (int64_t)g * BF_T)));
        }
        for (auto cc : cuts(b.c0, b.c1)) {
            int gc = (int)(cc.first / BF_T);
            inv_other[h_idx][gc].push_back(mk(BF_OP_ADD, 0, zi[L] + (int32_t)(cc.first - b.c0),
                                               (int)(cc.second - cc.first), 0,
                                               (int)(cc.first - (int64_t)gc * BF_T)));
        }
    }

    void run(int threads) {
        const int n = M.n;
        // halves and their arena vectors
        P.halves.resize((size_t)M.norders * 2);
        fwd_groups.resize(P.halves.size());
        fwd_other.resize(P.halves.size());
        inv_other.resize(P.halves.size());
        inv_groups.resize(P.halves.size());
        for (int o = 0; o < M.norders; ++o)
            for (int par = 0; par < 2; ++par) {
                bf_half &hf = P.halves[o * 2 + par];
                hf.m = M.m[o];
                hf.ncols = M.ncols[o * 2 + par];
                if (hf.ncols > 0) {
                    hf.x = alloc_entries(hf.ncols);
                    hf.y = alloc_entries(n);
                    fwd_groups[o * 2 + par].resize((n + BF_T - 1) / BF_T);
                    fwd_other[o * 2 + par].resize((n + BF_T - 1) / BF_T);
                    inv_other[o * 2 + par].resize((hf.ncols + BF_T - 1) / BF_T);
                    inv_groups[o * 2 + par].resize((hf.ncols + BF_T - 1) / BF_T);
                } else {
                    hf.x = hf.y = -1;
                }
            }
        if (M.regen > 0.0) {
            if (!M.x_pos || !M.mant0 || !M.exp0 || !(M.mag_min > 0.0))
                throw std::runtime_error("regen needs x_pos, start values and mag_min");
            build_rec();
        }
        // butterfly segmentation in parallel (the heavy part)
        std::vector<std::vector<FactorSegs>> segs((size_t)M.nblocks);
        std::vector<std::string> errs((size_t)M.nblocks);
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
        for (int64_t bi = 0; bi < M.nblocks; ++bi) {
            const bfsht_block &b = M.blocks[bi];
            if (b.kind != 0 || b.nfac < 2) continue;
            try {
                const int nv = 1 + b.levels - b.middle;
                segs[bi].resize(b.nfac);
                for (int i = 0; i < b.nfac; ++i) {
                    bool g_is_f = i <= nv;
                    int64_t fr = b.fshape[2 * i], fc = b.fshape[2 * i + 1];
                    if (g_is_f)
                        segment_factor(fr, fc, b.fnnz[i], b.frows[i], b.fcols[i], b.fvals[i], segs[bi][i]);
                    else
                        segment_factor(fc, fr, b.fnnz[i], b.fcols[i], b.frows[i], b.fvals[i], segs[bi][i]);
                }
            } catch (std::exception &e) {
                errs[bi] = e.what();
            }
        }
        for (int64_t bi = 0; bi < M.nblocks; ++bi)
            if (!errs[bi].empty())
                throw std::runtime_error("block " + std::to_string(bi) + ": " + errs[bi]);

        for (int64_t bi = 0; bi < M.nblocks; ++bi) {
            const bfsht_block &b = M.blocks[bi];
            if (b.order < 0 || b.order >= M.norders || b.parity < 0 || b.parity > 1)
                throw std::runtime_error("block order/parity out of range");
            const int h_idx = b.order * 2 + b.parity;
            const bf_half &hf = P.halves[h_idx];
            if (hf.ncols <= 0) throw std::runtime_error("block in an absent half");
            if (b.r0 < 0 || b.r1 > n || b.r0 >= b.r1 || b.c0 < 0 || b.c1 > hf.ncols || b.c0 >= b.c1)
                throw std::runtime_error("block trim outside its half");
            const int64_t h = b.r1 - b.r0, w = b.c1 - b.c0;
            if (b.kind == 2) {
                P.n_dn++;
                P.payload_values += h * w;
                dense(h_idx, b.a, w, b.r0, b.r1, b.c0, b.c1, true);
            } else if (b.kind == 1) {
                P.n_lr++;
                P.payload_values += (h + w + 1) * (int64_t)b.rank;
                lowrank(h_idx, b);
            } else if (b.kind == 0) {
                P.n_bf++;
                int64_t vals = 0;
                for (int i = 0; i < b.nfac; ++i) vals += b.fnnz[i];
                P.payload_values += vals;
                if (b.nfac < 1) throw std::runtime_error("butterfly without factors");
                if (b.fshape[1] != w || b.fshape[2 * (b.nfac - 1)] != h)
                    throw std::runtime_error("butterfly shape does not match its trim");
                for (int i = 1; i < b.nfac; ++i)
                    if (b.fshape[2 * i + 1] != b.fshape[2 * (i - 1)])
                        throw std::runtime_error("butterfly factor chain shapes mismatch");
                if (b.nfac == 1) {
                    // depth 0: a single dense factor (butterfly.py:132-142)
                    auto d = std::make_unique<std::vector<double>>((size_t)(h * w), 0.0);
                    for (int64_t e = 0; e < b.fnnz[0]; ++e)
                        (*d)[b.frows[0][e] * w + b.fcols[0][e]] = b.fvals[0][e];
                    const double *src = d->data();
                    keep.push_back(std::move(d));
                    dense(h_idx, src, w, b.r0, b.r1, b.c0, b.c1);
                } else {
                    butterfly(h_idx, b, segs[bi]);
                }
            } else {
                throw std::runtime_error("unknown block kind");
            }
        }
        // group tasks: the last stage of each direction
        int last = 0;
        for (int d = 0; d < 2; ++d) last = std::max(last, (int)stages[d].size());
        // forward results go to the row-major node array Yr[r][order][parity]
        // (one contiguous 2 x norders run per node row), which the phi-DFT
        // stage reads row pair by row pair; tasks write it with a stride
        const int64_t yr_stride = 2 * (int64_t)M.norders;
        if (yr_stride >= (1 << 23)) throw std::runtime_error("too many orders for the Yr stride");
        P.yr = alloc_entries((int64_t)n * yr_stride);
        // Group tasks.  The dense tiles of a group depend on nothing computed
        // on the GPU, so they are dealt over the earlier stages (greedy by
        // stage cost) where their big tiles keep HBM busy under the small,
        // latency-bound butterfly and low-rank-core tasks; only the low-rank
        // (u s) t / v t tiles and butterfly block outputs wait for the final
        // stage, in a fix-up task that also adds the dense partial sums.  Long
        // op lists (e.g. the single column group of a half with a few
        // columns, which collects every block of a tall thin matrix) are
        // chunked so no task runs for long on one warp.  Summation order is
        // fixed by the packer, so results stay bitwise reproducible.
        struct Pending {
            int32_t out, nout;
            std::vector<bf_op> dense, other;
        };
        std::vector<Pending> groups[2];
        for (size_t hi = 0; hi < P.halves.size(); ++hi) {
            const bf_half &hf = P.halves[hi];
            if (hf.ncols <= 0) continue;
            for (size_t g = 0; g < fwd_groups[hi].size(); ++g)
                groups[0].push_back(
                    {P.yr + (int32_t)((int64_t)g * BF_T * yr_stride + (int64_t)hi),
                     (int32_t)std::min<int64_t>(BF_T, n - (int64_t)g * BF_T) |
                         (int32_t)(yr_stride << 8),
                     std::move(fwd_groups[hi][g]), std::move(fwd_other[hi][g])});
            for (size_t g = 0; g < inv_groups[hi].size(); ++g)
                groups[1].push_back(
                    {hf.x + (int32_t)(g * BF_T),
                     (int32_t)std::min<int64_t>(BF_T, hf.ncols - (int64_t)g * BF_T),
                     std::move(inv_groups[hi][g]), std::move(inv_other[hi][g])});
        }
        // Every group task runs in the final stage (measured on B200 at
        // N=1024: dealing the dependency-free dense tiles over the chain
        // stages, or running them on a side stream, cost more in extra
        // fix-up work than it hid); long op lists are chunked into partial
        // sums + a combine stage.  The summation order is fixed here, so
        // results are bitwise reproducible.
        {
            for (int d = 0; d < 2; ++d) {
                for (auto &gp : groups[d]) {
                    std::vector<bf_op> ops = std::move(gp.dense);
                    ops.insert(ops.end(), gp.other.begin(), gp.other.end());
                    if (ops.size() <= (size_t)kMaxTaskOps) {
                        add_task(d, last, gp.out, gp.nout, std::move(ops));
                        continue;
                    }
                    const int nout = gp.nout & 0xff;
                    std::vector<bf_op> comb;
                    for (size_t b = 0; b < ops.size(); b += kMaxTaskOps) {
                        const size_t e = std::min(ops.size(), b + kMaxTaskOps);
                        const int32_t part = alloc_entries(nout);
                        add_task(d, last, part, nout,
                                 std::vector<bf_op>(ops.begin() + b, ops.begin() + e));
                        for (int h0 = 0; h0 < nout; h0 += BF_T)
                            comb.push_back(
                                mk(BF_OP_ADD, 0, part + h0, std::min(BF_T, nout - h0), 0, h0));
                    }
                    add_task(d, last + 1, gp.out, gp.nout, std::move(comb));
                }
            }
            groups[0].clear();
            groups[1].clear();
        }
        // flatten: stages in order, tasks by descending cost
        for (int d = 0; d < 2; ++d) {
            P.stage_bounds[d].clear();
            P.stage_bounds[d].push_back((int64_t)P.tasks.size());
            for (auto &st : stages[d]) {
                std::stable_sort(st.begin(), st.end(),
                                 [](const TaskBuild &x, const TaskBuild &y) { return x.cost > y.cost; });
                for (auto &t : st) {
                    bf_task tk;
                    tk.op_begin = (int32_t)P.ops.size();
                    tk.op_count = (int32_t)t.ops.size();
                    tk.out = t.out;
                    tk.nout = t.nout;
                    P.ops.insert(P.ops.end(), t.ops.begin(), t.ops.end());
                    if ((int64_t)P.ops.size() > INT32_MAX) throw std::runtime_error("ops exceed int32");
                    P.tasks.push_back(tk);
                }
                P.stage_bounds[d].push_back((int64_t)P.tasks.size());
            }
        }
        // fill tiles
        const int64_t nj = (int64_t)jobs.size();
        P.tiles.reset(new double[(size_t)std::max<int64_t>(P.n_tiles, 2)]);
        double *T = P.tiles.get();
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads)
        for (int64_t j = 0; j < nj; ++j) {
            const TileJob &t = jobs[j];
            double *dst = T + t.dst;
            const int C4 = (t.C + 3) / 4, R4 = (t.R + 3) / 4;
            std::memset(dst, 0, sizeof(double) * bf_tile_doubles(t.R, t.C));
            for (int r = 0; r < t.R; ++r)
                for (int c = 0; c < t.C; ++c)
                    dst[bf_tile_index(r, c, C4)] = t.src[r * t.rs + c * t.cs];
            (void)R4;
        }
        fill_seeds(threads);
    }
};

}  // namespace

extern "C" int bfsht_pack_plan(const bfsht_manifest *man, int threads, bfsht_packed **out) {
    try {
        if (!man || !out) throw std::runtime_error("null argument");
        if (man->n < 1 || man->norders < 0 || man->nblocks < 0) throw std::runtime_error("bad manifest sizes");
        if (threads <= 0) threads = omp_get_num_procs();
        auto p = std::make_unique<bfsht_packed>();
        p->n = man->n;
        p->norders = man->norders;
        Packer pk(*p, *man);
        pk.run(threads);
        *out = p.release();
        return 0;
    } catch (std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

extern "C" int bfsht_packed_info(const bfsht_packed *p, int64_t info[BFSHT_INFO_LEN]) {
    if (!p) return -1;
    std::memset(info, 0, BFSHT_INFO_LEN * sizeof(int64_t));
    info[16] = info[17] = -1;   // reserved (no split free stage)
    info[0] = p->n_tiles;
    info[1] = (int64_t)p->ops.size();
    info[2] = (int64_t)p->idx.size();
    info[3] = (int64_t)p->maps.size() / BF_SLOTS;
    info[4] = (int64_t)p->tasks.size();
    info[5] = p->arena;
    info[6] = (int64_t)p->halves.size();
    info[7] = (int64_t)p->stage_bounds[0].size() - 1;
    info[8] = (int64_t)p->stage_bounds[1].size() - 1;
    info[9] = p->payload_values;
    info[10] = p->yr;
    info[11] = p->n_bf;
    info[12] = p->n_lr;
    info[13] = p->n_dn;
    info[14] = p->n;
    info[15] = p->norders;
    info[18] = p->n_regen;
    info[19] = p->regen_values;
    info[20] = (int64_t)p->rec.size();
    info[21] = (int64_t)p->xpos.size();
    std::memcpy(&info[22], &p->mag_min, sizeof(double));
    info[23] = 0;               // reserved (no dataflow order)
    return 0;
}

// arrays: 0 tiles, 1 ops, 2 idx, 3 maps, 4 tasks, 5 halves,
//         6 stage bounds fwd (int64, stages+1), 7 stage bounds inv,
//         8 recurrence coefficients, 9 x_pos, 10 / 11 reserved (NULL)
extern "C" int bfsht_packed_arrays(const bfsht_packed *p, const void *arrays[12]) {
    if (!p) return -1;
    arrays[0] = p->tiles.get();
    arrays[1] = p->ops.data();
    arrays[2] = p->idx.data();
    arrays[3] = p->maps.data();
    arrays[4] = p->tasks.data();
    arrays[5] = p->halves.data();
    arrays[6] = p->stage_bounds[0].data();
    arrays[7] = p->stage_bounds[1].data();
    arrays[8] = p->rec.data();
    arrays[9] = p->xpos.data();
    arrays[10] = nullptr;
    arrays[11] = nullptr;
    return 0;
}

// ---------------------------------------------------------- chain schedule
// Re-encodes the stages made of small tasks (butterfly gather / scatter
// tasks, low-rank cores) for the chain kernel (engine.cu alt_chain_kernel):
// one 32-byte bf_crec per op, an index add folded into the tile op it
// follows when that tile leaves the tail of its ring slot free, tasks
// grouped by LPT into cost-balanced bundles.  Op order inside a task is
// kept, so the chain kernel's sums are those of the stage kernel.
struct bfsht_chain_sched {
    std::vector<bf_crec> recs;
    std::vector<int32_t> bund;
    std::vector<int64_t> stage;   // per stage: first bundle entry, bundles, records, folded adds
};

extern "C" int bfsht_chain_schedule(const void *ops_v, const void *tasks_v, const int64_t *bounds,
                                    int nstages, int warps, int mode, int per_warp, int cfix,
                                    bfsht_chain_sched **out) {
    try {
        if (!ops_v || !tasks_v || !bounds || !out || nstages < 0 || warps < 1 || per_warp < 1 ||
            cfix < 0)
            throw std::runtime_error("bad chain schedule arguments");
        const bf_op *ops = (const bf_op *)ops_v;
        const bf_task *tasks = (const bf_task *)tasks_v;
        auto sc = std::make_unique<bfsht_chain_sched>();
        sc->stage.assign((size_t)nstages * 4, 0);
        struct Span {
            int64_t r0;
            int n;
            double cost;
        };
        std::vector<bf_crec> trec;
        std::vector<Span> spans;
        for (int s = 0; s < nstages && mode > 0; ++s) {
            const int64_t t0 = bounds[s], t1 = bounds[s + 1];
            if (t1 <= t0) continue;
            bool regen = false, small = false;
            for (int64_t t = t0; t < t1 && !regen; ++t)
                for (int i = 0; i < tasks[t].op_count; ++i) {
                    const uint8_t f = ops[tasks[t].op_begin + i].flags;
                    if (f & BF_OPF_REGEN) regen = true;
                    if (f & (BF_OPF_GATHER | BF_OPF_LANEMAP)) small = true;
                }
            if (regen || (mode == 1 && !small)) continue;
            trec.clear();
            spans.clear();
            int64_t nfold = 0;
            for (int64_t t = t0; t < t1; ++t) {
                const bf_task &tk = tasks[t];
                Span sp;
                sp.r0 = (int64_t)trec.size();
                sp.cost = 0.0;
                for (int i = 0; i < tk.op_count; ++i) {
                    const bf_op &o = ops[tk.op_begin + i];
                    if (o.kind != BF_OP_ADD && (o.tile % 16 != 0 || o.tile / 16 > (int64_t)UINT32_MAX))
                        throw std::runtime_error("tile offset not representable in a chain record");
                    if (o.kind == BF_OP_ADD && (o.flags & BF_OPF_GATHER) &&
                        (int64_t)trec.size() > sp.r0) {
                        bf_crec &pr = trec.back();
                        if (pr.kind != BF_OP_ADD && !(pr.flags & BF_CF_ADD) &&
                            bf_tile_doubles(pr.R, pr.C) <= BF_FOLD_AT && o.R <= BF_T) {
                            pr.flags |= BF_CF_ADD;
                            pr.addR = o.R;
                            pr.addoff = o.off;
                            pr.add_in = o.in;
                            sp.cost += 32.0 * o.R;
                            ++nfold;
                            continue;
                        }
                        // a second add right behind a folded one (the two
                        // 32-lane adds of a 64-slot scatter task) extends the
                        // fold when it continues it — next sources, next
                        // slots — and the tile leaves 2 KB of its slot free
                        if (pr.kind != BF_OP_ADD && (pr.flags & BF_CF_ADD) && pr.addR == BF_T &&
                            o.in == pr.add_in + pr.addR && (int)o.off == (int)pr.addoff + pr.addR &&
                            (int)pr.addR + o.R <= 2 * BF_T &&
                            bf_tile_doubles(pr.R, pr.C) <= BF_FOLD_AT - BF_T * BF_NRHS) {
                            pr.addR = (uint8_t)(pr.addR + o.R);
                            sp.cost += 32.0 * o.R;
                            ++nfold;
                            continue;
                        }
                    }
                    bf_crec c;
                    std::memset(&c, 0, sizeof(c));
                    c.tile = o.kind == BF_OP_ADD ? 0u : (uint32_t)(o.tile / 16);
                    c.in = o.in;
                    c.aux = o.aux;
                    c.kind = o.kind;
                    c.R = o.R;
                    c.C = o.C;
                    c.off = o.off;
                    c.flags = (uint8_t)(o.flags & (BF_OPF_GATHER | BF_OPF_LANEMAP));
                    trec.push_back(c);
                    sp.cost += (double)cfix +
                               (o.kind == BF_OP_ADD ? 32.0 * o.R
                                                    : 8.0 * (double)bf_tile_doubles(o.R, o.C) +
                                                          32.0 * (o.kind == BF_OP_TILE_N ? o.C : o.R));
                }
                if ((int64_t)trec.size() == sp.r0) throw std::runtime_error("task without ops");
                bf_crec &last = trec.back();
                last.flags |= BF_CF_LAST;
                last.out = tk.out;
                last.nout = tk.nout;
                sp.n = (int)((int64_t)trec.size() - sp.r0);
                spans.push_back(sp);
            }
            // LPT: tasks by descending cost onto the least-loaded bundle
            const int64_t ntasks = t1 - t0;
            const int nb = (int)std::min<int64_t>(ntasks, (int64_t)warps * per_warp);
            std::vector<int32_t> order((size_t)ntasks);
            for (int64_t i = 0; i < ntasks; ++i) order[i] = (int32_t)i;
            std::stable_sort(order.begin(), order.end(),
                             [&](int32_t x, int32_t y) { return spans[x].cost > spans[y].cost; });
            std::vector<std::vector<int32_t>> members((size_t)nb);
            typedef std::pair<double, int> Load;
            std::vector<Load> heap;
            for (int i = 0; i < nb; ++i) heap.push_back({0.0, i});
            auto cmp = [](const Load &x, const Load &y) { return x > y; };
            std::make_heap(heap.begin(), heap.end(), cmp);
            for (int32_t t : order) {
                std::pop_heap(heap.begin(), heap.end(), cmp);
                Load &top = heap.back();
                members[top.second].push_back(t);
                top.first += spans[t].cost;
                std::push_heap(heap.begin(), heap.end(), cmp);
            }
            sc->stage[4 * s] = (int64_t)sc->bund.size();
            sc->stage[4 * s + 1] = nb;
            sc->stage[4 * s + 2] = (int64_t)trec.size();
            sc->stage[4 * s + 3] = nfold;
            for (int i = 0; i < nb; ++i) {
                sc->bund.push_back((int32_t)sc->recs.size());
                for (int32_t t : members[i])
                    sc->recs.insert(sc->recs.end(), trec.begin() + spans[t].r0,
                                    trec.begin() + spans[t].r0 + spans[t].n);
                if ((int64_t)sc->recs.size() > INT32_MAX)
                    throw std::runtime_error("chain records exceed int32");
            }
            sc->bund.push_back((int32_t)sc->recs.size());
        }
        *out = sc.release();
        return 0;
    } catch (std::exception &e) {
        g_err = e.what();
        return -1;
    }
}

extern "C" int bfsht_chain_sched_arrays(const bfsht_chain_sched *sc, const void **recs,
                                        int64_t *nrecs, const int32_t **bund, int64_t *nbund,
                                        const int64_t **stage) {
    if (!sc) return -1;
    if (recs) *recs = sc->recs.data();
    if (nrecs) *nrecs = (int64_t)sc->recs.size();
    if (bund) *bund = sc->bund.data();
    if (nbund) *nbund = (int64_t)sc->bund.size();
    if (stage) *stage = sc->stage.data();
    return 0;
}

extern "C" void bfsht_chain_sched_free(bfsht_chain_sched *sc) { delete sc; }

extern "C" int bfsht_rec_coeffs(int64_t m, int64_t k_max, double *out) {
    if (!out || m < 0) return -1;
    for (int64_t k = m; k < k_max; ++k) bfr_coeffs(m, k, &out[2 * (k - m)], &out[2 * (k - m) + 1]);
    return 0;
}

// Host twin of the engine's tile generation (engine.cu regen_tile): each
// chain (columns [0, 16) and [16, C)) re-runs the reference step sequence
// (bfr_step, range test after every step) from its own seed.
extern "C" int bfsht_regen_tile_host(const double *seed, int R, int C, const double *rec,
                                     const double *x_pos, double mag_min, double *out) {
    if (!seed || !rec || !x_pos || !out || R < 1 || R > BF_T || C < 1 || C > BF_T) return -1;
    int32_t hdr[2];
    std::memcpy(hdr, seed, sizeof(hdr));
    int64_t rb;
    std::memcpy(&rb, seed + 1, sizeof(rb));
    const int C4 = (C + 3) / 4;
    const int K = bf_seed_chains(C);
    std::memset(out, 0, sizeof(double) * bf_tile_doubles(R, C));
    for (int r = 0; r < R; ++r) {
        const double xr = x_pos[hdr[0] + r];
        for (int ch = 0; ch < K; ++ch) {
            const int c0 = ch * BF_SEED_SPLIT, c1 = (ch + 1 < K) ? c0 + BF_SEED_SPLIT : C;
            double pp = seed[2 + 3 * (ch * R + r)], pc = seed[3 + 3 * (ch * R + r)];
            int e = (int)seed[4 + 3 * (ch * R + r)];
            for (int c = c0; c < c1; ++c) {
                double v = std::ldexp(pc, e);
                if (std::fabs(v) < mag_min) v = 0.0;
                out[bf_tile_index(r, c, C4)] = v;
                if (c + 1 < c1) {
                    bfr_step(xr, rec[rb + 4 * c], rec[rb + 4 * c + 1], &pp, &pc, &e);
                    bfr_step(xr, rec[rb + 4 * c + 2], rec[rb + 4 * c + 3], &pp, &pc, &e);
                }
            }
        }
    }
    return 0;
}

extern "C" void bfsht_packed_free(bfsht_packed *p) { delete p; }
