"""Factor types and the sampled decompositions that build them (plan time).

The payload layout is the reference's, so a plan built here is
interchangeable with one built by ``bfsht``:

* ``SparseFactor`` / ``ButterflyFactorization`` — triplet-form factor chain,
  factors[0] applied first (pkg/src/bfsht/butterfly.py:45-80);
* ``LowRankFactor`` — u diag(s) v^T (pkg/src/bfsht/lowrank.py:184-202);
* dense turning payloads are plain C-contiguous float64 arrays.

The decompositions (mock-Chebyshev sampling, column ID by pivoted QR with
rank doubling, randomized SVD, IDBF sweeps) restate the reference
algorithms (pkg/src/bfsht/lowrank.py:205-375, butterfly.py:83-272) with the
same LAPACK calls and the same seeded random streams, so the factors are
bitwise identical.  None of this runs on the GPU: the device consumes the
finished factors through pack.py.
"""
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import scipy.linalg


class RankOverflowError(Exception):
    """An interpolative decomposition hit its rank cap short of tolerance."""

    def __init__(self, msg, cap=None, tail_ratio=None):
        super().__init__(msg)
        self.cap = cap
        self.tail_ratio = tail_ratio


def derived_rng(seed, *key):
    """Generator for a (seed, key...) slot (pkg/src/bfsht/lowrank.py:38-40)."""
    return np.random.default_rng(np.random.SeedSequence(seed,
                                                        spawn_key=tuple(key)))


@dataclass
class SamplingConfig:
    """Sampling knobs (pkg/src/bfsht/lowrank.py:134-167); ``tolerance`` is
    the IDBF tolerance named by the benchmark configs."""

    mode: str = "mock_chebyshev"
    tolerance: float = 1e-10
    adaptive_rank: int = 150
    oversampling: int = 2
    rsvd_rank: int = 30
    rsvd_oversample: int = 2
    seed: int = 0

    def __post_init__(self):
        if self.mode not in ("mock_chebyshev", "random"):
            raise ValueError(f"unknown sampling mode {self.mode!r}")
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.adaptive_rank < 1:
            raise ValueError("adaptive_rank must be >= 1")
        if self.oversampling < 1:
            raise ValueError("oversampling must be >= 1")
        if self.rsvd_rank < 1:
            raise ValueError("rsvd_rank must be >= 1")
        if self.rsvd_oversample < 2:
            raise ValueError("rsvd_oversample must be >= 2 for stability")


@dataclass
class InterpDecomp:
    side: str
    skeleton: np.ndarray
    interp: np.ndarray
    rank: int
    tail_ratio: float = 0.0


@dataclass
class LowRankFactor:
    """A ~= u @ diag(s) @ v.T."""

    u: np.ndarray
    s: np.ndarray
    v: np.ndarray

    @property
    def rank(self):
        return self.s.size


@dataclass
class SparseFactor:
    """One butterfly factor in triplet form."""

    shape: tuple
    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self):
        return self.vals.size


@dataclass
class ButterflyFactorization:
    """Factor chain; factors[0] is applied first (the leaf V stage)."""

    shape: tuple
    factors: list
    levels: int
    middle: int
    max_rank: int
    tolerance: float
    adaptive_rank: int

    @property
    def nnz(self):
        return int(sum(f.nnz for f in self.factors))


# ---------------------------------------------------------------- oracles
class TableOracle:
    """Entry access into a precomputed table through row/col index maps.

    Plays the role of the reference's EntryOracle views (lowrank.py:43-131)
    for matrices the planner has already materialized.
    """

    def __init__(self, table, rows=None, cols=None, transposed=False):
        self.table = table
        self.rows = np.arange(table.shape[0], dtype=np.intp) if rows is None \
            else np.asarray(rows, dtype=np.intp)
        self.cols = np.arange(table.shape[1], dtype=np.intp) if cols is None \
            else np.asarray(cols, dtype=np.intp)
        self.transposed = transposed

    @property
    def shape(self):
        return (self.cols.size, self.rows.size) if self.transposed \
            else (self.rows.size, self.cols.size)

    def _gather(self, rows, cols):
        # Same memory layout as the reference oracle's gather
        # (partition.py:140-169): ascending column requests come back
        # C-ordered, others through a unique/inverse column reindex.  The
        # layout matters because BLAS products round differently on
        # C- and F-ordered operands.
        if cols.size == 1 or np.all(cols[1:] > cols[:-1]):
            return self.table[np.ix_(rows, cols)]
        uniq, inv = np.unique(cols, return_inverse=True)
        return self.table[np.ix_(rows, uniq)][:, inv]

    def block(self, rows, cols):
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        if rows.size == 0 or cols.size == 0:
            return np.zeros((rows.size, cols.size))
        if self.transposed:
            return np.ascontiguousarray(
                self._gather(self.rows[cols], self.cols[rows]).T)
        return self._gather(self.rows[rows], self.cols[cols])

    def submatrix(self, rows, cols):
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        if self.transposed:
            return TableOracle(self.table, self.rows[cols], self.cols[rows],
                               transposed=True)
        return TableOracle(self.table, self.rows[rows], self.cols[cols])

    def transpose(self):
        return TableOracle(self.table, self.rows, self.cols,
                           transposed=not self.transposed)


class FunctionOracle:
    """Oracle over a broadcasting entry function fn(i, j) (test kernels)."""

    def __init__(self, fn, shape):
        self.fn = fn
        self._shape = tuple(shape)

    @property
    def shape(self):
        return self._shape

    def block(self, rows, cols):
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        return np.asarray(self.fn(rows[:, None], cols[None, :]),
                          dtype=np.float64)

    def submatrix(self, rows, cols):
        r = np.asarray(rows, dtype=np.intp)
        c = np.asarray(cols, dtype=np.intp)
        fn = self.fn
        return FunctionOracle(lambda i, j: fn(r[i], c[j]), (r.size, c.size))

    def transpose(self):
        fn = self.fn
        return FunctionOracle(lambda i, j: fn(j, i), self._shape[::-1])


# --------------------------------------------------------- sampled IDs
def sample_indices(count, total, mode="mock_chebyshev", rng=None):
    """min(count, total) distinct sorted indices (lowrank.py:205-249)."""
    if count <= 0 or total <= 0:
        raise ValueError("count and total must be positive")
    count = min(count, total)
    if count == total:
        return np.arange(total, dtype=np.intp)
    if mode == "random":
        if rng is None:
            raise ValueError("random mode needs an rng")
        return np.sort(rng.choice(total, size=count,
                                  replace=False)).astype(np.intp)
    if mode != "mock_chebyshev":
        raise ValueError(f"unknown sampling mode {mode!r}")
    return _mock_chebyshev(count, total)


@lru_cache(maxsize=8192)
def _mock_chebyshev(count, total):
    # deterministic in (count, total): the planner asks for the same few
    # shapes thousands of times, so the result is built once (read-only)
    out = _mock_chebyshev_build(count, total)
    out.setflags(write=False)
    return out


def _mock_chebyshev_build(count, total):
    t = np.cos(np.pi * (2.0 * np.arange(count, dtype=np.float64) + 1.0)
               / (2.0 * count))
    raw = np.rint((t + 1.0) * 0.5 * (total - 1)).astype(np.intp)
    if np.unique(raw).size == raw.size:
        return np.sort(raw)
    taken = np.zeros(total, dtype=bool)
    out = []
    for idx in raw.tolist():
        pick = idx
        if taken[idx]:
            # nearest free index, upper neighbour first at equal distance
            for delta in range(1, total):
                if idx + delta < total and not taken[idx + delta]:
                    pick = idx + delta
                    break
                if idx - delta >= 0 and not taken[idx - delta]:
                    pick = idx - delta
                    break
        taken[pick] = True
        out.append(pick)
    return np.sort(np.asarray(out, dtype=np.intp))


def _pivoted_r(a):
    r, perm = scipy.linalg.qr(a, mode="r", pivoting=True)
    return r, perm


def _rank_from_diag(dmag, eps):
    if dmag.size == 0 or dmag[0] == 0.0:
        return 0, 0.0
    ratios = dmag / dmag[0]
    hit = np.nonzero(ratios <= eps)[0]
    if hit.size:
        return int(hit[0]), float(ratios[hit[0]])
    return dmag.size, float(ratios[-1])


def _col_interp(r, perm, k, n, tail):
    if k == 0:
        return InterpDecomp("col", np.zeros(0, dtype=np.intp),
                            np.zeros((0, n)), 0, tail)
    lead = r[:k, :k]
    d = np.abs(np.diag(lead))
    floor = 1e-15 * d[0]
    if d.min() < floor:
        lead = lead.copy()
        ii = np.arange(k)
        sign = np.where(np.diag(lead) < 0, -1.0, 1.0)
        lead[ii, ii] = sign * np.maximum(d, floor)
    interp = np.zeros((k, n))
    interp[:, perm[:k]] = np.eye(k)
    if k < n:
        interp[:, perm[k:]] = scipy.linalg.solve_triangular(lead, r[:k, k:])
    return InterpDecomp("col", perm[:k].astype(np.intp), interp, k, tail)


def cid(oracle, cfg, rng=None):
    """Column ID from t*r_k sampled rows with rank doubling
    (lowrank.py:275-304)."""
    m, n = oracle.shape
    if m == 0 or n == 0:
        raise ValueError("cid needs a nonempty oracle")
    rk = cfg.adaptive_rank
    last = np.inf
    all_cols = np.arange(n, dtype=np.intp)
    for _ in range(5):
        cap = cfg.oversampling * rk
        rows = sample_indices(min(cap, m), m, cfg.mode, rng)
        r, perm = _pivoted_r(oracle.block(rows, all_cols))
        dmag = np.abs(np.diag(r))
        k, tail = _rank_from_diag(dmag, cfg.tolerance)
        if k < dmag.size or k >= n or rows.size >= m:
            return _col_interp(r, perm, k, n, tail)
        last = float(dmag[-1] / dmag[0])
        rk *= 2
    cap = cfg.oversampling * cfg.adaptive_rank * 16
    raise RankOverflowError(
        f"column ID did not reach tolerance {cfg.tolerance:g} at cap "
        f"{cap} (last ratio {last:.3e})", cap=cap, tail_ratio=last)


def _pinv(a, rcond):
    """np.linalg.pinv (LAPACK gesdd), as the reference calls it
    (lowrank.py:370-372).  gesdd can fail to converge on strongly graded
    blocks — the reference planner itself raises LinAlgError at N=4096,
    tol 1e-10, m=5561 (checked by running it) — and only then is the same
    pseudo-inverse formed from the QR-iteration driver gesvd: singular
    values above rcond * max(s) inverted, the rest dropped (numpy's pinv
    rule).  Factors of every order the reference can plan are unchanged."""
    try:
        return np.linalg.pinv(a, rcond=rcond)
    except np.linalg.LinAlgError:
        u, s, vt = scipy.linalg.svd(a, full_matrices=False, lapack_driver="gesvd")
        keep = s > rcond * (s.max() if s.size else 0.0)
        inv = np.zeros_like(s)
        inv[keep] = 1.0 / s[keep]
        return (vt.T * inv) @ u.T


def _svd(a):
    """np.linalg.svd (gesdd) with the same gesvd fallback as _pinv."""
    try:
        return np.linalg.svd(a)
    except np.linalg.LinAlgError:
        return scipy.linalg.svd(a, lapack_driver="gesvd")


def rsvd(oracle, row_samples, col_samples, rank, oversample=2, rng=None):
    """Sampled rank-r SVD (Algorithm 1, lowrank.py:335-375)."""
    if rng is None:
        rng = np.random.default_rng()
    m, n = oracle.shape
    r = int(min(rank, m, n))
    if r < 1:
        raise ValueError("rsvd needs rank >= 1 and a nonempty oracle")
    row_samples = np.asarray(row_samples, dtype=np.intp)
    col_samples = np.asarray(col_samples, dtype=np.intp)
    if row_samples.size < r or col_samples.size < r:
        raise ValueError("need at least `rank` sampled rows and columns")
    all_rows = np.arange(m, dtype=np.intp)
    all_cols = np.arange(n, dtype=np.intp)
    _, perm = _pivoted_r(oracle.block(row_samples, all_cols))
    pick_c = perm[:r]
    _, perm = _pivoted_r(oracle.block(all_rows, col_samples).T)
    pick_r = perm[:r]
    qc = scipy.linalg.qr(oracle.block(all_rows, pick_c), mode="economic",
                         pivoting=True)[0][:, :r]
    qr_ = scipy.linalg.qr(oracle.block(pick_r, all_cols).T, mode="economic",
                          pivoting=True)[0][:, :r]
    rows_aug = np.concatenate([pick_r, rng.choice(
        m, size=min(row_samples.size, m), replace=False)])
    cols_aug = np.concatenate([pick_c, rng.choice(
        n, size=min(col_samples.size, n), replace=False)])
    core = _pinv(qc[rows_aug, :], 1e-13) \
        @ oracle.block(rows_aug, cols_aug) \
        @ _pinv(qr_[cols_aug, :].T, 1e-13)
    u_m, s, vt_m = _svd(core)
    return LowRankFactor(u=qc @ u_m[:, :r], s=s[:r], v=qr_ @ vt_m[:r, :].T)


# ------------------------------------------------------------ butterfly
def _bisect(start, stop, depth):
    levels = [[(start, stop)]]
    for _ in range(depth):
        nxt = []
        for a, b in levels[-1]:
            mid = (a + b) // 2
            nxt += [(a, mid), (mid, b)]
        levels.append(nxt)
    return levels


def tree_levels(rows, cols, leaf_max):
    """Row/col dyadic interval levels of the shared depth
    (butterfly.py:83-116): depth = ceil(log2(min_dim/leaf_max)) capped at
    floor(log2(min_dim))."""
    r0, r1 = (0, rows) if np.isscalar(rows) else rows
    c0, c1 = (0, cols) if np.isscalar(cols) else cols
    if r1 <= r0 or c1 <= c0:
        raise ValueError("trees need nonempty index ranges")
    if leaf_max < 1:
        raise ValueError("leaf_max must be >= 1")
    small = min(r1 - r0, c1 - c0)
    depth = max(0, int(np.ceil(np.log2(small / leaf_max)))) \
        if small > leaf_max else 0
    depth = min(depth, int(np.floor(np.log2(small))))
    return depth, _bisect(r0, r1, depth), _bisect(c0, c1, depth)


def _triplets_to_factor(shape, parts):
    if parts:
        rows = np.concatenate([p[0] for p in parts]).astype(np.intp)
        cols = np.concatenate([p[1] for p in parts]).astype(np.intp)
        vals = np.concatenate([p[2] for p in parts]).astype(np.float64)
    else:
        rows = np.zeros(0, dtype=np.intp)
        cols = np.zeros(0, dtype=np.intp)
        vals = np.zeros(0)
    return SparseFactor(shape, rows, cols, vals)


def _node_id(view, cfg, sweep, level, i, j):
    try:
        return cid(view, cfg, rng=derived_rng(cfg.seed, sweep, level, i, j))
    except RankOverflowError as exc:
        raise RankOverflowError(
            f"butterfly ID overflow at level {level}, node pair ({i}, {j}): "
            f"{exc}", cap=exc.cap, tail_ratio=exc.tail_ratio) from exc


def _sweep(oracle, row_lv, col_lv, depth, stop, cfg, sweep):
    """Leaf-to-``stop`` column-ID sweep (butterfly.py:164-223).  Returns the
    factors leaf first, the skeleton/offset tables of the last level and the
    largest rank."""
    m, n = oracle.shape
    every_row = np.arange(m, dtype=np.intp)
    skel, offs, parts, pos, top = {}, {}, [], 0, 0
    for j, (c0, c1) in enumerate(col_lv[depth]):
        dec = _node_id(oracle.submatrix(every_row,
                                        np.arange(c0, c1, dtype=np.intp)),
                       cfg, sweep, depth, 0, j)
        skel[(0, j)] = (c0 + dec.skeleton).astype(np.intp)
        offs[(0, j)] = (pos, dec.rank)
        rr, cc = np.nonzero(dec.interp)
        parts.append((pos + rr, c0 + cc, dec.interp[rr, cc]))
        pos += dec.rank
        top = max(top, dec.rank)
    factors = [_triplets_to_factor((pos, n), parts)]
    for lev in range(depth - 1, stop - 1, -1):
        lam = depth - lev
        nskel, noffs, parts, npos = {}, {}, [], 0
        for i, (r0, r1) in enumerate(row_lv[lam]):
            p = i // 2
            for j in range(len(col_lv[lev])):
                a, b = (p, 2 * j), (p, 2 * j + 1)
                cand = np.concatenate([skel[a], skel[b]])
                src = np.concatenate([
                    offs[a][0] + np.arange(offs[a][1], dtype=np.intp),
                    offs[b][0] + np.arange(offs[b][1], dtype=np.intp)])
                if cand.size == 0:
                    nskel[(i, j)] = cand
                    noffs[(i, j)] = (npos, 0)
                    continue
                dec = _node_id(oracle.submatrix(
                    np.arange(r0, r1, dtype=np.intp), cand),
                    cfg, sweep, lev, i, j)
                nskel[(i, j)] = cand[dec.skeleton]
                noffs[(i, j)] = (npos, dec.rank)
                rr, cc = np.nonzero(dec.interp)
                parts.append((npos + rr, src[cc], dec.interp[rr, cc]))
                npos += dec.rank
                top = max(top, dec.rank)
        factors.append(_triplets_to_factor((npos, pos), parts))
        skel, offs, pos = nskel, noffs, npos
    return factors, skel, offs, top


def idbf_factor(oracle, cfg, leaf_max=None):
    """IDBF of an entry oracle: K ~= U^L..U^h S^h V^h..V^L
    (butterfly.py:119-161)."""
    m, n = oracle.shape
    if leaf_max is None:
        leaf_max = cfg.adaptive_rank
    depth, row_lv, col_lv = tree_levels(m, n, leaf_max)
    if depth == 0:
        dense = np.asarray(oracle.block(np.arange(m, dtype=np.intp),
                                        np.arange(n, dtype=np.intp)))
        rr, cc = np.nonzero(dense)
        f = SparseFactor((m, n), rr.astype(np.intp), cc.astype(np.intp),
                         dense[rr, cc].astype(np.float64))
        return ButterflyFactorization((m, n), [f], 0, 0, 0, cfg.tolerance,
                                      cfg.adaptive_rank)
    h_col = (depth + 1) // 2
    h_row = depth - h_col
    v_fac, col_skel, col_offs, rank_v = _sweep(oracle, row_lv, col_lv, depth,
                                               h_col, cfg, 0)
    u_fac, row_skel, row_offs, rank_u = _sweep(oracle.transpose(), col_lv,
                                               row_lv, depth, h_row, cfg, 1)
    # middle skeleton block (butterfly.py:226-242)
    n_out = sum(sz for _, sz in row_offs.values())
    n_in = sum(sz for _, sz in col_offs.values())
    parts = []
    for i in range(len(row_lv[h_row])):
        for j in range(len(col_lv[h_col])):
            ra, ca = row_skel[(j, i)], col_skel[(i, j)]
            if ra.size == 0 or ca.size == 0:
                continue
            blk = np.asarray(oracle.block(ra, ca))
            rr, cc = np.nonzero(blk)
            parts.append((row_offs[(j, i)][0] + rr, col_offs[(i, j)][0] + cc,
                          blk[rr, cc]))
    factors = list(v_fac)
    factors.append(_triplets_to_factor((n_out, n_in), parts))
    for f in reversed(u_fac):
        factors.append(SparseFactor((f.shape[1], f.shape[0]), f.cols.copy(),
                                    f.rows.copy(), f.vals.copy()))
    return ButterflyFactorization((m, n), factors, depth, h_col,
                                  max(rank_v, rank_u), cfg.tolerance,
                                  cfg.adaptive_rank)
