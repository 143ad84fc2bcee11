"""Factor-construction entry point: ``plan_alt`` / ``plan_sht``.

Same signatures, layout and results as the reference planner
(pkg/src/bfsht/alt.py:85-194, pkg/src/bfsht/sht.py:109-128,
pkg/src/bfsht/partition.py:38-333): every order m gets an ``AltPlan`` whose
odd/even half matrices are split along the turning-point curve, trimmed,
and compressed (oscillatory -> IDBF chain, non-oscillatory -> sampled
rank-30 SVD, turning -> dense trimmed block).

Differences are in how, not what: the half matrix of one (m, parity) is
tabulated once by the native recurrence (csrc/recur.c) instead of through
checkpointed per-block gathers, and ``plan_sht`` can fan orders out over
host processes.  The resulting factors are bitwise identical to the
reference's (tests/test_planner.py pins digests of reference plans), so
the GPU consumes exactly the factors the reference CPU planner builds.
This module is plan time only; nothing here runs in the apply path.
"""
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, replace

import numpy as np
from threadpoolctl import threadpool_limits

from .factors import (ButterflyFactorization, LowRankFactor,
                      RankOverflowError, SamplingConfig, TableOracle,
                      derived_rng, idbf_factor, rsvd, sample_indices)
from .legendre import QuadratureRule, gauss_legendre, half_table

N0_DEFAULT = 512          # pkg/src/bfsht/alt.py:38
TAU_DEFAULT = 1e-290      # pkg/src/bfsht/partition.py:35


@dataclass
class AltMatrixSpec:
    """One parity half of the order-m matrix (partition.py:38-65): n rows
    (positive nodes, ascending x), column j = degree m + offset + 2j."""

    n: int
    m: int
    parity: str
    num_cols: int
    quadrature: QuadratureRule

    @property
    def offset(self):
        return 1 if self.parity == "odd" else 0

    @property
    def x_pos(self):
        return self.quadrature.nodes[self.n:]

    @property
    def thetas(self):
        return np.arccos(self.x_pos)

    def col_degrees(self, cols):
        return self.m + self.offset + 2 * np.asarray(cols, dtype=np.int64)


def make_alt_spec(n, m, parity, quadrature=None):
    if parity not in ("odd", "even"):
        raise ValueError(f"parity must be 'odd' or 'even', got {parity!r}")
    if not 0 <= m <= 2 * n - 1:
        raise ValueError(f"order {m} outside [0, {2 * n - 1}]")
    half = (m + 1) // 2 if parity == "odd" else m // 2
    num_cols = n - half
    if num_cols < 1:
        raise ValueError(f"order {m} leaves no {parity} degrees at "
                         f"half-size {n}")
    if quadrature is None:
        quadrature = gauss_legendre(2 * n)
    elif quadrature.order != 2 * n:
        raise ValueError(f"quadrature order {quadrature.order} != {2 * n}")
    return AltMatrixSpec(n=n, m=m, parity=parity, num_cols=num_cols,
                         quadrature=quadrature)


@dataclass
class Block:
    """A partition leaf (partition.py:189-204); trim = (r0, r1, c0, c1) of
    the retained rectangle, payload = its compressed form."""

    row_range: tuple
    col_range: tuple
    kind: str
    level: int
    band: int
    trim: tuple = None
    payload: object = None

    @property
    def shape(self):
        return (self.row_range[1] - self.row_range[0],
                self.col_range[1] - self.col_range[0])


@dataclass
class AltPlan:
    n: int
    m: int
    spec_odd: object
    spec_even: object
    blocks_odd: list
    blocks_even: list
    params: SamplingConfig
    n0: int
    tau: float
    stats: dict

    @property
    def quadrature(self):
        spec = self.spec_even if self.spec_even is not None else self.spec_odd
        return spec.quadrature


def _turning_column(spec, rows):
    # fractional column where each row meets the turning curve
    # (partition.py:176-186)
    theta = np.arccos(spec.x_pos[rows])
    k_star = np.sqrt(spec.m**2 - 0.25) / np.sin(theta) - 0.5
    return (k_star - spec.m - spec.offset) / 2.0


def partition(spec, n0):
    """Band split + recursive quartering along the curve
    (partition.py:215-258); returns (blocks, levels_used)."""
    if n0 < 2:
        raise ValueError("n0 must be >= 2")
    n, nc = spec.n, spec.num_cols
    if spec.m == 0:
        return [Block((0, n), (0, nc), "oscillatory", 0, 0)], 0
    jstar = _turning_column(spec, np.arange(n))
    bands = int(np.floor(n / nc + 0.5))
    edges = [(i * n) // bands for i in range(bands + 1)]
    out, deepest = [], 0
    for band in range(bands):
        todo = [(edges[band], edges[band + 1], 0, nc, 0)]
        while todo:
            r0, r1, c0, c1, lev = todo.pop()
            deepest = max(deepest, lev)
            if c0 >= jstar[r1 - 1]:
                out.append(Block((r0, r1), (c0, c1), "oscillatory", lev, band))
            elif c1 <= jstar[r0]:
                out.append(Block((r0, r1), (c0, c1), "non_oscillatory", lev,
                                 band))
            elif r1 - r0 < n0 or c1 - c0 < n0:
                out.append(Block((r0, r1), (c0, c1), "turning", lev, band))
            else:
                rm, cm = (r0 + r1) // 2, (c0 + c1) // 2
                todo += [(r0, rm, c0, cm, lev + 1), (r0, rm, cm, c1, lev + 1),
                         (rm, r1, c0, cm, lev + 1), (rm, r1, cm, c1, lev + 1)]
    return out, deepest


def _alive_run(mags, tau):
    dead = np.nonzero(~(mags > tau))[0]
    return mags.size if dead.size == 0 else int(dead[0])


def _alive_prefix(table, r0, r1, col, tau):
    """Leading run of |entries| > tau down one column, located with the
    reference's probe ladder (partition.py:266-302) so the trim is the
    same even where decay is not monotone."""
    n = r1 - r0
    if n <= 256:
        return _alive_run(np.abs(table[r0:r1, col]), tau)
    ladder = [0]
    while ladder[-1] < n - 1:
        ladder.append(min(2 * ladder[-1] + 1, n - 1))
    ladder = np.asarray(ladder, dtype=np.intp)
    dead = ~(np.abs(table[r0 + ladder, col]) > tau)
    if dead[0]:
        return 0
    if not dead.any():
        return n
    j = int(np.argmax(dead))
    lo, hi = int(ladder[j - 1]), int(ladder[j])
    while hi - lo > 256:
        grid = np.unique(np.linspace(lo, hi, 18).astype(np.intp)[1:-1])
        gdead = ~(np.abs(table[r0 + grid, col]) > tau)
        if not gdead.any():
            lo = int(grid[-1])
        elif gdead[0]:
            hi = int(grid[0])
        else:
            k = int(np.argmax(gdead))
            lo, hi = int(grid[k - 1]), int(grid[k])
    span = np.arange(lo + 1, hi + 1, dtype=np.intp)
    return lo + 1 + _alive_run(np.abs(table[r0 + span, col]), tau)


def trim_block(table, block, tau=TAU_DEFAULT):
    """Corner rectangle holding every above-tau entry (partition.py:305-333);
    oscillatory blocks stay whole, all-dead blocks get trim None."""
    (r0, r1), (c0, c1) = block.row_range, block.col_range
    if block.kind == "oscillatory":
        return replace(block, trim=(r0, r1, c0, c1))
    h = _alive_prefix(table, r0, r1, c1 - 1, tau)
    if h == 0:
        return replace(block, trim=None)
    w = _alive_run(np.abs(table[r0, c0:c1])[::-1], tau)
    return replace(block, trim=(r0, r0 + h, c1 - w, c1))


def _compress(spec, table, blk, params):
    """Payload for one retained block (alt.py:155-194)."""
    r0, r1, c0, c1 = blk.trim
    h, w = r1 - r0, c1 - c0
    t0 = time.perf_counter()
    if blk.kind == "oscillatory":
        view = TableOracle(table, np.arange(r0, r1, dtype=np.intp),
                           np.arange(c0, c1, dtype=np.intp))
        try:
            payload = idbf_factor(view, params)
        except RankOverflowError as exc:
            raise RankOverflowError(
                f"{spec.parity} block rows {blk.row_range} cols "
                f"{blk.col_range}: {exc}", cap=exc.cap,
                tail_ratio=exc.tail_ratio) from exc
        rank, nnz = payload.max_rank, payload.nnz
    elif blk.kind == "non_oscillatory":
        view = TableOracle(table, np.arange(r0, r1, dtype=np.intp),
                           np.arange(c0, c1, dtype=np.intp))
        r = int(min(params.rsvd_rank, h, w))
        rng = derived_rng(params.seed, 2, blk.row_range[0], blk.col_range[0])
        rows = sample_indices(min(r * params.rsvd_oversample, h), h,
                              params.mode, rng)
        cols = sample_indices(min(r * params.rsvd_oversample, w), w,
                              params.mode, rng)
        payload = rsvd(view, rows, cols, r, oversample=params.rsvd_oversample,
                       rng=rng)
        rank = payload.rank
        nnz = payload.u.size + payload.s.size + payload.v.size
    else:
        payload = np.ascontiguousarray(table[r0:r1, c0:c1])
        rank, nnz = 0, payload.size
    blk.payload = payload
    return blk, {"parity": spec.parity, "class": blk.kind,
                 "rows": list(blk.row_range), "cols": list(blk.col_range),
                 "trim": list(blk.trim), "rank": rank, "nnz": int(nnz),
                 "seconds": time.perf_counter() - t0}


def _empty_stats():
    return {"per_block": [], "t_factor": 0.0,
            "t_by_class": {"oscillatory": 0.0, "non_oscillatory": 0.0,
                           "turning": 0.0},
            "block_counts": {"oscillatory": 0, "non_oscillatory": 0,
                             "turning": 0, "dropped": 0},
            "halves": {}, "max_rank": 0, "total_nnz": 0, "levels_used": 0}


def plan_alt(n, m, params=None, n0=N0_DEFAULT, tau=TAU_DEFAULT,
             quadrature=None, workers=1, device=None):
    """Compressed two-parity plan for order m at half-size n
    (alt.py:85-152).

    BLAS/LAPACK run single-threaded inside: a threaded reduction could
    change the last bits of a QR and with them the factors.  ``device``
    (CUDA ordinal) tabulates the entries on that GPU (same bits)."""
    with threadpool_limits(limits=1):
        return _plan_alt(n, m, params, n0, tau, quadrature, workers, device)


def _plan_alt(n, m, params, n0, tau, quadrature, workers, device=None):
    if not 0 <= m <= 2 * n - 1:
        raise ValueError(f"order {m} outside [0, {2 * n - 1}]")
    if params is None:
        params = SamplingConfig()
    if quadrature is None:
        quadrature = gauss_legendre(2 * n)
    stats = _empty_stats()
    halves = {}
    for parity in ("odd", "even"):
        half = (m + 1) // 2 if parity == "odd" else m // 2
        if n - half < 1:
            halves[parity] = (None, [])
            continue
        t0 = time.perf_counter()
        spec = make_alt_spec(n, m, parity, quadrature)
        table = half_table(m, spec.offset, spec.x_pos, spec.num_cols, device)
        leaves, deepest = partition(spec, n0)
        stats["levels_used"] = max(stats["levels_used"], deepest)
        kept, dropped = [], 0
        for blk in leaves:
            blk = trim_block(table, blk, tau)
            if blk.trim is None:
                dropped += 1
            else:
                kept.append(blk)
        if workers > 1 and len(kept) > 1:
            with ThreadPoolExecutor(max_workers=workers) as pool:
                done = list(pool.map(
                    lambda b: _compress(spec, table, b, params), kept))
        else:
            done = [_compress(spec, table, b, params) for b in kept]
        hstat = {"t_build": 0.0, "max_rank": 0, "total_nnz": 0,
                 "counts": {"oscillatory": 0, "non_oscillatory": 0,
                            "turning": 0, "dropped": dropped},
                 "partition_blocks": len(leaves)}
        blocks = []
        for blk, entry in done:
            blocks.append(blk)
            stats["per_block"].append(entry)
            stats["t_factor"] += entry["seconds"]
            stats["t_by_class"][blk.kind] += entry["seconds"]
            stats["block_counts"][blk.kind] += 1
            stats["max_rank"] = max(stats["max_rank"], entry["rank"])
            stats["total_nnz"] += entry["nnz"]
            hstat["counts"][blk.kind] += 1
            hstat["max_rank"] = max(hstat["max_rank"], entry["rank"])
            hstat["total_nnz"] += entry["nnz"]
        stats["block_counts"]["dropped"] += dropped
        hstat["t_build"] = time.perf_counter() - t0
        stats["halves"][parity] = hstat
        halves[parity] = (spec, blocks)
    return AltPlan(n=n, m=m, spec_odd=halves["odd"][0],
                   spec_even=halves["even"][0], blocks_odd=halves["odd"][1],
                   blocks_even=halves["even"][1], params=params, n0=n0,
                   tau=tau, stats=stats)


def plan_diagnostics(plan):
    st = plan.stats
    return {"n": plan.n, "m": plan.m, "n0": plan.n0,
            "max_rank": st["max_rank"], "total_nnz": st["total_nnz"],
            "block_counts": dict(st["block_counts"]),
            "levels_used": st["levels_used"], "t_factor": st["t_factor"],
            "t_by_class": dict(st["t_by_class"]),
            "per_block": list(st["per_block"])}


@dataclass
class ShtPlan:
    n: int
    alt_plans: list
    params: SamplingConfig

    @property
    def quadrature(self):
        return self.alt_plans[0].quadrature


class _ArrRef:
    """Placeholder for an array spilled to a shared scratch file."""

    __slots__ = ("off", "shape", "dtype")

    def __init__(self, off, shape, dtype):
        self.off, self.shape, self.dtype = off, shape, dtype


def _reap_spills(d):
    """Remove spill files of planner workers that no longer exist (a run
    killed between a worker's write and the parent's unlink leaves its
    payload file behind in tmpfs)."""
    try:
        names = os.listdir(d)
    except OSError:
        return
    for name in names:
        if not (name.startswith("bfsht_plan_") and name.endswith(".bin")):
            continue
        try:
            pid = int(name.split("_")[2])
            os.kill(pid, 0)
        except ProcessLookupError:
            try:
                os.unlink(os.path.join(d, name))
            except OSError:
                pass
        except (ValueError, IndexError, PermissionError):
            pass


def _spill_dir():
    # tmpfs when it has room for the payloads, else the regular temp dir
    _reap_spills("/dev/shm")
    try:
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize > (8 << 30):
            return "/dev/shm"
    except OSError:
        pass
    import tempfile
    return tempfile.gettempdir()


def _map_payloads(plans, fn):
    """Apply fn to every payload array of every plan, in place."""
    for pl in plans:
        for blocks in (pl.blocks_odd, pl.blocks_even):
            for blk in blocks:
                p = blk.payload
                if isinstance(p, ButterflyFactorization):
                    for f in p.factors:
                        f.rows, f.cols, f.vals = fn(f.rows), fn(f.cols), fn(f.vals)
                elif isinstance(p, LowRankFactor):
                    p.u, p.s, p.v = fn(p.u), fn(p.s), fn(p.v)
                else:
                    blk.payload = fn(p)


def _plan_orders(args):
    n, orders, params, n0, tau, spill, device = args
    quadrature = gauss_legendre(2 * n)
    out = []
    trace = os.environ.get("BFSHT_PLAN_TRACE")
    for m in orders:
        t0 = time.perf_counter()
        try:
            out.append(plan_alt(n, m, params, n0=n0, tau=tau,
                                quadrature=quadrature, device=device))
        except Exception as exc:
            raise RuntimeError(f"planning failed at order m={m}: {exc}") \
                from exc
        if trace:
            import sys
            print(f"[plan pid {os.getpid()}] m={m} {time.perf_counter() - t0:.2f}s",
                  file=sys.stderr, flush=True)
    if spill is None:
        return out, None
    # ship payloads through a shared file instead of the result pipe: the
    # parent maps it, so N=1024's ~17 GB of payload is never pickled
    path = os.path.join(spill, f"bfsht_plan_{os.getpid()}_{orders[0]}.bin")
    with open(path, "wb") as fh:
        pos = [0]

        def put(a):
            a = np.ascontiguousarray(a)
            ref = _ArrRef(pos[0], a.shape, a.dtype.str)
            if a.nbytes:
                fh.write(memoryview(a.reshape(-1)).cast("B"))
            pad = (-a.nbytes) % 64
            if pad:
                fh.write(b"\0" * pad)
            pos[0] += a.nbytes + pad
            return ref

        _map_payloads(out, put)
    for pl in out:
        for spec in (pl.spec_odd, pl.spec_even):
            if spec is not None:
                spec.quadrature = None
    return out, path


def _start_method():
    """fork is cheapest, but forking a process whose CUDA / NCCL threads are
    running can deadlock the child: use forkserver once CUDA is up."""
    import sys
    from . import legendre
    if legendre.device_tables_used():
        return "forkserver"   # this process holds a CUDA context (f3 tables)
    torch = sys.modules.get("torch")
    try:
        if torch is not None and torch.cuda.is_initialized():
            return "forkserver"
    except Exception:
        pass
    return "fork"


def plan_orders(n, orders, params=None, n0=None, tau=TAU_DEFAULT,
                processes=1, quadrature=None, device=None):
    """Plans for an arbitrary list of orders (one shard of an SHT), built in
    ``processes`` host processes (0/None = all cores); orders are dealt
    round-robin, which balances cost because it falls with m.  ``device``:
    tabulate matrix entries on that GPU (f3; the factors are unchanged)."""
    orders = [int(m) for m in orders]
    if params is None:
        params = SamplingConfig()
    n0 = N0_DEFAULT if n0 is None else n0
    if quadrature is None:
        quadrature = gauss_legendre(2 * n)
    if not processes or processes < 0:
        processes = os.cpu_count() or 1
    p = min(processes, len(orders))
    if p <= 1:
        plans = []
        for m in orders:
            try:
                plans.append(plan_alt(n, m, params, n0=n0, tau=tau,
                                      quadrature=quadrature, device=device))
            except Exception as exc:
                raise RuntimeError(
                    f"planning failed at order m={m}: {exc}") from exc
        return plans
    import multiprocessing as mp
    ctx = mp.get_context(_start_method())
    chunks = [orders[r::p] for r in range(p)]
    spill = _spill_dir()
    with ctx.Pool(p) as pool:
        res = pool.map(_plan_orders,
                       [(n, c, params, n0, tau, spill, device) for c in chunks])
    by_m = {}
    for chunk, (got, path) in zip(chunks, res):
        if path is not None:
            mm = np.memmap(path, dtype=np.uint8, mode="r")
            os.unlink(path)   # the mapping keeps the pages alive

            def get(ref, mm=mm):
                dt = np.dtype(ref.dtype)
                count = int(np.prod(ref.shape)) if ref.shape else 1
                return np.frombuffer(mm, dtype=dt, count=count,
                                     offset=ref.off).reshape(ref.shape)

            _map_payloads(got, get)
        for m, pl in zip(chunk, got):
            for spec in (pl.spec_odd, pl.spec_even):
                if spec is not None:
                    spec.quadrature = quadrature
            by_m[m] = pl
    return [by_m[m] for m in orders]


def plan_sht(n, params=None, n0=None, tau=TAU_DEFAULT, processes=1, device=None):
    """Plans for every order m = 0..2N-1 sharing one quadrature rule
    (sht.py:109-128).  ``processes > 1`` plans orders in parallel host
    processes; ``device`` tabulates entries on that GPU."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if params is None:
        params = SamplingConfig()
    if processes is not None and processes > 1 and n < 8:
        processes = 1
    plans = plan_orders(n, range(2 * n), params, n0, tau, processes, device=device)
    return ShtPlan(n=n, alt_plans=plans, params=params)
