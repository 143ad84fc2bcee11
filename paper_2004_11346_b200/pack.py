"""Reference-layout plans -> packed device format (host side).

``pack_plans(plans)`` flattens a list of ``AltPlan`` objects — from this
package's planner or from the reference ``bfsht`` itself; only the
reference attribute names are used (pkg/src/bfsht/alt.py:57-73,
butterfly.py:45-80, lowrank.py:184-202) — into a ``bfsht_manifest`` and
calls the native packer (csrc/packer.cpp) through the C ABI.  The result
is a ``PackedPlan`` holding numpy views of the packed arrays.
"""
import ctypes

import numpy as np

from . import native

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64


class BlockDesc(ctypes.Structure):
    _fields_ = [("order", _I32), ("parity", _I32), ("kind", _I32),
                ("r0", _I32), ("r1", _I32), ("c0", _I32), ("c1", _I32),
                ("rank", _I32), ("a", _P), ("b", _P), ("c", _P),
                ("nfac", _I32), ("levels", _I32), ("middle", _I32),
                ("fshape", _P), ("fnnz", _P), ("frows", _P), ("fcols", _P),
                ("fvals", _P)]


class Manifest(ctypes.Structure):
    _fields_ = [("n", _I32), ("norders", _I32), ("m", _P), ("ncols", _P),
                ("nblocks", _I64), ("blocks", _P), ("regen", ctypes.c_double),
                ("x_pos", _P), ("mant0", _P), ("exp0", _P),
                ("mag_min", ctypes.c_double)]


def declare(lib):
    lib.bfsht_pack_plan.restype = ctypes.c_int
    lib.bfsht_pack_plan.argtypes = [ctypes.POINTER(Manifest), ctypes.c_int,
                                    ctypes.POINTER(_P)]
    lib.bfsht_packed_info.restype = ctypes.c_int
    lib.bfsht_packed_info.argtypes = [_P, ctypes.POINTER(_I64)]
    lib.bfsht_packed_arrays.restype = ctypes.c_int
    lib.bfsht_packed_arrays.argtypes = [_P, ctypes.POINTER(_P)]
    lib.bfsht_rec_coeffs.restype = ctypes.c_int
    lib.bfsht_rec_coeffs.argtypes = [_I64, _I64, _P]
    lib.bfsht_regen_tile_host.restype = ctypes.c_int
    lib.bfsht_regen_tile_host.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P,
                                          ctypes.c_double, _P]
    lib.bfsht_packed_free.restype = None
    lib.bfsht_packed_free.argtypes = [_P]
    lib.bfsht_chain_schedule.restype = ctypes.c_int
    lib.bfsht_chain_schedule.argtypes = [_P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
    lib.bfsht_chain_sched_arrays.restype = ctypes.c_int
    lib.bfsht_chain_sched_arrays.argtypes = [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64),
                                             ctypes.POINTER(_P), ctypes.POINTER(_I64),
                                             ctypes.POINTER(_P)]
    lib.bfsht_chain_sched_free.restype = None
    lib.bfsht_chain_sched_free.argtypes = [_P]
    lib.bfsht_host_last_error.restype = ctypes.c_char_p
    lib.bfsht_host_last_error.argtypes = []


OP_DTYPE = np.dtype([("tile", "<i8"), ("in", "<i4"), ("aux", "<i4"),
                     ("kind", "u1"), ("R", "u1"), ("C", "u1"), ("off", "u1"),
                     ("flags", "u1"), ("pad0", "u1"), ("pad1", "<u2")])
TASK_DTYPE = np.dtype([("op_begin", "<i4"), ("op_count", "<i4"),
                       ("out", "<i4"), ("nout", "<i4")])
HALF_DTYPE = np.dtype([("x", "<i4"), ("y", "<i4"), ("ncols", "<i4"),
                       ("m", "<i4")])
NRHS = 4

INFO_KEYS = ("tile_doubles", "ops", "idx", "maps", "tasks", "arena",
             "halves", "stages_fwd", "stages_inv", "payload_values",
             "yr", "butterfly_blocks", "lowrank_blocks",
             "dense_blocks", "n", "norders", "free_fwd", "free_inv",
             "regen_tiles", "regen_values", "rec_doubles", "xpos_doubles")
INFO_LEN = 24


CREC_DTYPE = np.dtype([("tile", "<u4"), ("in", "<i4"), ("aux", "<i4"),
                       ("kind", "u1"), ("R", "u1"), ("C", "u1"), ("off", "u1"),
                       ("flags", "u1"), ("addR", "u1"), ("addoff", "u1"), ("pad", "u1"),
                       ("add_in", "<i4"), ("out", "<i4"), ("nout", "<i4")])


def chain_schedule(packed, direction, warps=148 * 12, mode=1, per_warp=8, cfix=3072):
    """Host chain schedule of one direction (include/bfsht_b200.h
    bfsht_chain_schedule): (records, bundle bounds, per-stage int64 (nst, 4)
    = first bound entry, bundles, records, folded adds) as numpy copies."""
    lib = native.host()
    bounds = np.ascontiguousarray(packed.stages_fwd if direction == 0 else packed.stages_inv)
    nst = len(bounds) - 1
    h = _P()
    rc = lib.bfsht_chain_schedule(packed.ops.ctypes.data, packed.tasks.ctypes.data,
                                  bounds.ctypes.data, nst, warps, mode, per_warp, cfix,
                                  ctypes.byref(h))
    if rc:
        raise RuntimeError("bfsht_chain_schedule: " + lib.bfsht_host_last_error().decode())
    try:
        recs, bund, stage = _P(), _P(), _P()
        nrec, nbund = _I64(), _I64()
        lib.bfsht_chain_sched_arrays(h, ctypes.byref(recs), ctypes.byref(nrec),
                                     ctypes.byref(bund), ctypes.byref(nbund),
                                     ctypes.byref(stage))

        def copy(ptr, dtype, count):
            if not count or not ptr.value:
                return np.zeros(0, dtype=dtype)
            buf = (ctypes.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr.value)
            return np.frombuffer(buf, dtype=dtype, count=count).copy()

        return (copy(recs, CREC_DTYPE, nrec.value), copy(bund, np.int32, nbund.value),
                copy(stage, np.int64, 4 * nst).reshape(nst, 4))
    finally:
        lib.bfsht_chain_sched_free(h)


def _addr(a):
    return a.ctypes.data if a is not None and a.size else 0


class PackedPlan:
    """Packed device-format plan (host memory, owned by the native packer)."""

    def __init__(self, handle, lib):
        self._h = handle
        self._lib = lib
        info = (_I64 * INFO_LEN)()
        lib.bfsht_packed_info(handle, info)
        self.info = np.array(list(info), dtype=np.int64)
        self.stats = dict(zip(INFO_KEYS, (int(v) for v in self.info)))
        arr = (_P * 12)()
        lib.bfsht_packed_arrays(handle, arr)
        s = self.stats

        def view(i, dtype, count):
            if count == 0 or not arr[i]:
                return np.zeros(0, dtype=dtype)
            buf = (ctypes.c_char * (count * np.dtype(dtype).itemsize)) \
                .from_address(arr[i])
            return np.frombuffer(buf, dtype=dtype, count=count)

        self.tiles = view(0, np.float64, s["tile_doubles"])
        self.ops = view(1, OP_DTYPE, s["ops"])
        self.idx = view(2, np.int32, s["idx"])
        self.maps = view(3, np.int8, s["maps"] * 64)
        self.tasks = view(4, TASK_DTYPE, s["tasks"])
        self.halves = view(5, HALF_DTYPE, s["halves"])
        self.stages_fwd = view(6, np.int64, s["stages_fwd"] + 1)
        self.stages_inv = view(7, np.int64, s["stages_inv"] + 1)
        self.rec = view(8, np.float64, s["rec_doubles"])
        self.xpos = view(9, np.float64, s["xpos_doubles"])
        nflow = int(self.info[23])
        self.flow = view(10, np.int32, nflow)
        self.tinfo = view(11, np.int32, s["tasks"] if nflow else 0)
        self.mag_min = float(self.info[22:23].view(np.float64)[0])

    @property
    def regen_tiles(self):
        return self.stats["regen_tiles"]

    def stored_payload_values(self):
        """Reference values that cross HBM (regenerated tiles excluded)."""
        return self.stats["payload_values"] - self.stats["regen_values"]

    def seed_bytes(self):
        """Bytes of the regeneration seed blocks (read instead of values)."""
        return 8 * self._seed_doubles()

    def _seed_doubles(self):
        sel = (self.ops["flags"] & 4) != 0
        if not sel.any():
            return 0
        tiles, first = np.unique(self.ops["tile"][sel], return_index=True)
        rows = self.ops["R"][sel][first].astype(np.int64)
        chains = np.where(self.ops["C"][sel][first] > 16, 2, 1)   # format.h bf_seed_chains
        return int(np.sum((2 + 3 * rows * chains + 15) // 16 * 16))

    @property
    def n(self):
        return self.stats["n"]

    @property
    def orders(self):
        return self.halves["m"][0::2].copy()

    def payload_bytes(self):
        """Algorithmic payload bytes read per direction (8 per stored value)."""
        return 8 * self.stats["payload_values"]

    def close(self):
        if self._h:
            self._lib.bfsht_packed_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------- plan cache
# Packed plans on disk ("compact device-plan cache"): the
# packed arrays exactly as uploaded, each 4 KB aligned so a load is a set of
# read-only memory maps that DevicePlan uploads without another host copy.
# Planning N=1024 takes seconds here but the reference needs minutes (hours
# at N=4096); a cached plan skips planning and packing entirely.
_PK_MAGIC = b"BFPK"
_PK_VERSION = 2   # 2: two-chain regeneration seed blocks
_PK_ALIGN = 4096
_PK_FIELDS = ("tiles", "ops", "idx", "maps", "tasks", "halves", "stages_fwd",
              "stages_inv", "rec", "xpos", "flow", "tinfo")


def save_packed(pk, path):
    """Write a PackedPlan (or a loaded one) to `path`."""
    import struct
    arrays = [np.ascontiguousarray(getattr(pk, f)) for f in _PK_FIELDS]
    head = _PK_MAGIC + struct.pack("<II", _PK_VERSION, len(arrays))
    head += np.asarray(pk.info, dtype="<i8").tobytes()
    offs, pos = [], _PK_ALIGN
    for a in arrays:
        offs.append(pos)
        pos += -(-a.nbytes // _PK_ALIGN) * _PK_ALIGN
    head += np.asarray([[o, a.nbytes] for o, a in zip(offs, arrays)], dtype="<i8").tobytes()
    if len(head) > _PK_ALIGN:
        raise ValueError("plan cache header too large")
    with open(path, "wb") as fh:
        fh.write(head.ljust(_PK_ALIGN, b"\0"))
        for o, a in zip(offs, arrays):
            fh.seek(o)
            fh.write(memoryview(a).cast("B"))
        fh.truncate(pos)


class LoadedPlan:
    """A packed plan memory-mapped from a cache file: the PackedPlan
    attributes DevicePlan and the tests read."""

    def __init__(self, path):
        import struct
        with open(path, "rb") as fh:
            head = fh.read(_PK_ALIGN)
        if head[:4] != _PK_MAGIC:
            raise ValueError(f"{path}: not a packed-plan file")
        ver, count = struct.unpack("<II", head[4:12])
        if ver != _PK_VERSION or count != len(_PK_FIELDS):
            raise ValueError(f"{path}: unsupported packed-plan version {ver}")
        self.info = np.frombuffer(head, dtype="<i8", count=INFO_LEN, offset=12).copy()
        self.stats = dict(zip(INFO_KEYS, (int(v) for v in self.info)))
        tab = np.frombuffer(head, dtype="<i8", count=2 * count, offset=12 + 8 * INFO_LEN)
        dtypes = (np.float64, OP_DTYPE, np.int32, np.int8, TASK_DTYPE, HALF_DTYPE,
                  np.int64, np.int64, np.float64, np.float64, np.int32, np.int32)
        for f, dt, (off, nb) in zip(_PK_FIELDS, dtypes, tab.reshape(-1, 2)):
            dt = np.dtype(dt)
            if nb == 0:
                setattr(self, f, np.zeros(0, dtype=dt))
            else:
                setattr(self, f, np.memmap(path, dtype=dt, mode="r", offset=int(off),
                                           shape=(int(nb) // dt.itemsize,)))
        self.mag_min = float(self.info[22:23].view(np.float64)[0])

    n = PackedPlan.n
    orders = PackedPlan.orders
    payload_bytes = PackedPlan.payload_bytes
    regen_tiles = PackedPlan.regen_tiles
    stored_payload_values = PackedPlan.stored_payload_values
    seed_bytes = PackedPlan.seed_bytes
    _seed_doubles = PackedPlan._seed_doubles


def load_packed(path):
    return LoadedPlan(path)


def _kind_of(payload):
    if hasattr(payload, "factors"):
        return 0
    if hasattr(payload, "u") and hasattr(payload, "s"):
        return 1
    return 2


def pack_plans(plans, n=None, threads=0, regen=0.0):
    """Pack AltPlans (all at the same half-size N) into the device format.

    regen in [0, 1]: fraction of the full-height dense turning tiles stored
    as recurrence seeds and regenerated on the GPU."""
    plans = list(plans)
    if not plans and n is None:
        raise ValueError("nothing to pack")
    n = plans[0].n if n is None else n
    keep = []
    ms = np.array([p.m for p in plans], dtype=np.int32)
    ncols = np.zeros(2 * len(plans), dtype=np.int32)
    descs = []
    for o, plan in enumerate(plans):
        if plan.n != n:
            raise ValueError(f"plan for m={plan.m} has N={plan.n}, expected {n}")
        for par, (spec, blocks) in enumerate(((plan.spec_odd, plan.blocks_odd),
                                              (plan.spec_even,
                                               plan.blocks_even))):
            if spec is None:
                continue
            ncols[2 * o + par] = spec.num_cols
            for blk in blocks:
                d = BlockDesc()
                d.order, d.parity = o, par
                d.r0, d.r1, d.c0, d.c1 = (int(v) for v in blk.trim)
                p = blk.payload
                d.kind = _kind_of(p)
                if d.kind == 2:
                    a = np.ascontiguousarray(p, dtype=np.float64)
                    if a.shape != (d.r1 - d.r0, d.c1 - d.c0):
                        raise ValueError("dense payload shape does not match "
                                         "its trim")
                    keep.append(a)
                    d.a = _addr(a)
                elif d.kind == 1:
                    u = np.ascontiguousarray(p.u, dtype=np.float64)
                    s = np.ascontiguousarray(p.s, dtype=np.float64)
                    v = np.ascontiguousarray(p.v, dtype=np.float64)
                    keep += [u, s, v]
                    d.rank = s.size
                    d.a, d.b, d.c = _addr(u), _addr(s), _addr(v)
                else:
                    nf = len(p.factors)
                    shape = np.array([x for f in p.factors for x in f.shape],
                                     dtype=np.int64)
                    nnz = np.array([f.vals.size for f in p.factors],
                                   dtype=np.int64)
                    rows = [np.ascontiguousarray(f.rows, dtype=np.int64)
                            for f in p.factors]
                    cols = [np.ascontiguousarray(f.cols, dtype=np.int64)
                            for f in p.factors]
                    vals = [np.ascontiguousarray(f.vals, dtype=np.float64)
                            for f in p.factors]
                    rp = (_P * nf)(*[_addr(x) for x in rows])
                    cp = (_P * nf)(*[_addr(x) for x in cols])
                    vp = (_P * nf)(*[_addr(x) for x in vals])
                    keep += [shape, nnz, rows, cols, vals, rp, cp, vp]
                    d.nfac, d.levels, d.middle = nf, p.levels, p.middle
                    d.fshape, d.fnnz = _addr(shape), _addr(nnz)
                    d.frows = ctypes.cast(rp, _P)
                    d.fcols = ctypes.cast(cp, _P)
                    d.fvals = ctypes.cast(vp, _P)
                descs.append(d)
    arr = (BlockDesc * max(len(descs), 1))(*descs)
    man = Manifest(n=n, norders=len(plans), m=_addr(ms), ncols=_addr(ncols),
                   nblocks=len(descs), blocks=ctypes.cast(arr, _P))
    if regen > 0.0 and plans:
        from .legendre import MAG_MIN, start_values
        spec = plans[0].spec_odd if plans[0].spec_odd is not None else plans[0].spec_even
        x_pos = np.ascontiguousarray(spec.x_pos, dtype=np.float64)
        mant0 = np.empty((len(plans), n), dtype=np.float64)
        exp0 = np.empty((len(plans), n), dtype=np.int32)
        for o, plan in enumerate(plans):
            mant0[o], exp0[o] = start_values(plan.m, x_pos)
        keep += [x_pos, mant0, exp0]
        man.regen = float(regen)
        man.x_pos, man.mant0, man.exp0 = _addr(x_pos), _addr(mant0), _addr(exp0)
        man.mag_min = MAG_MIN
    lib = native.host()
    out = _P()
    rc = lib.bfsht_pack_plan(ctypes.byref(man), int(threads), ctypes.byref(out))
    if rc != 0:
        raise RuntimeError("bfsht_pack_plan failed: "
                           + lib.bfsht_host_last_error().decode())
    del keep
    return PackedPlan(out, lib)
