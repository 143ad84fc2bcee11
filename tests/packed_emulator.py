"""Numpy interpreter of the packed device format — test infrastructure.

Executes a PackedPlan's stages task by task with the exact semantics the
CUDA engine implements (csrc/engine.cu, format.h), so the packer can be
checked against the oracle on CPU, without a GPU.
"""
import numpy as np

from paper_2004_11346_b200.pack import NRHS

OP_N, OP_T, OP_ADD = 0, 1, 2
F_GATHER, F_LANEMAP, F_REGEN = 1, 2, 4
SLOTS = 64   # outputs per task (format.h BF_SLOTS)


def tile_matrix(pk, off, R, C):
    """R x C tile stored as zero-padded 4x4 blocks (format.h)."""
    c4 = (C + 3) // 4
    r = np.arange(R)[:, None]
    c = np.arange(C)[None, :]
    return pk.tiles[off + ((r >> 2) * c4 + (c >> 2)) * 16 + (r & 3) * 4 + (c & 3)]


def regen_matrix(pk, off, R, C):
    """R x C values of a regenerated tile, through the host twin of the
    engine's generation (bfsht_regen_tile_host)."""
    import ctypes
    from paper_2004_11346_b200 import native
    lib = native.host()
    c4 = (C + 3) // 4
    buf = np.zeros(((R + 3) // 4) * c4 * 16)
    seed = pk.tiles[off:]
    rc = lib.bfsht_regen_tile_host(seed.ctypes.data, R, C, pk.rec.ctypes.data,
                                   pk.xpos.ctypes.data, pk.mag_min, buf.ctypes.data)
    assert rc == 0
    r = np.arange(R)[:, None]
    c = np.arange(C)[None, :]
    return buf[((r >> 2) * c4 + (c >> 2)) * 16 + (r & 3) * 4 + (c & 3)]


CF_LAST, CF_ADD = 8, 16   # format.h bf_crec_flags


def run_chain_stage(pk, arena, recs, bund):
    """One stage from its chain schedule (format.h bf_crec records in
    bundles; engine.cu alt_chain_kernel): every bundle's records in order,
    a folded index add right after its tile op, outputs stored on the
    record flagged last-of-task."""
    for b in range(len(bund) - 1):
        acc = np.zeros((SLOTS, NRHS))
        for r in recs[bund[b]:bund[b + 1]]:
            kind, R, C, off = int(r["kind"]), int(r["R"]), int(r["C"]), int(r["off"])
            flags = int(r["flags"])
            gather = bool(flags & F_GATHER)
            if kind == OP_ADD:
                for j in range(R):
                    src = int(pk.idx[r["in"] + j]) if gather else int(r["in"]) + j
                    if src >= 0:
                        acc[off + j] += arena[src]
            else:
                a = tile_matrix(pk, int(r["tile"]) * 16, R, C)
                nin = C if kind == OP_N else R
                src = pk.idx[r["in"]:r["in"] + nin] if gather \
                    else np.arange(r["in"], r["in"] + nin)
                v = arena[src]
                res = a @ v if kind == OP_N else a.T @ v
                width = res.shape[0]
                for slot in range(SLOTS):
                    if flags & F_LANEMAP:
                        sl = int(pk.maps[int(r["aux"]) * SLOTS + slot])
                    else:
                        sl = slot - off
                    if 0 <= sl < width:
                        acc[slot] += res[sl]
                if flags & CF_ADD:
                    for j in range(int(r["addR"])):
                        src = int(pk.idx[r["add_in"] + j])
                        if src >= 0:
                            acc[int(r["addoff"]) + j] += arena[src]
            if flags & CF_LAST:
                nout = int(r["nout"]) & 0xFF
                stride = (int(r["nout"]) >> 8) or 1
                arena[r["out"] + stride * np.arange(nout)] = acc[:nout]
                acc[:] = 0.0


def run_direction(pk, arena, direction, chain=None):
    """chain = (records, bundle bounds, per-stage info) from
    pack.chain_schedule: the stages it covers run from their records."""
    bounds = pk.stages_fwd if direction == 0 else pk.stages_inv
    for s in range(len(bounds) - 1):
        if chain is not None and chain[2][s, 1] > 0:
            b0, nb = int(chain[2][s, 0]), int(chain[2][s, 1])
            run_chain_stage(pk, arena, chain[0], chain[1][b0:b0 + nb + 1])
            continue
        for t in pk.tasks[bounds[s]:bounds[s + 1]]:
            acc = np.zeros((SLOTS, NRHS))
            for op in pk.ops[t["op_begin"]:t["op_begin"] + t["op_count"]]:
                kind, R, C, off = int(op["kind"]), int(op["R"]), int(op["C"]), int(op["off"])
                gather = bool(op["flags"] & F_GATHER)
                if kind == OP_ADD:
                    for j in range(R):
                        src = int(pk.idx[op["in"] + j]) if gather else int(op["in"]) + j
                        if src >= 0:
                            acc[off + j] += arena[src]
                    continue
                if op["flags"] & F_REGEN:
                    a = regen_matrix(pk, int(op["tile"]), R, C)
                else:
                    a = tile_matrix(pk, int(op["tile"]), R, C)
                nin = C if kind == OP_N else R
                src = pk.idx[op["in"]:op["in"] + nin] if gather \
                    else np.arange(op["in"], op["in"] + nin)
                v = arena[src]
                res = a @ v if kind == OP_N else a.T @ v
                width = res.shape[0]
                for slot in range(SLOTS):
                    if op["flags"] & F_LANEMAP:
                        sl = int(pk.maps[int(op["aux"]) * SLOTS + slot])
                    else:
                        sl = slot - off
                    if 0 <= sl < width:
                        acc[slot] += res[sl]
            nout = int(t["nout"]) & 0xFF
            stride = (int(t["nout"]) >> 8) or 1
            arena[t["out"] + stride * np.arange(nout)] = acc[:nout]


def alt_orders(pk, plans, direction, vectors, weights=None):
    """Per-order ALT through the emulated engine: complex vectors in/out."""
    n = pk.n
    arena = np.full((pk.stats["arena"], NRHS), np.nan)
    h = pk.halves
    outs = []
    if direction == 0:
        for o, vec in enumerate(vectors):
            for par in range(2):
                hf = h[2 * o + par]
                if hf["ncols"] == 0:
                    continue
                k0 = 1 if par == 0 else 0
                vals = np.asarray(vec, dtype=np.complex128)[k0::2][:hf["ncols"]]
                arena[hf["x"]:hf["x"] + hf["ncols"]] = np.stack(
                    [vals.real, vals.imag, 0 * vals.real, 0 * vals.real], 1)
        run_direction(pk, arena, 0)
        yr, no = int(pk.info[10]), len(vectors)
        for o in range(len(vectors)):
            go = np.zeros(n, complex)
            ge = np.zeros(n, complex)
            for par, g in ((0, go), (1, ge)):
                hf = h[2 * o + par]
                if hf["ncols"]:
                    # forward results: row-major Yr[r][order][parity]
                    e = arena[yr + np.arange(n) * 2 * no + 2 * o + par]
                    g[:] = e[:, 0] + 1j * e[:, 1]
            col = np.empty(2 * n, complex)
            col[n:] = ge + go
            col[n - 1::-1] = ge - go
            outs.append(col)
        return outs
    for o, f in enumerate(vectors):
        f = np.asarray(f, dtype=np.complex128)
        up, lo = f[n:], f[n - 1::-1]
        w = weights[n:]
        for par, val in ((0, w * (up - lo)), (1, w * (up + lo))):
            hf = h[2 * o + par]
            if hf["ncols"]:
                arena[hf["y"]:hf["y"] + n] = np.stack(
                    [val.real, val.imag, 0 * val.real, 0 * val.real], 1)
    run_direction(pk, arena, 1)
    for o, plan in enumerate(plans):
        beta = np.zeros(2 * n - plan.m, complex)
        for par in range(2):
            hf = h[2 * o + par]
            if hf["ncols"]:
                e = arena[hf["x"]:hf["x"] + hf["ncols"]]
                beta[(1 if par == 0 else 0)::2] = e[:, 0] + 1j * e[:, 1]
        outs.append(beta)
    return outs
