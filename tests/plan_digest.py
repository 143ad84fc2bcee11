"""Canonical digest of an AltPlan in the reference layout.

Works on plans from this package and from the reference ``bfsht`` alike
(duck-typed on the reference attribute names, pkg/src/bfsht/alt.py:57-73),
so a digest recorded from the reference pins our planner bitwise.
"""
import hashlib

import numpy as np


def _arr(h, a, dtype):
    a = np.ascontiguousarray(np.asarray(a, dtype=dtype))
    h.update(str(a.shape).encode())
    h.update(a.tobytes())


def plan_digest(plan):
    h = hashlib.sha256()
    h.update(f"{plan.n}:{plan.m}:{plan.n0}:{plan.tau!r}".encode())
    for blocks in (plan.blocks_odd, plan.blocks_even):
        h.update(f"#{len(blocks)}".encode())
        for b in blocks:
            h.update(f"{tuple(b.row_range)}{tuple(b.col_range)}{b.kind}"
                     f"{b.level}{b.band}{tuple(b.trim)}".encode())
            p = b.payload
            if hasattr(p, "factors"):
                h.update(f"BF{tuple(p.shape)}{p.levels}{p.middle}"
                         f"{p.max_rank}".encode())
                for f in p.factors:
                    h.update(str(tuple(f.shape)).encode())
                    _arr(h, f.rows, np.int64)
                    _arr(h, f.cols, np.int64)
                    _arr(h, f.vals, np.float64)
            elif hasattr(p, "u"):
                h.update(b"LR")
                _arr(h, p.u, np.float64)
                _arr(h, p.s, np.float64)
                _arr(h, p.v, np.float64)
            else:
                h.update(b"DN")
                _arr(h, p, np.float64)
    return h.hexdigest()
