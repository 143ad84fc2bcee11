"""Write the golden fixtures from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``bfsht`` from /root/reference/pkg/src (or baseline/_ref), builds
reference plans, and records
  * plan digests (tests/plan_digest.py) for a set of (N, m, n0, tol) cases —
    these pin our planner to the reference planner bitwise;
  * reference alt_forward / alt_inverse outputs on seeded complex inputs;
  * reference sht_forward / sht_inverse outputs for small N;
  * a reference IDBF of the synthetic DFT kernel (test_butterfly.py:14-18)
    with its apply / apply-transpose outputs.
Inputs are regenerated from the recorded seeds, so only outputs are stored.
The fixtures travel with the repo; the reference does not.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
for cand in ("/root/reference/pkg/src",
             os.path.join(os.path.dirname(os.path.dirname(HERE)), "baseline", "_ref")):
    if os.path.isdir(cand):
        sys.path.insert(0, cand)
        break

import bfsht.alt as RA  # noqa: E402
import bfsht.butterfly as RB  # noqa: E402
import bfsht.sht as RS  # noqa: E402
from bfsht.lowrank import FunctionOracle, SamplingConfig  # noqa: E402
from bfsht.special import gauss_legendre  # noqa: E402

from plan_digest import plan_digest  # noqa: E402

# (n, m, n0, tol): small-N cases mirror pkg/tests/test_alt.py:19; the N=256
# and N=1024 cases are BASELINE configs 1-2 (tol 1e-12, default n0=512) at
# orders spanning butterfly depths 0-3, low-rank and turning blocks.
ALT_CASES = [(32, 20, 16, 1e-10), (64, 0, 16, 1e-10), (64, 3, 16, 1e-10),
             (64, 64, 16, 1e-10), (64, 126, 16, 1e-10), (64, 127, 16, 1e-10),
             (128, 100, 16, 1e-10), (256, 256, 64, 1e-10),
             (256, 0, 512, 1e-12), (256, 1, 512, 1e-12), (256, 300, 512, 1e-12),
             (256, 511, 512, 1e-12),
             (1024, 0, 512, 1e-12), (1024, 1, 512, 1e-12),
             (1024, 100, 512, 1e-12), (1024, 1000, 512, 1e-12),
             (1024, 2000, 512, 1e-12), (1024, 2047, 512, 1e-12)]
SHT_NS = [4, 8, 16, 32]


def seeded_complex(seed, size):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(size) + 1j * rng.standard_normal(size)


def sht_flat(n, seed):
    rng = np.random.default_rng(seed)
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        k = np.arange(abs(m), 2 * n)
        parts.append((rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
                     / (1.0 + k))
    return np.concatenate(parts)


def main():
    meta = {"alt": [], "sht": [], "butterfly": {}}
    arrays = {}
    quads = {}
    for i, (n, m, n0, tol) in enumerate(ALT_CASES):
        q = quads.setdefault(n, gauss_legendre(2 * n))
        plan = RA.plan_alt(n, m, SamplingConfig(tolerance=tol), n0=n0,
                           quadrature=q)
        beta = seeded_complex(1000 + i, 2 * n - m)
        f = seeded_complex(2000 + i, 2 * n)
        arrays[f"alt{i}_fwd"] = RA.alt_forward(plan, beta).values
        arrays[f"alt{i}_inv"] = RA.alt_inverse(plan, f).values
        meta["alt"].append({"n": n, "m": m, "n0": n0, "tol": tol,
                            "seed_fwd": 1000 + i, "seed_inv": 2000 + i,
                            "digest": plan_digest(plan),
                            "total_nnz": int(plan.stats["total_nnz"])})
        print("alt", n, m, flush=True)
    for n in SHT_NS:
        plan = RS.plan_sht(n)
        flat = sht_flat(n, 3 * n)
        coeffs = RS.ShtCoeffs.unpack(n, flat)
        grid = RS.sht_forward(plan, coeffs).values
        rng = np.random.default_rng(100 + n)
        vals = rng.standard_normal((2 * n, 4 * n - 1)) \
            + 1j * rng.standard_normal((2 * n, 4 * n - 1))
        arrays[f"sht{n}_fwd"] = grid
        arrays[f"sht{n}_inv"] = RS.sht_inverse(plan, vals).pack()
        meta["sht"].append({"n": n, "seed_coeffs": 3 * n, "seed_grid": 100 + n,
                            "digests": [plan_digest(p) for p in plan.alt_plans]})
        print("sht", n, flush=True)
    nk = 128
    scale = 1.0 / np.sqrt(nk)
    oracle = FunctionOracle(
        lambda i, j: np.cos(2.0 * np.pi * i * j / nk) * scale, (nk, nk))
    fac = RB.idbf_factor(oracle, SamplingConfig(), leaf_max=16)
    x = seeded_complex(77, nk).real
    arrays["bf_fwd"] = RB.idbf_apply(fac, x)
    arrays["bf_inv"] = RB.idbf_apply_transpose(fac, x)
    meta["butterfly"] = {"n": nk, "leaf_max": 16, "seed": 77,
                         "levels": fac.levels, "nnz": fac.nnz,
                         "shapes": [list(f.shape) for f in fac.factors]}
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", sum(a.nbytes for a in arrays.values()), "bytes")


if __name__ == "__main__":
    main()
