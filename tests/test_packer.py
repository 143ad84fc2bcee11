"""Packed device format vs the oracle, on CPU (numpy interpreter of the
exact engine semantics), incl. edge cases: single-parity top order, 1x1
blocks, depth-0..3 butterflies, low-rank blocks, reference-built plans."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt
from paper_2004_11346_b200.pack import pack_plans

import oracle.apply as OA
import packed_emulator as EMU

CASES = [(32, [20], 16, 1e-10), (64, [0, 3, 64, 126, 127], 16, 1e-10),
         (128, [100, 0, 1, 255], 16, 1e-10), (256, [0, 1, 300, 511], 512, 1e-12),
         (256, [256], 64, 1e-10)]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,ms,n0,tol", CASES)
def test_emulated_engine_matches_oracle(n, ms, n0, tol):
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=tol), n0=n0, quadrature=q)
             for m in ms]
    pk = pack_plans(plans)
    rng = np.random.default_rng(n)
    vecs = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
            for m in ms]
    for got, p, v in zip(EMU.alt_orders(pk, plans, 0, vecs), plans, vecs):
        assert rel(got, OA.alt_forward(p, v)) < 1e-14
    fs = [rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n) for _ in ms]
    for got, p, f in zip(EMU.alt_orders(pk, plans, 1, fs, q.weights), plans, fs):
        assert rel(got, OA.alt_inverse(p, f)) < 1e-14
    # every stored reference value lands in the tile store once; zero fill
    # (rotated tiles, structural zeros of ID blocks) stays small
    s = pk.stats
    assert s["tile_doubles"] >= s["payload_values"] - sum(
        len(p.blocks_odd) + len(p.blocks_even) for p in plans) * 64
    assert s["tile_doubles"] <= 1.5 * s["payload_values"] + 64 * 64


def test_pack_rejects_bad_trim():
    plan = plan_alt(16, 2, n0=8)
    blk = plan.blocks_even[0]
    blk.trim = (0, 99, 0, 1)
    with pytest.raises((RuntimeError, ValueError)):
        pack_plans([plan])


def test_tile_rotation_layout():
    plan = plan_alt(16, 0, n0=8)
    pk = pack_plans([plan])
    op = pk.ops[0]
    a = EMU.tile_matrix(pk, int(op["tile"]), int(op["R"]), int(op["C"]))
    assert a.shape == (op["R"], op["C"])
