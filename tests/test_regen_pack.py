"""On-GPU regeneration of dense turning tiles, host half:
  * the packer's recurrence coefficients equal the planner's
    (kernels/common.py:37-53) bitwise;
  * every regenerated tile, rebuilt by the host twin of the engine's
    generation from its seed block, equals the stored reference values
    bitwise (the gate SURVEY f1 names: regenerated tile == stored payload);
  * the emulated engine gives bitwise the same ALT with and without
    regeneration, and the oracle's result."""
import ctypes

import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, native, plan_alt
from paper_2004_11346_b200.legendre import recurrence_coefficients
from paper_2004_11346_b200.pack import pack_plans

import oracle.apply as OA
import packed_emulator as EMU


@pytest.mark.parametrize("m,k_max", [(0, 512), (1, 700), (37, 400), (255, 511), (1000, 2047)])
def test_rec_coeffs_match_planner(m, k_max):
    a, b = recurrence_coefficients(m, k_max)
    out = np.empty(2 * (k_max - m))
    assert native.host().bfsht_rec_coeffs(m, k_max, out.ctypes.data) == 0
    assert np.array_equal(out[0::2], a) and np.array_equal(out[1::2], b)


def _plans(n, ms, n0):
    q = gauss_legendre(2 * n)
    return [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=n0, quadrature=q) for m in ms]


def _dense_tiles(plan, h):
    """(r0, c0) -> the stored values of every 32-grid tile of turning blocks."""
    blocks = plan.blocks_odd if h == 0 else plan.blocks_even
    out = {}
    for blk in blocks:
        if blk.kind != "turning":
            continue
        r0, r1, c0, c1 = blk.trim
        a = np.asarray(blk.payload)
        for ra in range((r0 // 32) * 32, r1, 32):
            for ca in range((c0 // 32) * 32, c1, 32):
                rs, re_ = max(ra, r0), min(ra + 32, r1)
                cs, ce = max(ca, c0), min(ca + 32, c1)
                out[(rs, cs)] = a[rs - r0:re_ - r0, cs - c0:ce - c0]
    return out


@pytest.mark.parametrize("n,ms,n0", [(256, [3, 100, 300, 511], 64), (128, [0, 1, 64, 200], 32)])
def test_regenerated_tiles_equal_stored(n, ms, n0):
    plans = _plans(n, ms, n0)
    pk = pack_plans(plans, regen=1.0)
    assert pk.regen_tiles > 0
    ops = pk.ops[(pk.ops["flags"] & EMU.F_REGEN) != 0]
    ops = ops[ops["kind"] == EMU.OP_N]
    halves = pk.halves
    checked = 0
    for op in ops:
        seed = pk.tiles[int(op["tile"]):]
        r_a = int(seed[:1].view(np.int32)[0])
        # which half: the op's input entry lies in that half's x region
        h = int(np.nonzero((halves["x"] <= op["in"]) &
                           (op["in"] < halves["x"] + halves["ncols"]))[0][0])
        c_a = int(op["in"]) - int(halves["x"][h])
        got = EMU.regen_matrix(pk, int(op["tile"]), int(op["R"]), int(op["C"]))
        want = _dense_tiles(plans[h // 2], h % 2)[(r_a, c_a)]
        assert got.shape == want.shape
        assert np.array_equal(got, want), (h, r_a, c_a)
        checked += 1
    assert checked == pk.regen_tiles


@pytest.mark.parametrize("frac", [0.35, 1.0])
def test_emulated_alt_bitwise_with_regen(frac):
    n = 256
    ms = [2, 150, 400]
    plans = _plans(n, ms, 64)
    base = pack_plans(plans)
    pk = pack_plans(plans, regen=frac)
    assert 0 < pk.regen_tiles
    assert pk.stats["tile_doubles"] < base.stats["tile_doubles"]
    rng = np.random.default_rng(7)
    vecs = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m) for m in ms]
    for a, b, p, v in zip(EMU.alt_orders(pk, plans, 0, vecs), EMU.alt_orders(base, plans, 0, vecs),
                          plans, vecs):
        assert np.array_equal(a, b)
        want = OA.alt_forward(p, v)
        assert np.linalg.norm(a - want) <= 1e-14 * np.linalg.norm(want)
    q = plans[0].quadrature
    fs = [rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n) for _ in ms]
    for a, b in zip(EMU.alt_orders(pk, plans, 1, fs, q.weights),
                    EMU.alt_orders(base, plans, 1, fs, q.weights)):
        assert np.array_equal(a, b)
