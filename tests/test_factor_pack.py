"""A single ButterflyFactorization packed as a one-half plan (api._FactorPlan,
the device path of idbf_apply / idbf_apply_transpose, butterfly.py:275-292):
the emulated engine reproduces the oracle on the golden DFT-kernel factor
and on rectangular factors, on CPU."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig
from paper_2004_11346_b200.factors import FunctionOracle, idbf_factor
from paper_2004_11346_b200.pack import NRHS, pack_plans
from paper_2004_11346_b200.api import _FactorPlan

import golden_data
import oracle.apply as OA
import packed_emulator as EMU


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def emulate(fac, x, direction):
    pk = pack_plans([_FactorPlan(fac)])
    h = pk.halves[0]
    arena = np.full((pk.stats["arena"], NRHS), np.nan)
    k = x.shape[1]
    if direction == 0:
        arena[h["x"]:h["x"] + h["ncols"]] = 0.0
        arena[h["x"]:h["x"] + h["ncols"], :k] = x
        EMU.run_direction(pk, arena, 0)
        yr = int(pk.info[10])
        return arena[yr + 2 * np.arange(pk.n), :k]
    arena[h["y"]:h["y"] + pk.n] = 0.0
    arena[h["y"]:h["y"] + pk.n, :k] = x
    EMU.run_direction(pk, arena, 1)
    return arena[h["x"]:h["x"] + h["ncols"], :k]


def dft_factor(nk, leaf_max):
    scale = 1.0 / np.sqrt(nk)
    return idbf_factor(FunctionOracle(
        lambda i, j: np.cos(2.0 * np.pi * i * j / nk) * scale, (nk, nk)),
        SamplingConfig(), leaf_max=leaf_max)


def test_golden_factor_emulated():
    fac = dft_factor(128, 16)
    x = golden_data.seeded_complex(77, 128).real
    got = emulate(fac, x[:, None], 0)[:, 0]
    assert rel(got, OA.idbf_apply(fac, x)) < 1e-14
    got = emulate(fac, x[:, None], 1)[:, 0]
    assert rel(got, OA.idbf_apply_transpose(fac, x)) < 1e-14


@pytest.mark.parametrize("shape,leaf", [((96, 160), 12), ((200, 72), 16), ((64, 64), 64)])
def test_rectangular_factor_emulated(shape, leaf):
    h, w = shape
    fac = idbf_factor(FunctionOracle(
        lambda i, j: np.cos(0.37 * i * j / np.sqrt(h * w) * 40.0 + 0.1 * i), shape),
        SamplingConfig(), leaf_max=leaf)
    rng = np.random.default_rng(h + w)
    x = rng.standard_normal((w, 3))
    assert rel(emulate(fac, x, 0), OA.idbf_apply(fac, x)) < 1e-14
    y = rng.standard_normal((h, 3))
    assert rel(emulate(fac, y, 1), OA.idbf_apply_transpose(fac, y)) < 1e-14
