"""The CPU oracle, pinned to the reference's own outputs (golden vectors)."""
import numpy as np
import pytest

from paper_2004_11346_b200 import (SamplingConfig, gauss_legendre,
                                   idbf_factor, plan_alt, plan_sht)
from paper_2004_11346_b200.factors import FunctionOracle

import golden_data
import oracle.apply as OA
import oracle.dense as OD

META, ARR = golden_data.load()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("i", range(len(META["alt"])),
                         ids=lambda i: f"n{META['alt'][i]['n']}m{META['alt'][i]['m']}")
def test_oracle_alt_reproduces_reference(i):
    c = META["alt"][i]
    n, m = c["n"], c["m"]
    plan = plan_alt(n, m, SamplingConfig(tolerance=c["tol"]), n0=c["n0"],
                    quadrature=gauss_legendre(2 * n))
    beta = golden_data.seeded_complex(c["seed_fwd"], 2 * n - m)
    f = golden_data.seeded_complex(c["seed_inv"], 2 * n)
    # identical plans + identical scipy/BLAS calls => bitwise equal
    assert np.array_equal(OA.alt_forward(plan, beta), ARR[f"alt{i}_fwd"])
    assert np.array_equal(OA.alt_inverse(plan, f), ARR[f"alt{i}_inv"])


@pytest.mark.parametrize("entry", META["sht"], ids=lambda e: f"n{e['n']}")
def test_oracle_sht_reproduces_reference(entry):
    n = entry["n"]
    plan = plan_sht(n)
    flat = golden_data.sht_flat(n, entry["seed_coeffs"])
    grid = OA.sht_forward(plan.alt_plans, n, flat)
    assert rel(grid, ARR[f"sht{n}_fwd"]) < 1e-15
    vals = golden_data.sht_grid(n, entry["seed_grid"])
    assert rel(OA.sht_inverse(plan.alt_plans, n, vals), ARR[f"sht{n}_inv"]) < 1e-15


def test_oracle_butterfly_dft_kernel():
    b = META["butterfly"]
    nk = b["n"]
    scale = 1.0 / np.sqrt(nk)
    fac = idbf_factor(FunctionOracle(
        lambda i, j: np.cos(2.0 * np.pi * i * j / nk) * scale, (nk, nk)),
        SamplingConfig(), leaf_max=b["leaf_max"])
    assert fac.levels == b["levels"] == 3
    assert fac.nnz == b["nnz"]
    x = golden_data.seeded_complex(b["seed"], nk).real
    assert rel(OA.idbf_apply(fac, x), ARR["bf_fwd"]) < 1e-15
    assert rel(OA.idbf_apply_transpose(fac, x), ARR["bf_inv"]) < 1e-15
    with pytest.raises(ValueError, match="against shape"):
        OA.idbf_apply(fac, np.zeros(nk - 1))


@pytest.mark.parametrize("n,m", [(32, 20), (64, 0), (64, 64), (64, 126),
                                 (128, 100)])
def test_oracle_alt_vs_dense(n, m):
    # pkg/tests/test_alt.py:27-46 bars
    plan = plan_alt(n, m, n0=16)
    rng = np.random.default_rng(n + m)
    beta = rng.standard_normal(2 * n - m)
    want = OD.dense_alt_forward(n, m, beta)
    assert rel(OA.alt_forward(plan, beta), want) < 1e-13
    f = rng.standard_normal(2 * n)
    want = OD.dense_alt_inverse(n, m, f)
    assert rel(OA.alt_inverse(plan, f), want) < 1e-13


@pytest.mark.parametrize("n", [4, 16])
def test_oracle_sht_vs_dense(n):
    plan = plan_sht(n)
    flat = golden_data.sht_flat(n, 5)
    assert rel(OA.sht_forward(plan.alt_plans, n, flat),
               OD.dense_sht_forward(n, flat)) < 1e-12
    vals = golden_data.sht_grid(n, 6)
    assert rel(OA.sht_inverse(plan.alt_plans, n, vals),
               OD.dense_sht_inverse(n, vals)) < 1e-12
