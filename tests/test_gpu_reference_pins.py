"""GPU mirrors of the reference's own apply-path pins.

Each test restates one reference test on the CUDA path (through the C ABI
behind api.sht_forward / api.alt_forward):

* pkg/tests/test_sht.py:82-90   constant mode  beta_{0,0}=2 -> sqrt(2)
* pkg/tests/test_sht.py:93-105  single mode    Pbar_5^3(cos t) e^{3 i phi}
* pkg/tests/test_sht.py:108-117 Parseval on the 2N-node x (4N-1) grid
* pkg/tests/test_alt.py:70-78   complex = re + i im, bitwise
* pkg/tests/test_sht.py:51-68   forward / inverse vs the dense transform
"""
import math

import numpy as np
import pytest

from paper_2004_11346_b200 import (ShtCoeffs, legendre_table, make_grid,
                                   plan_alt, plan_sht)

import oracle.dense as OD

pytestmark = pytest.mark.gpu


def random_coeffs(n, seed):
    rng = np.random.default_rng(seed)
    coeffs = ShtCoeffs.zeros(n)
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        coeffs[m] = rng.standard_normal(ln) + 1j * rng.standard_normal(ln)
    return coeffs


def test_constant_mode():
    from paper_2004_11346_b200.api import sht_forward
    n = 8
    coeffs = ShtCoeffs.zeros(n)
    coeffs[0] = np.r_[2.0, np.zeros(2 * n - 1)]
    got = sht_forward(plan_sht(n), coeffs).values
    np.testing.assert_allclose(got, np.sqrt(2.0) + 0j, atol=1e-10)


def _pbar_closed_form(k, m, x):
    # independent of the recurrence: sqrt((2k+1)/2 (k-m)!/(k+m)!) P_k^m(x),
    # P_k^m without the Condon-Shortley phase (the reference convention,
    # checked against legendre_table below)
    from scipy.special import lpmv
    norm = math.sqrt((2 * k + 1) / 2 * math.factorial(k - m) / math.factorial(k + m))
    return norm * lpmv(m, k, x) * (-1) ** m


def test_single_mode():
    from paper_2004_11346_b200.api import sht_forward
    n = 8
    k, m = 5, 3
    coeffs = ShtCoeffs.zeros(n)
    vec = np.zeros(2 * n - m, dtype=np.complex128)
    vec[k - m] = 1.0
    coeffs[m] = vec
    got = sht_forward(plan_sht(n), coeffs).values
    grid = make_grid(n)
    pk = legendre_table(m, np.cos(grid.thetas), np.array([k]))[:, 0]
    np.testing.assert_allclose(pk, _pbar_closed_form(k, m, np.cos(grid.thetas)),
                               atol=1e-13)
    want = pk[:, None] * np.exp(1j * m * grid.phis)[None, :]
    np.testing.assert_allclose(got, want, atol=1e-10)


def test_parseval():
    from paper_2004_11346_b200.api import sht_forward
    n = 16
    coeffs = random_coeffs(n, 9)
    plan = plan_sht(n)
    f = sht_forward(plan, coeffs).values
    w = plan.quadrature.weights
    grid_energy = float(np.sum(w[:, None] * np.abs(f) ** 2)) / (4 * n - 1)
    coeff_energy = float(np.sum(np.abs(coeffs.pack()) ** 2))
    assert grid_energy == pytest.approx(coeff_energy, rel=1e-12)


@pytest.mark.parametrize("n,m", [(32, 9), (32, 0), (256, 3), (256, 511)])
def test_complex_coefficients_split(n, m):
    from paper_2004_11346_b200.api import alt_forward, alt_inverse
    plan = plan_alt(n, m, n0=16 if n == 32 else 512)
    rng = np.random.default_rng(4)
    ln = 2 * n - m
    beta = rng.standard_normal(ln) + 1j * rng.standard_normal(ln)
    got = alt_forward(plan, beta).values
    want = (alt_forward(plan, beta.real).values
            + 1j * alt_forward(plan, beta.imag).values)
    assert np.array_equal(got, want)
    assert got.dtype == np.complex128
    f = rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)
    got = alt_inverse(plan, f).values
    want = (alt_inverse(plan, f.real).values
            + 1j * alt_inverse(plan, f.imag).values)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [4, 16])
def test_inverse_matches_dense(n):
    from paper_2004_11346_b200.api import sht_inverse
    rng = np.random.default_rng(100 + n)
    values = (rng.standard_normal((2 * n, 4 * n - 1))
              + 1j * rng.standard_normal((2 * n, 4 * n - 1)))
    got = sht_inverse(plan_sht(n), values).pack()
    want = OD.dense_sht_inverse(n, values)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12
