"""Reference-facing API contract that does not need a GPU: argument checks
and messages (pkg/tests/test_alt.py:92-97, test_sht.py:28-48,130-137)."""
import numpy as np
import pytest

from paper_2004_11346_b200 import ShtCoeffs, make_grid, plan_alt, plan_sht
from paper_2004_11346_b200 import api


def test_alt_shape_validation():
    plan = plan_alt(16, 2, n0=8)
    with pytest.raises(ValueError, match="expected 30 coefficients"):
        api.alt_forward(plan, np.zeros(29))
    with pytest.raises(ValueError, match="expected 32 node values"):
        api.alt_inverse(plan, np.zeros(31))


def test_sht_size_validation():
    plan = plan_sht(4)
    with pytest.raises(ValueError, match="plan N=4"):
        api.sht_forward(plan, ShtCoeffs.zeros(5))
    with pytest.raises(ValueError, match="expected grid shape"):
        api.sht_inverse(plan, np.zeros((8, 14), dtype=np.complex128))


def test_coeffs_container():
    c = ShtCoeffs.zeros(4)
    assert len(c.by_m) == 15
    assert c[0].shape == (8,) and c[7].shape == (1,) and c[-7].shape == (1,)
    c[3] = np.arange(5)
    assert np.array_equal(c[3], np.arange(5).astype(np.complex128))
    with pytest.raises(IndexError, match="outside band limit"):
        c[8]
    with pytest.raises(ValueError, match="expects"):
        c[2] = np.zeros(3)
    flat = c.pack()
    back = ShtCoeffs.unpack(4, flat)
    for m in range(-7, 8):
        assert np.array_equal(back[m], c[m])
    with pytest.raises(ValueError):
        ShtCoeffs.unpack(4, flat[:-1])


def test_grid_conventions():
    grid = make_grid(8)
    assert grid.thetas.shape == (16,) and grid.phis.shape == (31,)
    assert np.all(np.diff(grid.thetas) < 0)
    assert grid.phis[0] == pytest.approx(np.pi / 31)


def test_plan_shares_quadrature():
    plan = plan_sht(8)
    assert len(plan.alt_plans) == 16
    for p in plan.alt_plans:
        assert p.quadrature is plan.alt_plans[0].quadrature
