"""GPU batched paths over the wide (16 RHS per entry) engine:
  * idbf_apply / idbf_apply_transpose on one ButterflyFactorization
    (butterfly.py:275-292): 1-D, 2-D, complex, > 16 columns, error text;
  * alt_forward / alt_inverse on (2N-m, F) fields (SURVEY 8(b) extension,
    config 4) vs the oracle per field, and bitwise equal to the single-field
    SHT-path engine (each RHS column sums in the same order)."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt, plan_orders
from paper_2004_11346_b200.factors import FunctionOracle, idbf_factor

import golden_data
import oracle.apply as OA

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def dft_factor(nk, leaf_max):
    scale = 1.0 / np.sqrt(nk)
    return idbf_factor(FunctionOracle(
        lambda i, j: np.cos(2.0 * np.pi * i * j / nk) * scale, (nk, nk)),
        SamplingConfig(), leaf_max=leaf_max)


def test_idbf_apply_golden_factor():
    from paper_2004_11346_b200.api import idbf_apply, idbf_apply_transpose
    fac = dft_factor(128, 16)
    x = golden_data.seeded_complex(77, 128).real
    assert rel(idbf_apply(fac, x), OA.idbf_apply(fac, x)) < 1e-14
    assert rel(idbf_apply_transpose(fac, x), OA.idbf_apply_transpose(fac, x)) < 1e-14
    with pytest.raises(ValueError, match="length 127 against shape"):
        idbf_apply(fac, np.zeros(127))
    with pytest.raises(ValueError, match="against shape"):
        idbf_apply_transpose(fac, np.zeros((5, 2)))


@pytest.mark.parametrize("k,cplx", [(1, False), (7, False), (20, False), (9, True)])
def test_idbf_apply_2d(k, cplx):
    from paper_2004_11346_b200.api import idbf_apply, idbf_apply_transpose
    h, w = 300, 180
    fac = idbf_factor(FunctionOracle(
        lambda i, j: np.cos(0.37 * i * j / np.sqrt(h * w) * 40.0 + 0.1 * i), (h, w)),
        SamplingConfig(), leaf_max=24)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((w, k))
    y = rng.standard_normal((h, k))
    if cplx:
        x = x + 1j * rng.standard_normal((w, k))
        y = y + 1j * rng.standard_normal((h, k))
    gx = idbf_apply(fac, x)
    assert gx.shape == (h, k) and np.iscomplexobj(gx) == cplx
    assert rel(gx, OA.idbf_apply(fac, x)) < 1e-14
    assert rel(idbf_apply_transpose(fac, y), OA.idbf_apply_transpose(fac, y)) < 1e-14


@pytest.mark.parametrize("n,m,nf", [(64, 0, 3), (64, 5, 8), (128, 40, 13), (256, 300, 1),
                                       (128, 3, 40), (64, 1, 64)])
def test_alt_fields_vs_oracle(n, m, nf):
    from paper_2004_11346_b200.api import alt_forward, alt_inverse
    plan = plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=64)
    rng = np.random.default_rng(n + m + nf)
    beta = rng.standard_normal((2 * n - m, nf)) + 1j * rng.standard_normal((2 * n - m, nf))
    got = alt_forward(plan, beta).values
    assert got.shape == (2 * n, nf)
    for f in range(nf):
        want = OA.alt_forward(plan, beta[:, f])
        assert rel(got[:, f], want) < 1e-13
        # same bits as the single-field (4-RHS) engine
        assert np.array_equal(got[:, f], alt_forward(plan, beta[:, f]).values)
    back = alt_inverse(plan, got).values
    assert back.shape == (2 * n - m, nf)
    for f in range(nf):
        want = OA.alt_inverse(plan, got[:, f])
        assert rel(back[:, f], want) < 1e-13
        assert np.array_equal(back[:, f], alt_inverse(plan, got[:, f]).values)
    with pytest.raises(ValueError, match="coefficients, got shape"):
        alt_forward(plan, np.zeros((2 * n - m + 1, 2)))


def test_alt_fields_all_orders_device():
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    n, nf = 64, 11
    q = gauss_legendre(2 * n)
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12),
                        processes=0, quadrature=q)
    dp = DevicePlan(plans)
    rng = np.random.default_rng(5)
    blocks = [rng.standard_normal((2 * n - m, nf)) + 1j * rng.standard_normal((2 * n - m, nf))
              for m in range(2 * n)]
    out = dp.alt_fields(FORWARD, torch.from_numpy(np.concatenate(blocks)).cuda()).cpu().numpy()
    out = out.reshape(2 * n, 2 * n, nf)
    for m, (p, b) in enumerate(zip(plans, blocks)):
        for f in (0, nf - 1):
            assert rel(out[m][:, f], OA.alt_forward(p, b[:, f])) < 1e-13
    back = dp.alt_fields(INVERSE, torch.from_numpy(out.reshape(-1, nf)).cuda()).cpu().numpy()
    pos = 0
    for p, col in zip(plans, out):
        ln = 2 * n - p.m
        for f in (0, 5):
            assert rel(back[pos:pos + ln, f], OA.alt_inverse(p, col[:, f])) < 1e-13
        pos += ln
