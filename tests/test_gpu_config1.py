"""BASELINE config C1 on the GPU: forward ALT at N=256 for every order
m = 0..511, coefficients iid N(0,1) (seeded), IDBF tolerance 1e-12, default
n0 = 512; compared with the reference apply (oracle, <= 1e-12) and with the
dense ALT (no worse than the reference's own error, SURVEY hard part 7).
Also the inverse for every order (weighted transpose, alt.py:239-253).
"""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_orders

import oracle.apply as OA
import oracle.dense as OD

pytestmark = pytest.mark.gpu


def test_config1_all_orders_n256():
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    n = 256
    q = gauss_legendre(2 * n)
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12),
                        processes=0, quadrature=q)
    dp = DevicePlan(plans)
    rng = np.random.default_rng(256)
    vecs = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
            for m in range(2 * n)]
    out = dp.alt_orders(FORWARD, torch.from_numpy(np.concatenate(vecs)).cuda())
    out = out.cpu().numpy().reshape(2 * n, 2 * n)
    worst_oracle, worst_excess = 0.0, 0.0
    for m, (p, v) in enumerate(zip(plans, vecs)):
        want = OA.alt_forward(p, v)
        e_or = np.linalg.norm(out[m] - want) / np.linalg.norm(want)
        dense = OD.dense_alt_forward(n, m, v, q)
        e_gpu = np.linalg.norm(out[m] - dense) / np.linalg.norm(dense)
        e_ref = np.linalg.norm(want - dense) / np.linalg.norm(dense)
        worst_oracle = max(worst_oracle, e_or)
        worst_excess = max(worst_excess, e_gpu - (e_ref * (1 + 1e-3) + 1e-14))
    assert worst_oracle < 1e-12
    assert worst_excess <= 0.0
    back = dp.alt_orders(INVERSE, torch.from_numpy(out.reshape(-1)).cuda()).cpu().numpy()
    pos = 0
    for p, col in zip(plans, out):
        ln = 2 * n - p.m
        want = OA.alt_inverse(p, col)
        assert np.linalg.norm(back[pos:pos + ln] - want) <= 1e-12 * np.linalg.norm(want)
        pos += ln
