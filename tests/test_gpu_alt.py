"""GPU parity: per-order ALT through the C ABI vs the CPU oracle."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt

import oracle.apply as OA

pytestmark = pytest.mark.gpu

CASES = [(32, [20], 16), (64, [0, 3, 64, 126, 127], 16),
         (128, [100, 0, 1], 16), (256, [0, 1, 300, 511], 512),
         (512, [0, 1, 100, 700, 1023], 512)]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("n,ms,n0", CASES)
def test_alt_orders_match_oracle(n, ms, n0):
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=n0,
                      quadrature=q) for m in ms]
    dp = DevicePlan(plans)
    rng = np.random.default_rng(n)
    vecs = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
            for m in ms]
    flat = torch.from_numpy(np.concatenate(vecs)).cuda()
    out = dp.alt_orders(FORWARD, flat).cpu().numpy().reshape(len(ms), 2 * n)
    for o, (p, v) in enumerate(zip(plans, vecs)):
        assert rel(out[o], OA.alt_forward(p, v)) < 1e-12
    fs = [rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)
          for _ in ms]
    back = dp.alt_orders(INVERSE, torch.from_numpy(np.concatenate(fs)).cuda())
    back = back.cpu().numpy()
    pos = 0
    for p, f in zip(plans, fs):
        ln = 2 * n - p.m
        assert rel(back[pos:pos + ln], OA.alt_inverse(p, f)) < 1e-12
        pos += ln
