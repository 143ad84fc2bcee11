"""On-GPU regeneration of dense turning tiles: ALT and SHT
results with regenerated tiles are bitwise equal to the stored-tile engine
(the regenerated values are the stored ones), on the 4-RHS and the
16-RHS (batched fields) engines."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_orders, plan_sht

import oracle.apply as OA

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,frac", [(256, 1.0), (256, 0.3), (512, 0.5)])
def test_alt_orders_bitwise_with_regen(n, frac):
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    q = gauss_legendre(2 * n)
    orders = list(range(0, 2 * n, 7)) + [2 * n - 1]
    plans = plan_orders(n, orders, SamplingConfig(tolerance=1e-12), processes=0, quadrature=q)
    base = DevicePlan(plans)
    dp = DevicePlan(plans, regen=frac)
    assert dp.packed.regen_tiles > 0
    rng = np.random.default_rng(n)
    vec = np.concatenate([rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
                          for m in orders])
    x = torch.from_numpy(vec).cuda()
    a = dp.alt_orders(FORWARD, x).cpu().numpy()
    b = base.alt_orders(FORWARD, x).cpu().numpy()
    assert np.array_equal(a, b)
    want = OA.alt_forward(plans[3], vec[sum(2 * n - m for m in orders[:3]):][:2 * n - orders[3]])
    assert np.linalg.norm(a[3 * 2 * n:4 * 2 * n] - want) <= 1e-12 * np.linalg.norm(want)
    g = torch.from_numpy(a).cuda()
    assert np.array_equal(dp.alt_orders(INVERSE, g).cpu().numpy(),
                          base.alt_orders(INVERSE, g).cpu().numpy())
    # batched fields through the wide engine
    f = torch.from_numpy(np.stack([vec, 2 * vec, vec.conj()], 1)).cuda()
    assert np.array_equal(dp.alt_fields(FORWARD, f).cpu().numpy(),
                          base.alt_fields(FORWARD, f).cpu().numpy())


def test_sht_bitwise_with_regen():
    import torch
    from paper_2004_11346_b200.api import DevicePlan
    n = 128
    plan = plan_sht(n)
    base = DevicePlan(plan.alt_plans, weights=plan.quadrature.weights)
    dp = DevicePlan(plan.alt_plans, weights=plan.quadrature.weights, regen=1.0)
    assert dp.packed.regen_tiles > 0
    rng = np.random.default_rng(1)
    c = torch.from_numpy(rng.standard_normal(4 * n * n) + 1j * rng.standard_normal(4 * n * n)).cuda()
    ga, gb = dp.sht_forward(c), base.sht_forward(c)
    assert torch.equal(ga, gb)
    assert torch.equal(dp.sht_inverse(ga), base.sht_inverse(gb))
