"""End-to-end parity at the headline configuration (BASELINE C2).

The final engine's whole-transform path — coef_pack -> every ALT stage ->
fused synthesis / phi-DFT, and the reverse — at N=1024 (2048 x 4095 grid,
tol 1e-12, the bench's own seeded (1+k)^-1 input) against the CPU oracle
(oracle/apply.py: the reference's sht_forward / sht_inverse,
pkg/src/bfsht/sht.py:137-166, with numpy's pocketfft) on the same factors.
Bar (north_star): <= 1e-12 relative l2, globally and per order.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 1024


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def c2():
    from paper_2004_11346_b200 import SamplingConfig, plan_orders
    from bench import synthetic_coeffs
    plans = plan_orders(N, range(2 * N), SamplingConfig(tolerance=1e-12),
                        processes=os.cpu_count() or 1)
    return plans, synthetic_coeffs(N)


def test_c2_forward_and_inverse_match_oracle(c2):
    import torch
    import oracle.apply as OA
    from paper_2004_11346_b200.api import DevicePlan
    plans, flat = c2
    dp = DevicePlan(plans, weights=plans[0].quadrature.weights)
    grid = dp.sht_forward(torch.from_numpy(flat).cuda()).cpu().numpy()
    want = OA.sht_forward(plans, N, flat)
    assert rel(grid, want) <= 1e-12
    # every colatitude row on its own
    row_err = np.linalg.norm(grid - want, axis=1) / np.linalg.norm(want, axis=1)
    assert row_err.max() <= 1e-12, row_err.max()
    # inverse of the oracle's grid (the GPU's grid would hide a DFT error)
    back = dp.sht_inverse(torch.from_numpy(want).cuda()).cpu().numpy()
    back_want = OA.sht_inverse(plans, N, want)
    assert rel(back, back_want) <= 1e-12
    ms, offs = OA.coeff_offsets(N)
    worst = max(rel(back[offs[i]:offs[i + 1]], back_want[offs[i]:offs[i + 1]])
                for i in range(len(ms)))
    assert worst <= 1e-12, worst
    # round trip at the reference's accuracy for this plan (SURVEY: 9.5e-12)
    assert rel(back_want, flat) < 2e-11
    assert rel(dp.sht_inverse(torch.from_numpy(grid).cuda()).cpu().numpy(), flat) < 2e-11
