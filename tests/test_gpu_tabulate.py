"""Device-side entry evaluation for factor construction:
bfsht_half_table_device must reproduce the host recurrence table bit for
bit, and plans built from it must keep the reference plan digests."""
import numpy as np
import pytest

import golden_data
from plan_digest import plan_digest
from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt, plan_orders
from paper_2004_11346_b200.legendre import half_table

pytestmark = pytest.mark.gpu

META, ARR = golden_data.load()


@pytest.mark.parametrize("n,m,offset", [(8, 0, 0), (64, 0, 1), (64, 37, 0), (1024, 0, 0),
                                        (1024, 700, 1), (1024, 2047, 0), (4096, 0, 1),
                                        (4096, 5000, 0), (4096, 8191, 0)])
def test_device_table_is_host_table(n, m, offset):
    q = gauss_legendre(2 * n)
    half = (m + 1) // 2 if offset else m // 2
    ncols = n - half
    if ncols < 1:
        pytest.skip("absent half")
    x = q.nodes[n:]
    host = half_table(m, offset, x, ncols)
    dev = half_table(m, offset, x, ncols, device=0)
    assert dev.shape == host.shape
    assert np.array_equal(dev.view(np.uint64), host.view(np.uint64))


@pytest.mark.parametrize("case", META["alt"][:8], ids=lambda c: f"n{c['n']}m{c['m']}")
def test_device_tabulated_plan_keeps_reference_digest(case):
    n, m = case["n"], case["m"]
    plan = plan_alt(n, m, SamplingConfig(tolerance=case["tol"]), n0=case["n0"],
                    quadrature=gauss_legendre(2 * n), device=0)
    assert plan.stats["total_nnz"] == case["total_nnz"]
    assert plan_digest(plan) == case["digest"]


def test_device_tabulated_processes_match_host():
    n = 32
    host = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), n0=16, processes=1)
    dev = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), n0=16, processes=3,
                      device=0)
    assert [plan_digest(p) for p in host] == [plan_digest(p) for p in dev]
