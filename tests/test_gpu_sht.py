"""GPU parity: full SHT and the batched odd-length DFT vs the CPU oracle."""
import numpy as np
import pytest

from paper_2004_11346_b200 import ShtCoeffs, plan_sht

import oracle.apply as OA
import oracle.dense as OD

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def random_flat(n, seed, decay=0):
    rng = np.random.default_rng(seed)
    out = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        k = np.arange(abs(m), 2 * n)
        out.append((rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
                   * (1.0 + k) ** (-decay))
    return np.concatenate(out)


@pytest.mark.parametrize("L", [15, 31, 63, 127, 255, 1023, 4095,
                               # prime factor > 255: Bluestein rows
                               263, 1021, 8191, 3 * 257, 2 * 4099])
def test_dft_rows_match_numpy(L):
    import torch
    from paper_2004_11346_b200.api import dft_rows
    rng = np.random.default_rng(L)
    x = rng.standard_normal((7, L)) + 1j * rng.standard_normal((7, L))
    xt = torch.from_numpy(x).cuda()
    got = dft_rows(xt).cpu().numpy()
    assert rel(got, np.fft.fft(x, axis=1)) < 2e-14
    got = dft_rows(xt, inverse=True).cpu().numpy()
    assert rel(got, L * np.fft.ifft(x, axis=1)) < 2e-14


@pytest.mark.parametrize("L,above", [(4095, 12), (255, 4), (15, 2), (1024, 3)])
def test_dft_rows_forced_bluestein(L, above, monkeypatch):
    # BFSHT_BLUESTEIN_ABOVE lowers the Bluestein threshold: the same lengths
    # through the chirp-z path (smem rows and, for 4095 -> M = 8192, 2 rows
    # of 128 KB: global scratch)
    monkeypatch.setenv("BFSHT_BLUESTEIN_ABOVE", str(above))
    test_dft_rows_match_numpy(L)


@pytest.mark.parametrize("n", [4, 8, 16, 32, 66])
def test_sht_matches_oracle_and_dense(n):
    from paper_2004_11346_b200.api import sht_forward, sht_inverse
    plan = plan_sht(n)
    flat = random_flat(n, n)
    coeffs = ShtCoeffs.unpack(n, flat)
    got = sht_forward(plan, coeffs).values
    want = OA.sht_forward(plan.alt_plans, n, flat)
    assert rel(got, want) < 1e-12
    assert rel(got, OD.dense_sht_forward(n, flat)) < 1e-12
    back = sht_inverse(plan, got).pack()
    assert rel(back, OA.sht_inverse(plan.alt_plans, n, got)) < 1e-12
    assert rel(back, flat) < 1e-12


@pytest.mark.parametrize("n", [16, 64])
def test_real_grid_inverse_tol_1e10(n):
    # config C5 semantics: a real grid (iid U(-1,1)) into sht_inverse is
    # promoted to complex (sht.py:151-166); plans at tolerance 1e-10 (C3/C5)
    from paper_2004_11346_b200 import SamplingConfig
    from paper_2004_11346_b200.api import sht_inverse
    plan = plan_sht(n, SamplingConfig(tolerance=1e-10))
    rng = np.random.default_rng(n)
    grid = rng.uniform(-1.0, 1.0, (2 * n, 4 * n - 1))
    got = sht_inverse(plan, grid).pack()
    want = OA.sht_inverse(plan.alt_plans, n, grid.astype(np.complex128))
    assert rel(got, want) < 1e-12
    # (1+k)^-2 spectrum forward (C5 forward input) round trip
    flat = random_flat(n, n + 1, decay=2)
    from paper_2004_11346_b200.api import sht_forward
    g = sht_forward(plan, ShtCoeffs.unpack(n, flat)).values
    assert rel(g, OA.sht_forward(plan.alt_plans, n, flat)) < 1e-12


@pytest.mark.parametrize("n,batch", [(16, 1), (32, 3), (64, 4)])
def test_sht_batch_bitwise(n, batch):
    # batched transforms on the 16-RHS engine == single-transform calls
    import torch
    from paper_2004_11346_b200.api import ShtDevice
    dev = ShtDevice(plan_sht(n))
    flats = np.stack([random_flat(n, 10 * n + b) for b in range(batch)])
    c = torch.from_numpy(flats).cuda()
    g = dev.forward_batch(c)
    back = dev.inverse_batch(g)
    for b in range(batch):
        gs = dev.forward(c[b])
        assert torch.equal(g[b], gs)
        assert torch.equal(back[b], dev.inverse(gs))
    assert rel(back.cpu().numpy(), flats) < 1e-11


def test_plan_reuse_after_smaller_length():
    # the DFT kernels' dynamic shared-memory limit is per kernel: a small-L
    # plan (or a standalone dft_rows call) in between must not break a later
    # launch of a large-L plan (the limit used to be lowered)
    import torch
    from paper_2004_11346_b200 import SamplingConfig, plan_orders
    from paper_2004_11346_b200.api import DevicePlan, dft_rows
    n = 1024
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
    big = DevicePlan(plans, weights=plans[0].quadrature.weights)
    c = torch.from_numpy(random_flat(n, 5)).cuda()
    g1 = big.sht_forward(c)
    small = DevicePlan(plan_sht(64).alt_plans, weights=plan_sht(64).quadrature.weights)
    small.sht_forward(torch.from_numpy(random_flat(64, 6)).cuda())
    dft_rows(torch.zeros((3, 15), dtype=torch.complex128, device="cuda"))
    g2 = big.sht_forward(c)
    torch.cuda.synchronize()
    assert torch.equal(g1, g2)
    assert torch.equal(big.sht_inverse(g1), big.sht_inverse(g2))
