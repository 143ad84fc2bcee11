"""GPU: the chunked (out-of-core) SHT on one GPU vs the CPU oracle.

ChunkedSht plans / packs / applies the orders chunk by chunk and runs the
φ DFT once over a θ-major buffer holding every order (paper_2004_11346_b200/
ooc.py) — the path the full N=4096 transform (BASELINE config 3) takes on
one B200.  Here at sizes the oracle finishes in seconds, with chunks that
are dropped after the forward (re-planned for the inverse) and chunks that
stay resident.
"""
import numpy as np
import pytest

import oracle.apply as OA

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def random_flat(n, seed):
    rng = np.random.default_rng(seed)
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        k = np.arange(abs(m), 2 * n)
        parts.append((rng.standard_normal(ln) + 1j * rng.standard_normal(ln)) / (1.0 + k))
    return np.concatenate(parts)


@pytest.mark.parametrize("n,chunks,reserve", [(16, 3, 1 << 50), (32, 5, 0)])
def test_chunked_sht_matches_oracle(n, chunks, reserve):
    import torch
    from paper_2004_11346_b200 import plan_orders
    from paper_2004_11346_b200.ooc import ChunkedSht

    run = ChunkedSht(n, chunks, n0=16, processes=1, reserve_bytes=reserve)
    plans = plan_orders(n, range(2 * n), n0=16, processes=1)
    flat = random_flat(n, n)
    grid = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128, device="cuda")
    fwd = run.forward(flat, grid)
    got = grid.cpu().numpy()
    want = OA.sht_forward(plans, n, flat)
    assert rel(got, want) < 1e-12
    inv = run.inverse(grid)
    want_b = OA.sht_inverse(plans, n, got)
    assert rel(inv["coeffs"], want_b) < 1e-12
    assert rel(inv["coeffs"], flat) < 1e-11
    # re-planned chunks give the same numbers as resident ones
    assert inv["replanned"] == (len(run.chunks) if reserve > (1 << 40) else 0)
    assert fwd["device_ms"] > 0 and inv["alt_ms"] > 0
    # θ-major node entries of a sampled order assemble to its ALT output
    m = n // 2
    fwd2 = run.forward(flat, grid)
    e = run.node_entries(m)
    g_o, g_e = e[0], e[1]            # parity 0 = odd degrees, 1 = even
    plus = np.concatenate([(g_e - g_o)[::-1], g_e + g_o])
    s = OA.coeff_offsets(n)[1][(2 * n - 1) + m]
    want_col = OA.alt_forward(plans[m], flat[s:s + 2 * n - m])
    assert rel(plus[:, 0] + 1j * plus[:, 1], want_col) < 1e-12
    assert fwd2["alt_bytes"] == fwd["alt_bytes"]
    run.close()


@pytest.mark.parametrize("L", [16383, 32767])
def test_dft_rows_large_prime_radices(L):
    # the N=4096 / N=8192 row lengths (4N-1 = 3 * 43 * 127 / 7 * 31 * 151)
    # do not fit the shared-memory DFT path (the global-scratch variant runs)
    # and have prime radices above 13 (the cooperative generic pass)
    import torch
    from paper_2004_11346_b200.api import dft_rows
    rng = np.random.default_rng(L)
    x = rng.standard_normal((5, L)) + 1j * rng.standard_normal((5, L))
    xt = torch.from_numpy(x).cuda()
    assert rel(dft_rows(xt).cpu().numpy(), np.fft.fft(x, axis=1)) < 1e-14
    assert rel(dft_rows(xt, inverse=True).cpu().numpy(), L * np.fft.ifft(x, axis=1)) < 1e-14


def test_chunked_sht_subset_of_chunks():
    # a chunk subset (the sampled N=8192 run's mode): coefficients on those
    # orders only; the full-size DFT stage sees zeros elsewhere
    import torch
    from paper_2004_11346_b200 import plan_orders
    from paper_2004_11346_b200.ooc import ChunkedSht

    n = 16
    run = ChunkedSht(n, 4, n0=16, processes=1, only=[2])
    plans = plan_orders(n, range(2 * n), n0=16, processes=1)
    sub = set(run.chunks[2])
    flat = random_flat(n, 3)
    _, offs = OA.coeff_offsets(n)
    for i, m in enumerate(range(-(2 * n - 1), 2 * n)):
        if abs(m) not in sub:
            flat[offs[i]:offs[i + 1]] = 0.0
    grid = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128, device="cuda")
    run.forward(flat, grid)
    got = grid.cpu().numpy()
    want = OA.sht_forward(plans, n, flat)
    assert rel(got, want) < 1e-12
    back = run.inverse(grid)["coeffs"]
    want_b = OA.sht_inverse(plans, n, got)
    sel = np.concatenate([np.arange(offs[i], offs[i + 1])
                          for i, m in enumerate(range(-(2 * n - 1), 2 * n)) if abs(m) in sub])
    assert rel(back[sel], want_b[sel]) < 1e-12
    run.close()
