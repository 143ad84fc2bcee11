"""GPU: the SHT's DFT stage at lengths whose rows do not fit one CTA's
shared memory — N=4096 (L = 16383 = 3 * 43 * 127, direct mixed radix with
the generic prime passes) and N=2048 (L = 8191, prime: Bluestein rows of
length M = 16384) — vs numpy.

Synthesis: random θ-major node halves for every order -> grid rows,
checked against a numpy restatement of sht.py:137-148 on the same node
halves.  Analysis: a random grid -> weighted folds of its spectrum,
checked against numpy's FFT of the same rows (sht.py:151-166, alt.py:239-253).
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n", [4096, 2048, 66])
def test_synthesis_and_analysis_rows(n):
    import torch
    from paper_2004_11346_b200.ooc import ChunkedSht

    L = 4 * n - 1
    run = ChunkedSht(n, min(48, n), processes=1, only=[])
    lib, st = run.lib, run._stream()
    rng = np.random.default_rng(7)
    yb = rng.standard_normal(tuple(run.ybuf.shape))
    run.ybuf.copy_(torch.from_numpy(yb))
    grid = torch.empty((2 * n, L), dtype=torch.complex128, device="cuda")
    assert lib.bfsht_synth_rows(run.ctx.handle, _ptr(run.layout_dev), _ptr(run.ybuf), 0, n,
                                _ptr(grid), st) == 0
    torch.cuda.synchronize()
    lay = run.layout
    ms = np.arange(2 * n)
    phi0 = np.pi / L
    for r in sorted({0, min(1234, n // 2), n - 1}):
        ent = np.zeros((2, 2 * n, 4))
        for par in range(2):
            h = lay[2 * ms + par]
            ok = h["ncols"] > 0
            ent[par][ok] = yb[h["y"][ok].astype(np.int64) + r * h["x"][ok].astype(np.int64)]
        go, ge = ent[0], ent[1]
        for row, v in ((n + r, ge + go), (n - 1 - r, ge - go)):
            spec = np.zeros(L, dtype=np.complex128)
            spec[ms] = (v[:, 0] + 1j * v[:, 1]) * np.exp(1j * ms * phi0)
            spec[L - ms[1:]] = (v[1:, 2] + 1j * v[1:, 3]) * np.exp(-1j * ms[1:] * phi0)
            want = L * np.fft.ifft(spec)
            got = grid[row].cpu().numpy()
            assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)

    g = rng.standard_normal((2 * n, L)) + 1j * rng.standard_normal((2 * n, L))
    gd = torch.from_numpy(g).cuda()
    assert lib.bfsht_anal_rows(run.ctx.handle, _ptr(run.layout_dev), _ptr(run.ybuf), 0, n,
                               _ptr(gd), _ptr(run.weights), st) == 0
    torch.cuda.synchronize()
    w = run.quadrature.weights
    for m in sorted({0, 5, min(3000, n), 2 * n - 1}):
        e = run.node_entries(m)
        for r in sorted({0, min(777, n // 3), n - 1}):
            up = np.fft.fft(g[n + r]) / L
            lo = np.fft.fft(g[n - 1 - r]) / L
            for sgn, cols in ((1, (0, 1)), (-1, (2, 3))):
                if m == 0 and sgn < 0:
                    continue
                b = (sgn * m) % L
                t = np.exp(-1j * sgn * m * phi0)
                a, c = up[b] * t, lo[b] * t
                for par, want in ((0, w[n + r] * (a - c)), (1, w[n + r] * (a + c))):
                    if lay[2 * m + par]["ncols"] <= 0:
                        continue
                    got = e[par][r, cols[0]] + 1j * e[par][r, cols[1]]
                    assert abs(got - want) <= 1e-12 * (abs(want) + 1e-3 * w[n + r])
    run.close()
