"""Chunked (out-of-core) SHT host logic on CPU.

ChunkedSht (paper_2004_11346_b200/ooc.py) runs the full transform on one GPU
chunk by chunk: per chunk of orders pack, ALT, copy the chunk's forward
node array into a θ-major buffer (chunk_layout), and, for the inverse,
scatter that buffer's block back to the chunk's node halves
(scatter_index).  Here the same layout and index code drives the numpy
interpreter of the packed format (packed_emulator) and a numpy DFT stage
that addresses entries exactly like the row-path kernels; the result must
match the CPU oracle's whole-plan transform.
"""
import numpy as np
import pytest

import packed_emulator as EMU


def _flat(n, seed):
    rng = np.random.default_rng(seed)
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        parts.append(rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
    return np.concatenate(parts)


def _entry(layout, ybuf, m, par, r):
    hf = layout[2 * m + par]
    return ybuf[hf["y"] + r * hf["x"]] if hf["ncols"] else np.zeros(4)


@pytest.mark.parametrize("n,nchunks", [(8, 3), (16, 5)])
def test_chunked_layout_roundtrip_matches_oracle(n, nchunks):
    import oracle.apply as OA
    from paper_2004_11346_b200 import gauss_legendre, plan_orders, plan_sht
    from paper_2004_11346_b200.dist import _flat_offset
    from paper_2004_11346_b200.ooc import chunk_layout, scatter_index
    from paper_2004_11346_b200.pack import pack_plans

    L = 4 * n - 1
    q = gauss_legendre(2 * n)
    chunks, layout, blocks, entries = chunk_layout(n, nchunks)
    assert sorted(m for c in chunks for m in c) == list(range(2 * n))
    assert entries == 4 * n * n
    assert blocks[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    flat = _flat(n, 5)
    full = plan_sht(n, n0=8)
    want_grid = OA.sht_forward(full.alt_plans, n, flat)
    want_back = OA.sht_inverse(full.alt_plans, n, want_grid)

    packed = []
    ybuf = np.zeros((entries, 4))
    for c, orders in enumerate(chunks):
        pk = pack_plans(plan_orders(n, orders, n0=8, processes=1, quadrature=q))
        packed.append(pk)
        arena = np.zeros((pk.stats["arena"], 4))
        for o, m in enumerate(orders):
            cp = flat[_flat_offset(n, m):_flat_offset(n, m) + 2 * n - m]
            cm = flat[_flat_offset(n, -m):_flat_offset(n, -m) + 2 * n - m] if m \
                else np.zeros(2 * n)
            for par in range(2):
                hf = pk.halves[2 * o + par]
                if hf["ncols"]:
                    k = slice(1 if par == 0 else 0, None, 2)
                    a, b = cp[k][:hf["ncols"]], cm[k][:hf["ncols"]]
                    arena[hf["x"]:hf["x"] + hf["ncols"]] = np.stack(
                        [a.real, a.imag, b.real, b.imag], 1)
        EMU.run_direction(pk, arena, 0)
        yr = int(pk.info[10])
        pos, cnt = blocks[c]
        ybuf[pos:pos + cnt] = arena[yr:yr + cnt]     # the one-memcpy move

    # synthesis over all row pairs through the layout
    phi0 = np.pi / L
    grid = np.zeros((2 * n, L), dtype=np.complex128)
    for r in range(n):
        up = np.zeros(L, complex)
        lo = np.zeros(L, complex)
        for b in range(L):
            m = b if b <= 2 * n - 1 else b - L
            sel = 0 if m >= 0 else 2
            g = [complex(*_entry(layout, ybuf, abs(m), par, r)[sel:sel + 2]) for par in range(2)]
            t = np.exp(1j * m * phi0)
            up[b] = (g[1] + g[0]) * t
            lo[b] = (g[1] - g[0]) * t
        grid[n + r] = L * np.fft.ifft(up)
        grid[n - 1 - r] = L * np.fft.ifft(lo)
    assert np.linalg.norm(grid - want_grid) <= 1e-13 * np.linalg.norm(want_grid)

    # analysis into the θ-major buffer, then per chunk scatter + ALT^T
    ybuf[:] = 0.0
    w = q.weights
    for r in range(n):
        su = np.fft.fft(want_grid[n + r]) / L
        sl = np.fft.fft(want_grid[n - 1 - r]) / L
        for b in range(L):
            m = b if b <= 2 * n - 1 else b - L
            sel = 0 if m >= 0 else 2
            t = np.exp(-1j * m * phi0)
            a, c = su[b] * t, sl[b] * t
            for par, v in ((0, w[n + r] * (a - c)), (1, w[n + r] * (a + c))):
                hf = layout[2 * abs(m) + par]
                if hf["ncols"]:
                    ybuf[hf["y"] + r * hf["x"], sel:sel + 2] = (v.real, v.imag)
    for c, orders in enumerate(chunks):
        pk = packed[c]
        idx = scatter_index(pk.halves, n)
        pos, cnt = blocks[c]
        assert idx.size == cnt
        arena = np.zeros((pk.stats["arena"], 4))
        keep = idx >= 0
        arena[idx[keep]] = ybuf[pos:pos + cnt][keep]
        EMU.run_direction(pk, arena, 1)
        for o, m in enumerate(orders):
            for sign in ((1, -1) if m else (1,)):
                got = np.zeros(2 * n - m, complex)
                sel = 0 if sign > 0 else 2
                for par in range(2):
                    hf = pk.halves[2 * o + par]
                    if hf["ncols"]:
                        e = arena[hf["x"]:hf["x"] + hf["ncols"]]
                        got[(1 if par == 0 else 0)::2] = e[:, sel] + 1j * e[:, sel + 1]
                s = _flat_offset(n, sign * m)
                ref = want_back[s:s + 2 * n - m]
                assert np.linalg.norm(got - ref) <= 1e-12 * max(np.linalg.norm(ref), 1e-300)
