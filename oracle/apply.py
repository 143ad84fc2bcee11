"""Restated reference apply path (CPU, numpy/scipy) — TEST INFRASTRUCTURE.

Follows, operation for operation:
  idbf_apply / idbf_apply_transpose   pkg/src/bfsht/butterfly.py:275-292
  LowRankFactor.apply(_transpose)     pkg/src/bfsht/lowrank.py:196-202
  _apply_half / _apply_half_transpose pkg/src/bfsht/alt.py:197-222
  _forward_real / _inverse_real       pkg/src/bfsht/alt.py:225-253
  _dispatch, alt_forward/alt_inverse  pkg/src/bfsht/alt.py:256-282
  _bins, sht_forward / sht_inverse    pkg/src/bfsht/sht.py:131-166
The butterfly factors are applied as scipy CSR matvecs exactly as the
reference does, so on identical plans the oracle reproduces the reference
outputs bitwise (pinned in tests/test_oracle_golden.py).  Plans are duck
typed on the reference attribute names, so reference AltPlans and this
package's AltPlans both work.
"""
import numpy as np
import scipy.sparse


def _csr(f):
    c = getattr(f, "_oracle_csr", None)
    if c is None:
        c = scipy.sparse.csr_matrix((f.vals, (f.rows, f.cols)), shape=f.shape)
        try:
            f._oracle_csr = c
        except AttributeError:
            pass
    return c


def idbf_apply(fac, x):
    """y = K x through the factor chain (butterfly.py:275-282)."""
    x = np.asarray(x)
    if x.shape[0] != fac.shape[1]:
        raise ValueError(f"length {x.shape[0]} against shape {fac.shape}")
    for f in fac.factors:
        x = _csr(f) @ x
    return x


def idbf_apply_transpose(fac, y):
    """x = K^T y through the reversed chain (butterfly.py:285-292)."""
    y = np.asarray(y)
    if y.shape[0] != fac.shape[0]:
        raise ValueError(f"length {y.shape[0]} against shape {fac.shape}")
    for f in reversed(fac.factors):
        y = _csr(f).T @ y
    return y


def _lr_apply(p, x):
    return p.u @ (p.s[:, None] * (p.v.T @ x) if x.ndim > 1
                  else p.s * (p.v.T @ x))


def _lr_apply_t(p, x):
    return p.v @ (p.s[:, None] * (p.u.T @ x) if x.ndim > 1
                  else p.s * (p.u.T @ x))


def apply_half(blocks, vec, n_out):
    """Sum of block payload applies (alt.py:197-208)."""
    out = np.zeros(n_out)
    for blk in blocks:
        r0, r1, c0, c1 = blk.trim
        sub = vec[c0:c1]
        p = blk.payload
        if hasattr(p, "factors"):
            out[r0:r1] += idbf_apply(p, sub)
        elif hasattr(p, "u"):
            out[r0:r1] += _lr_apply(p, sub)
        else:
            out[r0:r1] += p @ sub
    return out


def apply_half_transpose(blocks, vec, n_out):
    """Transposed block sum (alt.py:211-222)."""
    out = np.zeros(n_out)
    for blk in blocks:
        r0, r1, c0, c1 = blk.trim
        sub = vec[r0:r1]
        p = blk.payload
        if hasattr(p, "factors"):
            out[c0:c1] += idbf_apply_transpose(p, sub)
        elif hasattr(p, "u"):
            out[c0:c1] += _lr_apply_t(p, sub)
        else:
            out[c0:c1] += p.T @ sub
    return out


def forward_real(plan, beta):
    """Parity split + symmetric assembly (alt.py:225-236)."""
    n = plan.n
    g_odd = np.zeros(n)
    g_even = np.zeros(n)
    if plan.spec_odd is not None:
        g_odd = apply_half(plan.blocks_odd, beta[1::2], n)
    if plan.spec_even is not None:
        g_even = apply_half(plan.blocks_even, beta[0::2], n)
    out = np.empty(2 * n)
    out[n:] = g_even + g_odd
    out[n - 1::-1] = g_even - g_odd
    return out


def inverse_real(plan, f, weights):
    """Weighted fold + transposed halves (alt.py:239-253)."""
    n = plan.n
    w_pos = weights[n:]
    upper = f[n:]
    lower = f[n - 1::-1]
    beta = np.zeros(2 * n - plan.m)
    if plan.spec_odd is not None:
        beta[1::2] = apply_half_transpose(plan.blocks_odd,
                                          w_pos * (upper - lower),
                                          plan.spec_odd.num_cols)
    if plan.spec_even is not None:
        beta[0::2] = apply_half_transpose(plan.blocks_even,
                                          w_pos * (upper + lower),
                                          plan.spec_even.num_cols)
    return beta


def _weights(plan):
    return plan.quadrature.weights


def alt_forward(plan, values):
    """Complex -> two real applies (alt.py:256-272)."""
    values = np.asarray(values)
    if values.shape != (2 * plan.n - plan.m,):
        raise ValueError(f"expected {2 * plan.n - plan.m} coefficients, "
                         f"got shape {values.shape}")
    if np.iscomplexobj(values):
        return forward_real(plan, values.real.astype(np.float64)) \
            + 1j * forward_real(plan, values.imag.astype(np.float64))
    return forward_real(plan, values.astype(np.float64))


def alt_inverse(plan, values):
    """(alt.py:275-282)"""
    values = np.asarray(values)
    if values.shape != (2 * plan.n,):
        raise ValueError(f"expected {2 * plan.n} node values, "
                         f"got shape {values.shape}")
    w = _weights(plan)
    if np.iscomplexobj(values):
        return inverse_real(plan, values.real.astype(np.float64), w) \
            + 1j * inverse_real(plan, values.imag.astype(np.float64), w)
    return inverse_real(plan, values.astype(np.float64), w)


def bins(n):
    """(sht.py:131-134)"""
    num_phi = 4 * n - 1
    ms = np.arange(-(2 * n - 1), 2 * n)
    return num_phi, ms, np.where(ms >= 0, ms, ms + num_phi)


def coeff_offsets(n):
    """Start of each order in the flat m-major layout (sht.py:68-81)."""
    ms = np.arange(-(2 * n - 1), 2 * n)
    lens = 2 * n - np.abs(ms)
    return ms, np.concatenate([[0], np.cumsum(lens)])


def sht_forward(alt_plans, n, flat):
    """Synthesis (sht.py:137-148); flat = ShtCoeffs.pack() layout."""
    num_phi, ms, bns = bins(n)
    _, offs = coeff_offsets(n)
    phi0 = np.pi / num_phi
    buf = np.zeros((2 * n, num_phi), dtype=np.complex128)
    for i, (m, b) in enumerate(zip(ms, bns)):
        g = alt_forward(alt_plans[abs(m)], flat[offs[i]:offs[i + 1]])
        buf[:, b] = g * np.exp(1j * m * phi0)
    return num_phi * np.fft.ifft(buf, axis=1)


def sht_inverse(alt_plans, n, values):
    """Analysis (sht.py:151-166); returns the flat coefficient layout."""
    num_phi, ms, bns = bins(n)
    _, offs = coeff_offsets(n)
    phi0 = np.pi / num_phi
    spectrum = np.fft.fft(values, axis=1) / num_phi
    out = np.zeros(offs[-1], dtype=np.complex128)
    for i, (m, b) in enumerate(zip(ms, bns)):
        g = spectrum[:, b] * np.exp(-1j * m * phi0)
        out[offs[i]:offs[i + 1]] = alt_inverse(alt_plans[abs(m)], g)
    return out
