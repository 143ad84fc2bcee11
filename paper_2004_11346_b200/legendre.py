"""Quadrature and Legendre-function tables used at plan time.

Conventions are the reference's (pkg/src/bfsht/special.py:1-10): Pbar_k^m is
L2-normalized on (-1, 1) without the Condon-Shortley phase, quadrature nodes
ascend in x = cos(theta).  Every routine here reproduces the reference's
floating-point operation sequence so that the plans built on top of it are
bitwise identical to the reference planner's (checked against committed
plan digests in tests/test_planner.py).
"""
import ctypes
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import native

# rescaling / flush constants of the reference recurrence
# (pkg/src/bfsht/kernels/common.py:27-32)
MAG_MIN = float(np.exp(-700.0))
_LN2 = float(np.log(2.0))


@dataclass
class QuadratureRule:
    """Gauss-Legendre rule: nodes ascending in (-1, 1), positive weights."""

    order: int
    nodes: np.ndarray
    weights: np.ndarray


def _poly_and_slope(order, x):
    # degree-`order` Legendre polynomial and derivative by the three-term
    # recurrence (pkg/src/bfsht/special.py:33-43), same evaluation order
    lo = np.ones_like(x)
    hi = x.copy()
    for k in range(1, order):
        nxt = ((2.0 * k + 1.0) * x * hi - k * lo) / (k + 1.0)
        lo = hi
        hi = nxt
    return hi, order * (x * hi - lo) / (x * x - 1.0)


def gauss_legendre(order):
    """Newton-refined Gauss-Legendre rule (pkg/src/bfsht/special.py:46-73)."""
    if order < 1:
        raise ValueError("order must be >= 1")
    idx = np.arange(order, dtype=np.float64)
    x = np.cos(np.pi * (idx + 0.75) / (order + 0.5))
    if order == 1:
        x[0] = 0.0
    for _ in range(20):
        p, dp = _poly_and_slope(order, x)
        step = p / dp
        x -= step
        if np.max(np.abs(step)) <= 1e-15:
            break
    p, dp = _poly_and_slope(order, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    x = 0.5 * (x - x[::-1])
    w = 0.5 * (w + w[::-1])
    return QuadratureRule(order=order, nodes=x[::-1].copy(),
                          weights=w[::-1].copy())


def recurrence_coefficients(m, k_max):
    """alpha_s, beta_s of the degree step k -> k+1 for k = m..k_max-1
    (pkg/src/bfsht/kernels/common.py:37-53)."""
    if k_max <= m:
        z = np.zeros(0)
        return z, z
    k = np.arange(m, k_max, dtype=np.float64)
    den = (k + 1.0 - m) * (k + 1.0 + m)
    alpha = np.sqrt((2.0 * k + 1.0) * (2.0 * k + 3.0) / den)
    num_b = (2.0 * k + 3.0) * (k - m) * (k + m)
    with np.errstate(divide="ignore", invalid="ignore"):
        beta = np.sqrt(num_b / ((2.0 * k - 1.0) * den))
    beta[k == m] = 0.0
    return alpha, beta


@lru_cache(maxsize=4096)
def _log_prefactor(m):
    j = np.arange(1, m + 1, dtype=np.float64)
    s = float(np.sum(np.log((2.0 * j - 1.0) / (2.0 * j))))
    return 0.5 * (float(np.log(m + 0.5)) + s)


def start_values(m, x):
    """Pbar_m^m(x) as mantissa * 2**exp (pkg/src/bfsht/kernels/common.py:65-77)."""
    x = np.asarray(x, dtype=np.float64)
    lp = _log_prefactor(m) + 0.5 * m * (np.log1p(-x) + np.log1p(x))
    e2 = np.floor(lp / _LN2)
    mant = np.exp(lp - e2 * _LN2)
    return mant, e2.astype(np.int32)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def half_table(m, offset, x, ncols, device=None):
    """Dense parity half: out[r, j] = Pbar_{m+offset+2j}^m(x[r]).

    ``device`` (a CUDA ordinal) evaluates the entries on that GPU
    (bfsht_half_table_device): the same bits, returned as the
    transpose of a column-major buffer (the planner reads the table only
    through copies, so its layout does not reach the factors)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if device is not None and x.size and ncols:
        return _half_table_device(m, offset, x, ncols, int(device))
    out = np.empty((x.size, ncols))
    if x.size == 0 or ncols == 0:
        return out
    k_last = m + offset + 2 * (ncols - 1)
    alpha, beta = recurrence_coefficients(m, k_last)
    alpha = np.ascontiguousarray(alpha)
    beta = np.ascontiguousarray(beta)
    mant, e2 = start_values(m, x)
    mant = np.ascontiguousarray(mant)
    e2 = np.ascontiguousarray(e2, dtype=np.int32)
    native.host().bfsht_legendre_half_table(
        m, offset, x.size, ncols, _ptr(x), _ptr(alpha), _ptr(beta),
        _ptr(mant), _ptr(e2), MAG_MIN, _ptr(out))
    return out


_DEVICE_USED = False


def device_tables_used():
    """True once this process has tabulated on a GPU (it then holds a CUDA
    context, so planner workers must not be forked from it)."""
    return _DEVICE_USED


def _half_table_device(m, offset, x, ncols, device):
    global _DEVICE_USED
    _DEVICE_USED = True
    k_last = m + offset + 2 * (ncols - 1)
    alpha, beta = recurrence_coefficients(m, k_last)
    alpha = np.ascontiguousarray(alpha)
    beta = np.ascontiguousarray(beta)
    mant, e2 = start_values(m, x)
    mant = np.ascontiguousarray(mant)
    e2 = np.ascontiguousarray(e2, dtype=np.int32)
    out = np.empty((ncols, x.size))
    lib = native.cuda()
    rc = lib.bfsht_half_table_device(device, m, offset, x.size, ncols, _ptr(x), _ptr(alpha),
                                     _ptr(beta), _ptr(mant), _ptr(e2), MAG_MIN, _ptr(out))
    if rc != 0:
        raise RuntimeError("bfsht_half_table_device: "
                           + lib.bfsht_last_error().decode())
    return out.T


def legendre_table(m, x, degrees):
    """Table of Pbar_degree^m(x), shape (len(x), len(degrees)); degrees
    ascending and >= m (pkg/src/bfsht/kernels/__init__.py:81-105)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    degrees = np.ascontiguousarray(degrees, dtype=np.int64)
    out = np.zeros((x.size, degrees.size))
    if degrees.size == 0 or x.size == 0:
        return out
    if degrees[0] < m or np.any(np.diff(degrees) <= 0):
        raise ValueError("degrees must be sorted ascending, distinct, >= m")
    if np.any(np.abs(x) >= 1.0):
        raise ValueError("x must lie strictly inside (-1, 1)")
    alpha, beta = recurrence_coefficients(m, int(degrees[-1]))
    alpha = np.ascontiguousarray(alpha)
    beta = np.ascontiguousarray(beta)
    mant, e2 = start_values(m, x)
    mant = np.ascontiguousarray(mant)
    e2 = np.ascontiguousarray(e2, dtype=np.int32)
    native.host().bfsht_legendre_table(
        m, x.size, _ptr(x), degrees.size, _ptr(degrees), _ptr(alpha),
        _ptr(beta), _ptr(mant), _ptr(e2), MAG_MIN, _ptr(out))
    return out
