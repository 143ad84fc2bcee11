"""Dense O(N^2)-per-order references — TEST INFRASTRUCTURE.

Restates pkg/src/bfsht/oracle.py:38-92: the materialized order-m ALT matrix
over all 2N nodes (rows node-ascending, columns degrees m..2N-1) and direct
(FFT-free) SHT sums.  Matrix entries come from the same scaled recurrence
the plans are built from (paper_2004_11346_b200.legendre, bitwise equal to
the reference's legendre_table).
"""
import numpy as np

from paper_2004_11346_b200.legendre import gauss_legendre, legendre_table


def alt_matrix(n, m, quadrature=None):
    """Full 2N x (2N-m) matrix Pbar_k^m(x_l) (test_alt.py:21-24 form)."""
    q = gauss_legendre(2 * n) if quadrature is None else quadrature
    return legendre_table(m, q.nodes, np.arange(m, 2 * n, dtype=np.int64)), q


def dense_alt_forward(n, m, beta, quadrature=None):
    a, _ = alt_matrix(n, m, quadrature)
    return a @ beta


def dense_alt_inverse(n, m, f, quadrature=None):
    a, q = alt_matrix(n, m, quadrature)
    return a.T @ (q.weights * f)


def dense_sht_forward(n, flat):
    """Direct synthesis (oracle.py:61-73); flat = ShtCoeffs.pack() layout."""
    q = gauss_legendre(2 * n)
    num_phi = 4 * n - 1
    phis = 2.0 * np.pi * (np.arange(num_phi) + 0.5) / num_phi
    out = np.zeros((2 * n, num_phi), dtype=np.complex128)
    pos = 0
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        table = legendre_table(abs(m), q.nodes, np.arange(abs(m), 2 * n))
        g = table @ flat[pos:pos + ln]
        out += g[:, None] * np.exp(1j * m * phis)[None, :]
        pos += ln
    return out


def dense_sht_inverse(n, values):
    """Direct analysis (oracle.py:76-92); returns the flat layout."""
    q = gauss_legendre(2 * n)
    num_phi = 4 * n - 1
    phis = 2.0 * np.pi * (np.arange(num_phi) + 0.5) / num_phi
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        g = values @ np.exp(-1j * m * phis) / num_phi
        table = legendre_table(abs(m), q.nodes, np.arange(abs(m), 2 * n))
        parts.append(table.T @ (q.weights * g))
    return np.concatenate(parts)
