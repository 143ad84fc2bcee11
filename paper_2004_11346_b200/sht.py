"""SHT containers and grid (reference layout, pkg/src/bfsht/sht.py:34-106).

``ShtCoeffs`` stores beta_{k,m} per order m = -(2N-1)..2N-1 (k ascending
from |m|); ``pack()`` gives the flat m-major layout the device path
consumes.  ``ShtGridValues.values`` is the 2N x (4N-1) grid, rows
node-ascending (theta descending), phis at half-sample offsets.
"""
from dataclasses import dataclass

import numpy as np

from .legendre import gauss_legendre


@dataclass
class ShtGrid:
    n: int
    thetas: np.ndarray
    phis: np.ndarray


@dataclass
class ShtCoeffs:
    """beta_{k,m} for |m| <= k <= 2N-1, stored per m ascending from -(2N-1)."""

    n: int
    by_m: list

    @classmethod
    def zeros(cls, n):
        return cls(n=n, by_m=[np.zeros(2 * n - abs(m), dtype=np.complex128)
                              for m in range(-(2 * n - 1), 2 * n)])

    def _idx(self, m):
        if abs(m) > 2 * self.n - 1:
            raise IndexError(f"order {m} outside band limit {2 * self.n - 1}")
        return m + 2 * self.n - 1

    def __getitem__(self, m):
        return self.by_m[self._idx(m)]

    def __setitem__(self, m, values):
        values = np.asarray(values, dtype=np.complex128)
        if values.shape != (2 * self.n - abs(m),):
            raise ValueError(f"order {m} expects {2 * self.n - abs(m)} "
                             f"coefficients, got {values.shape}")
        self.by_m[self._idx(m)] = values

    def pack(self):
        return np.concatenate(self.by_m)

    @classmethod
    def unpack(cls, n, flat):
        out, pos = [], 0
        for m in range(-(2 * n - 1), 2 * n):
            ln = 2 * n - abs(m)
            out.append(np.asarray(flat[pos:pos + ln], dtype=np.complex128))
            pos += ln
        if pos != len(flat):
            raise ValueError(f"expected {pos} coefficients, got {len(flat)}")
        return cls(n=n, by_m=out)


@dataclass
class ShtGridValues:
    n: int
    values: np.ndarray


def make_grid(n, quadrature=None):
    if quadrature is None:
        quadrature = gauss_legendre(2 * n)
    num_phi = 4 * n - 1
    phis = 2.0 * np.pi * (np.arange(num_phi) + 0.5) / num_phi
    return ShtGrid(n=n, thetas=np.arccos(quadrature.nodes), phis=phis)


def num_coeffs(n):
    return 4 * n * n
