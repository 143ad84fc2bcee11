"""Loader for tests/golden (written from the reference by make_golden.py)."""
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load():
    with open(os.path.join(HERE, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(HERE, "golden.npz"))
    return meta, arrays


def seeded_complex(seed, size):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(size) + 1j * rng.standard_normal(size)


def sht_flat(n, seed):
    rng = np.random.default_rng(seed)
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        k = np.arange(abs(m), 2 * n)
        parts.append((rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
                     / (1.0 + k))
    return np.concatenate(parts)


def sht_grid(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((2 * n, 4 * n - 1)) \
        + 1j * rng.standard_normal((2 * n, 4 * n - 1))
