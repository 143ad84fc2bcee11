"""Write SHTC/SHTG fixture files with the reference package itself
(pkg/src/bfsht/io.py), for tests/test_io.py.  Run once in a container that
has /root/reference; the outputs are committed (tests/golden/io_*.bin).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py
"""
import os

import numpy as np

from bfsht import io as RIO
from bfsht.sht import ShtCoeffs

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    n = 3
    rng = np.random.default_rng(11)
    c = ShtCoeffs.unpack(n, rng.standard_normal(4 * n * n) + 1j * rng.standard_normal(4 * n * n))
    g = rng.standard_normal((2 * n, 4 * n - 1)) + 1j * rng.standard_normal((2 * n, 4 * n - 1))
    for dt, tag in ((np.complex128, "c16"), (np.complex64, "c8")):
        with open(os.path.join(HERE, f"io_coeffs_{tag}.bin"), "wb") as fh:
            RIO.save_coeffs(c, fh, dtype=dt)
        with open(os.path.join(HERE, f"io_grid_{tag}.bin"), "wb") as fh:
            RIO.save_grid(g, fh, dtype=dt)
    np.savez(os.path.join(HERE, "io_values.npz"), coeffs=c.pack(), grid=g)


if __name__ == "__main__":
    main()
