"""SHTC / SHTG files (paper_2004_11346_b200/io.py): byte-exact
against files the reference wrote (tests/golden/make_io_golden.py), and the
reference's ValueError messages for malformed input (pkg/src/bfsht/io.py)."""
import io
import os
import struct

import numpy as np
import pytest

from paper_2004_11346_b200 import io as BIO
from paper_2004_11346_b200.sht import ShtCoeffs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
VALS = np.load(os.path.join(GOLD, "io_values.npz"))


def _bytes(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("tag,dt", [("c16", np.complex128), ("c8", np.complex64)])
def test_reference_files_round_trip(tag, dt):
    c = BIO.load_coeffs(io.BytesIO(_bytes(f"io_coeffs_{tag}.bin")))
    assert np.array_equal(c.pack(), VALS["coeffs"].astype(dt).astype(np.complex128))
    out = io.BytesIO()
    BIO.save_coeffs(ShtCoeffs.unpack(3, VALS["coeffs"]), out, dtype=dt)
    assert out.getvalue() == _bytes(f"io_coeffs_{tag}.bin")
    g = BIO.load_grid(io.BytesIO(_bytes(f"io_grid_{tag}.bin")))
    assert g.n == 3
    assert np.array_equal(g.values, VALS["grid"].astype(dt).astype(np.complex128))
    out = io.BytesIO()
    BIO.save_grid(VALS["grid"], out, dtype=dt)
    assert out.getvalue() == _bytes(f"io_grid_{tag}.bin")


def test_malformed_messages():
    good = _bytes("io_coeffs_c16.bin")
    cases = [
        (b"SHTX" + good[4:], "bad magic b'SHTX' at offset 0, expected b'SHTC'"),
        (good[:9], "truncated header at offset 9"),
        (good[:4] + struct.pack("<III", 2, 3, 0) + good[16:], "unsupported version 2 at offset 4"),
        (good[:4] + struct.pack("<III", 1, 3, 7) + good[16:], "unknown dtype code 7 at offset 12"),
        (good[:4] + struct.pack("<III", 1, 0, 0), "invalid N=0 at offset 8"),
        (good[:100], "truncated coefficient payload: wanted 576 bytes at offset 16, got 84"),
        (good + b"\0", "trailing garbage at offset 592"),
    ]
    for raw, msg in cases:
        with pytest.raises(ValueError) as ei:
            BIO.load_coeffs(io.BytesIO(raw))
        assert str(ei.value) == msg
    with pytest.raises(ValueError, match="unsupported dtype"):
        BIO.save_grid(VALS["grid"], io.BytesIO(), dtype=np.float64)
    with pytest.raises(ValueError, match=r"grid shape \(6, 10\) is not 2N x \(4N-1\)"):
        BIO.save_grid(np.zeros((6, 10)), io.BytesIO())


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["c16", "c8"])
def test_device_io_round_trip(tag):
    import torch
    from paper_2004_11346_b200 import plan_sht
    from paper_2004_11346_b200.api import ShtDevice, sht_forward
    n, flat = BIO.load_coeffs_device(io.BytesIO(_bytes(f"io_coeffs_{tag}.bin")))
    assert n == 3 and flat.is_cuda and flat.dtype == torch.complex128
    host = BIO.load_coeffs(io.BytesIO(_bytes(f"io_coeffs_{tag}.bin")))
    assert np.array_equal(flat.cpu().numpy(), host.pack())
    plan = plan_sht(n)
    grid = ShtDevice(plan).forward(flat)
    out = io.BytesIO()
    BIO.save_grid_device(grid, out)
    back = BIO.load_grid(io.BytesIO(out.getvalue()))
    assert np.array_equal(back.values, sht_forward(plan, host).values)
    n2, g2 = BIO.load_grid_device(io.BytesIO(out.getvalue()))
    assert n2 == n and torch.equal(g2, grid)
    out = io.BytesIO()
    BIO.save_coeffs_device(n, flat, out, dtype=np.complex64 if tag == "c8" else np.complex128)
    assert out.getvalue() == _bytes(f"io_coeffs_{tag}.bin")
