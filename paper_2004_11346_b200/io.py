"""SHTC / SHTG binary files, host and direct-to-device.

Same formats, names and ValueError messages as the reference
(pkg/src/bfsht/io.py:1-100): a 16-byte little-endian header (4-byte magic,
u32 version = 1, u32 N, u32 dtype code 0 = complex128 / 1 = complex64), then
the payload — coefficients ("SHTC") as ShtCoeffs.pack() order (m from
-(2N-1) ascending, 2N-|m| values each), grid values ("SHTG") 2N x (4N-1)
row-major.

The device variants move the payload between the file and HBM through one
pinned staging buffer (file -> pinned host -> device with no intermediate
numpy copy; complex64 files widen on the device), which is how the
transform CLI's read-transform-write loop (cli.py:100-158) would feed
``ShtDevice`` without the host round trips of ``load_* -> pack()``.
"""
import struct

import numpy as np

from .sht import ShtCoeffs, ShtGridValues

__all__ = ["save_coeffs", "load_coeffs", "save_grid", "load_grid",
           "load_coeffs_device", "load_grid_device", "save_coeffs_device",
           "save_grid_device"]

_MAGIC_COEFFS = b"SHTC"
_MAGIC_GRID = b"SHTG"
_VERSION = 1
_DTYPES = {0: np.dtype("<c16"), 1: np.dtype("<c8")}
_CODES = {np.dtype(np.complex128): 0, np.dtype(np.complex64): 1}


def _header(magic, n, dtype):
    code = _CODES.get(np.dtype(dtype))
    if code is None:
        raise ValueError(f"unsupported dtype {dtype}; use complex128 or complex64")
    return magic + struct.pack("<III", _VERSION, n, code)


def _parse_header(fh, magic):
    got = fh.read(4)
    if got != magic:
        raise ValueError(f"bad magic {got!r} at offset 0, expected {magic!r}")
    raw = fh.read(12)
    if len(raw) < 12:
        raise ValueError(f"truncated header at offset {4 + len(raw)}")
    ver, n, code = struct.unpack("<III", raw)
    if ver != _VERSION:
        raise ValueError(f"unsupported version {ver} at offset 4")
    if code not in _DTYPES:
        raise ValueError(f"unknown dtype code {code} at offset 12")
    if n < 1:
        raise ValueError(f"invalid N={n} at offset 8")
    return n, _DTYPES[code]


def _read_into(fh, buf, what):
    """Fill a writable byte view from fh, raising the reference's
    truncation message on a short read."""
    start = fh.tell()
    mv = memoryview(buf).cast("B")
    got = 0
    while got < len(mv):
        k = fh.readinto(mv[got:])
        if not k:
            break
        got += k
    if got < len(mv):
        raise ValueError(f"truncated {what}: wanted {len(mv)} bytes at offset "
                         f"{start}, got {got}")


def _check_tail(fh):
    if fh.read(1):
        raise ValueError(f"trailing garbage at offset {fh.tell() - 1}")


def _grid_of(grid_values):
    if isinstance(grid_values, ShtGridValues):
        n, values = grid_values.n, grid_values.values
    else:
        values = np.asarray(grid_values)
        n = values.shape[0] // 2 if values.ndim == 2 else 0
    if values.shape != (2 * n, 4 * n - 1) or n < 1:
        raise ValueError(f"grid shape {values.shape} is not 2N x (4N-1)")
    return n, values


# ------------------------------------------------------------------ host
def save_coeffs(coeffs, fh, dtype=np.complex128):
    fh.write(_header(_MAGIC_COEFFS, coeffs.n, dtype))
    fh.write(coeffs.pack().astype(np.dtype(dtype).newbyteorder("<")).tobytes())


def load_coeffs(fh):
    n, dt = _parse_header(fh, _MAGIC_COEFFS)
    flat = np.empty(4 * n * n, dtype=dt)
    _read_into(fh, flat, "coefficient payload")
    _check_tail(fh)
    return ShtCoeffs.unpack(n, flat.astype(np.complex128))


def save_grid(grid_values, fh, dtype=np.complex128):
    n, values = _grid_of(grid_values)
    fh.write(_header(_MAGIC_GRID, n, dtype))
    fh.write(np.ascontiguousarray(values).astype(np.dtype(dtype).newbyteorder("<")).tobytes())


def load_grid(fh):
    n, dt = _parse_header(fh, _MAGIC_GRID)
    values = np.empty((2 * n, 4 * n - 1), dtype=dt)
    _read_into(fh, values, "grid payload")
    _check_tail(fh)
    return ShtGridValues(n=n, values=values.astype(np.complex128))


# ---------------------------------------------------------------- device
def _torch_dtype(torch, dt):
    return torch.complex128 if dt == _DTYPES[0] else torch.complex64


def _load_device(fh, magic, shape_of, what, device):
    import torch
    n, dt = _parse_header(fh, magic)
    shape = shape_of(n)
    staged = torch.empty(shape, dtype=_torch_dtype(torch, dt)).pin_memory()
    _read_into(fh, staged.numpy(), what)
    _check_tail(fh)
    out = staged.to(device, non_blocking=True)
    if out.dtype != torch.complex128:
        out = out.to(torch.complex128)
    torch.cuda.current_stream(out.device).synchronize()   # staging buffer reusable
    return n, out


def load_coeffs_device(fh, device="cuda"):
    """SHTC file -> (N, flat complex128 CUDA tensor in ShtCoeffs.pack()
    order), ready for ShtDevice.forward."""
    return _load_device(fh, _MAGIC_COEFFS, lambda n: (4 * n * n,),
                        "coefficient payload", device)


def load_grid_device(fh, device="cuda"):
    """SHTG file -> (N, 2N x (4N-1) complex128 CUDA tensor), ready for
    ShtDevice.inverse."""
    return _load_device(fh, _MAGIC_GRID, lambda n: (2 * n, 4 * n - 1),
                        "grid payload", device)


def _save_device(fh, magic, n, t, dtype):
    import torch
    header = _header(magic, n, dtype)
    want = torch.complex128 if np.dtype(dtype) == np.complex128 else torch.complex64
    src = t.to(want) if t.dtype != want else t
    staged = torch.empty(tuple(src.shape), dtype=want).pin_memory()
    staged.copy_(src)
    fh.write(header)
    fh.write(memoryview(staged.numpy()).cast("B"))


def save_coeffs_device(n, flat, fh, dtype=np.complex128):
    """Flat coefficient CUDA tensor (pack() order) -> SHTC file."""
    if tuple(flat.shape) != (4 * n * n,):
        raise ValueError(f"expected {4 * n * n} coefficients, got shape {tuple(flat.shape)}")
    _save_device(fh, _MAGIC_COEFFS, n, flat, dtype)


def save_grid_device(grid, fh, dtype=np.complex128):
    """2N x (4N-1) CUDA tensor -> SHTG file."""
    shape = tuple(grid.shape)
    n = shape[0] // 2 if len(shape) == 2 else 0
    if shape != (2 * n, 4 * n - 1) or n < 1:
        raise ValueError(f"grid shape {shape} is not 2N x (4N-1)")
    _save_device(fh, _MAGIC_GRID, n, grid, dtype)
