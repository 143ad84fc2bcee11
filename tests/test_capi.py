"""C ABI: both libraries load on a CPU-only box and export every symbol the
headers declare (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_2004_11346_b200 import _capi, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "bfsht_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bfsht_[a-z_]+)\s*\(", src)))


def test_header_symbols_listed():
    assert set(_declared()) == set(_capi.EXPORTS)


def test_cuda_library_exports_every_symbol():
    from paper_2004_11346_b200 import build
    build.build_cuda()
    lib = ctypes.CDLL(native.CUDA_LIB)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing


def test_host_library_exports_packer_and_recurrence():
    lib = native.host()
    for s in ("bfsht_pack_plan", "bfsht_packed_info", "bfsht_packed_arrays",
              "bfsht_packed_free", "bfsht_legendre_half_table",
              "bfsht_legendre_table"):
        assert hasattr(lib, s), s


def test_declared_argtypes_cover_exports():
    lib = ctypes.CDLL(native.CUDA_LIB)
    _capi.declare(lib)
    for s in _capi.EXPORTS:
        assert getattr(lib, s).restype is not None or s.endswith("_free")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2004_11346_b200 import api, plan_alt
    plan = plan_alt(8, 2, n0=8)
    with pytest.raises(RuntimeError, match="CUDA device"):
        api.alt_forward(plan, [0.0] * 14)
