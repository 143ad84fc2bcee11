"""ctypes loader for the two in-tree native libraries.

* ``libbfsht_host.so`` — plan-time C/C++: the Legendre recurrence table
  builder (csrc/recur.c) and the device-plan packer (csrc/packer.cpp).
* ``libbfsht_b200.so`` — the sm_100a CUDA kernels behind the C ABI declared
  in include/bfsht_b200.h.

Both are built in-tree by ``__graft_entry__.build()`` (or ``python -m
paper_2004_11346_b200.build``).  There is no fallback: a missing library is
an ImportError at first use, never a silent CPU path.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(_HERE, "libbfsht_host.so")
CUDA_LIB = os.path.join(_HERE, "libbfsht_b200.so")

_host = None
_cuda = None


def host():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise ImportError(f"{HOST_LIB} is not built; run "
                              "python -m paper_2004_11346_b200.build")
        lib = ctypes.CDLL(HOST_LIB)
        _declare_host(lib)
        _host = lib
    return _host


def cuda():
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB):
            raise ImportError(f"{CUDA_LIB} is not built; run "
                              "python -m paper_2004_11346_b200.build")
        lib = ctypes.CDLL(CUDA_LIB)
        from . import _capi
        _capi.declare(lib)
        _cuda = lib
    return _cuda


_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def _declare_host(lib):
    lib.bfsht_legendre_half_table.restype = ctypes.c_int
    lib.bfsht_legendre_half_table.argtypes = [_I64, _I64, _I64, _I64, _P, _P,
                                              _P, _P, _P, ctypes.c_double, _P]
    lib.bfsht_legendre_table.restype = ctypes.c_int
    lib.bfsht_legendre_table.argtypes = [_I64, _I64, _P, _I64, _P, _P, _P,
                                         _P, _P, ctypes.c_double, _P]
    if hasattr(lib, "bfsht_pack_plan"):
        from . import pack
        pack.declare(lib)
