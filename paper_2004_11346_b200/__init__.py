"""bfsht-b200: B200-native apply phase of the IDBF-accelerated SHT.

Reference package: ``bfsht`` (arXiv 2004.11346).  Plan construction keeps
the reference API and produces bitwise-identical factors (``plan_alt``,
``plan_sht``); the apply path (``alt_forward``, ``alt_inverse``,
``sht_forward``, ``sht_inverse``) runs hand-written sm_100a CUDA kernels
through the C ABI in include/bfsht_b200.h.
"""
from .factors import (ButterflyFactorization, LowRankFactor, RankOverflowError,
                      SamplingConfig, SparseFactor, idbf_factor)
from .legendre import QuadratureRule, gauss_legendre, legendre_table
from .plan import (N0_DEFAULT, TAU_DEFAULT, AltPlan, Block, ShtPlan,
                   make_alt_spec, plan_alt, plan_diagnostics, plan_orders,
                   plan_sht)
from .sht import ShtCoeffs, ShtGrid, ShtGridValues, make_grid

__all__ = [
    "ButterflyFactorization", "LowRankFactor", "RankOverflowError",
    "SamplingConfig", "SparseFactor", "idbf_factor", "QuadratureRule",
    "gauss_legendre", "legendre_table", "N0_DEFAULT", "TAU_DEFAULT",
    "AltPlan", "Block", "ShtPlan", "make_alt_spec", "plan_alt",
    "plan_diagnostics", "plan_orders", "plan_sht", "ShtCoeffs", "ShtGrid", "ShtGridValues",
    "make_grid", "alt_forward", "alt_inverse", "sht_forward", "sht_inverse",
    "CoeffVector", "GridFunctionColumn", "DevicePlan", "ShtDevice",
    "HostPipeline", "idbf_apply", "idbf_apply_transpose",
]


def __getattr__(name):
    # the device API loads torch + the CUDA library lazily
    if name in ("alt_forward", "alt_inverse", "sht_forward", "sht_inverse",
                "CoeffVector", "GridFunctionColumn", "DevicePlan",
                "ShtDevice", "dft_rows", "HostPipeline", "idbf_apply",
                "idbf_apply_transpose"):
        from . import api
        return getattr(api, name)
    raise AttributeError(name)
