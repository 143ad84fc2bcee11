"""Packed-plan cache (pack.save_packed / load_packed): the
memory-mapped plan has the same arrays and runs the same in the emulated
engine; a DevicePlan built from it gives bitwise the same SHT (GPU)."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt, plan_sht
from paper_2004_11346_b200.pack import load_packed, pack_plans, save_packed

import packed_emulator as EMU

FIELDS = ("tiles", "ops", "idx", "maps", "tasks", "halves", "stages_fwd",
          "stages_inv", "rec", "xpos", "flow", "tinfo")


@pytest.mark.parametrize("regen", [0.0, 0.5])
def test_cache_round_trip(tmp_path, regen):
    n = 128
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=32, quadrature=q)
             for m in (0, 5, 100, 255)]
    pk = pack_plans(plans, regen=regen)
    path = str(tmp_path / "plan.bfpk")
    save_packed(pk, path)
    lp = load_packed(path)
    assert np.array_equal(lp.info, pk.info)
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(lp, f)), getattr(pk, f)), f
    assert lp.mag_min == pk.mag_min and lp.n == pk.n
    rng = np.random.default_rng(3)
    vecs = [rng.standard_normal(2 * n - p.m) + 1j * rng.standard_normal(2 * n - p.m) for p in plans]
    for a, b in zip(EMU.alt_orders(lp, plans, 0, vecs), EMU.alt_orders(pk, plans, 0, vecs)):
        assert np.array_equal(a, b)


def test_cache_rejects_other_files(tmp_path):
    p = tmp_path / "x.bin"
    p.write_bytes(b"nope" * 2000)
    with pytest.raises(ValueError, match="not a packed-plan file"):
        load_packed(str(p))


@pytest.mark.gpu
def test_device_plan_from_cache(tmp_path):
    import torch
    from paper_2004_11346_b200.api import DevicePlan
    n = 64
    plan = plan_sht(n)
    pk = pack_plans(plan.alt_plans)
    path = str(tmp_path / "sht.bfpk")
    save_packed(pk, path)
    a = DevicePlan(plan.alt_plans, weights=plan.quadrature.weights)
    b = DevicePlan([], packed=load_packed(path), weights=plan.quadrature.weights)
    c = torch.randn(4 * n * n, dtype=torch.complex128, device="cuda")
    ga, gb = a.sht_forward(c), b.sht_forward(c)
    assert torch.equal(ga, gb)
    assert torch.equal(a.sht_inverse(ga), b.sht_inverse(gb))
