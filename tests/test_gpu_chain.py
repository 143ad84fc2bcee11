"""GPU: the chain kernel (alt_chain_kernel: bundle schedule, 32-byte records,
folded index adds) runs the butterfly-chain stages bitwise like the stage
kernel, and both match the oracle.  BFSHT_CHAIN is read when a device plan
is created: 0 = every stage on alt_stage_kernel, 1 = default (stages with
gather / lane-map ops on the chain kernel), 2 = every stage."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt

import oracle.apply as OA

pytestmark = pytest.mark.gpu

CASES = [(64, [0, 3, 64, 126, 127], 16), (128, [100, 0, 1], 16),
         (256, [0, 1, 300, 511], 32), (512, [0, 1, 100, 700], 512)]


def _run(monkeypatch, mode, plans, flat_f, flat_i, **env):
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    monkeypatch.setenv("BFSHT_CHAIN", str(mode))
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    dp = DevicePlan(plans)
    f = dp.alt_orders(FORWARD, torch.from_numpy(flat_f).cuda()).cpu().numpy()
    i = dp.alt_orders(INVERSE, torch.from_numpy(flat_i).cuda()).cpu().numpy()
    n_launch = dp.launches()
    dp.close()
    return f, i, n_launch


@pytest.mark.parametrize("n,ms,n0", CASES)
def test_chain_kernel_bitwise_equals_stage_kernel(monkeypatch, n, ms, n0):
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=n0, quadrature=q)
             for m in ms]
    rng = np.random.default_rng(n)
    vf = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m) for m in ms]
    vi = [rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n) for _ in ms]
    ff, fi = np.concatenate(vf), np.concatenate(vi)
    f0, i0, _ = _run(monkeypatch, 0, plans, ff, fi)
    for mode, env in ((1, {}), (2, {}), (2, {"BFSHT_CHAIN_BUNDLES": 1}),
                      (1, {"BFSHT_CHAIN_BUNDLES": 64, "BFSHT_CHAIN_CFIX": 0})):
        f1, i1, _ = _run(monkeypatch, mode, plans, ff, fi, **env)
        assert np.array_equal(f0, f1), (mode, env)
        assert np.array_equal(i0, i1), (mode, env)
    out = f0.reshape(len(ms), 2 * n)
    pos = 0
    for o, (p, v, f) in enumerate(zip(plans, vf, vi)):
        assert np.linalg.norm(out[o] - OA.alt_forward(p, v)) <= 1e-12 * np.linalg.norm(out[o])
        ln = 2 * n - p.m
        want = OA.alt_inverse(p, f)
        assert np.linalg.norm(i0[pos:pos + ln] - want) <= 1e-12 * np.linalg.norm(want)
        pos += ln


def test_chain_kernel_sht_bitwise(monkeypatch):
    """Whole SHT at N=64 (n0=16: butterflies at every low order) with and
    without the chain kernel."""
    import torch
    from paper_2004_11346_b200 import ShtCoeffs, plan_sht
    from paper_2004_11346_b200.api import ShtDevice
    n = 64
    plan = plan_sht(n, n0=16)
    rng = np.random.default_rng(5)
    flat = rng.standard_normal(4 * n * n) + 1j * rng.standard_normal(4 * n * n)
    res = []
    for mode in (0, 1, 2):
        monkeypatch.setenv("BFSHT_CHAIN", str(mode))
        dev = ShtDevice(plan)
        g = dev.forward(torch.from_numpy(flat).cuda())
        b = dev.inverse(g)
        res.append((g.cpu().numpy(), b.cpu().numpy()))
    for g, b in res[1:]:
        assert np.array_equal(g, res[0][0])
        assert np.array_equal(b, res[0][1])


def test_chain_kernel_with_regenerated_tiles(monkeypatch):
    """Plans with regenerated turning tiles (f1): mode 2 must leave the
    stages that hold seeded tiles on the stage kernel; results bitwise those
    of the stage kernel alone."""
    import torch
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    n, ms = 256, [0, 1, 300]
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=32, quadrature=q) for m in ms]
    rng = np.random.default_rng(3)
    ff = np.concatenate([rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
                         for m in ms])
    fi = np.concatenate([rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)
                         for _ in ms])
    res = []
    for mode in (0, 1, 2):
        monkeypatch.setenv("BFSHT_CHAIN", str(mode))
        dp = DevicePlan(plans, regen=1.0)
        assert dp.packed.regen_tiles > 0
        nst = len(dp.packed.stages_fwd) - 1
        info = [dp.chain_info(FORWARD, s) for s in range(nst)]
        if mode == 0:
            assert all(i[0] == 0 for i in info)
        else:
            assert any(i[0] > 0 for i in info)
        f = dp.alt_orders(FORWARD, torch.from_numpy(ff).cuda()).cpu().numpy()
        i = dp.alt_orders(INVERSE, torch.from_numpy(fi).cuda()).cpu().numpy()
        res.append((f, i))
        dp.close()
    for f, i in res[1:]:
        assert np.array_equal(f, res[0][0]) and np.array_equal(i, res[0][1])


def test_plan_upload_path_builds_the_chain_schedule():
    """The C-only residency path (bfsht_plan_upload: the library owns every
    device array) builds the same chain schedule as bfsht_plan_wrap and gives
    the same results, bit for bit."""
    import ctypes
    import torch
    from paper_2004_11346_b200 import native
    from paper_2004_11346_b200._capi import check
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    from paper_2004_11346_b200.pack import pack_plans
    n, ms = 256, [0, 1, 300]
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=32, quadrature=q) for m in ms]
    rng = np.random.default_rng(11)
    ff = np.concatenate([rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m)
                         for m in ms])
    fi = np.concatenate([rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)
                         for _ in ms])
    dp = DevicePlan(plans)
    want_f = dp.alt_orders(FORWARD, torch.from_numpy(ff).cuda()).cpu().numpy()
    want_i = dp.alt_orders(INVERSE, torch.from_numpy(fi).cuda()).cpu().numpy()
    nst = len(dp.packed.stages_fwd) - 1
    want_info = [dp.chain_info(FORWARD, s) for s in range(nst)]
    assert any(i[0] > 0 for i in want_info)

    lib = native.cuda()
    packed = pack_plans(plans)
    h = ctypes.c_void_p()
    check(lib, lib.bfsht_plan_upload(packed._h, ctypes.byref(h)), "bfsht_plan_upload")
    try:
        out = (ctypes.c_int64 * 3)()
        for s in range(nst):
            check(lib, lib.bfsht_plan_chain_info(h, FORWARD, s, out), "bfsht_plan_chain_info")
            assert tuple(int(v) for v in out) == want_info[s]
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        x = torch.from_numpy(ff).cuda()
        y = torch.empty(len(ms) * 2 * n, dtype=torch.complex128, device="cuda")
        check(lib, lib.bfsht_alt_orders(h, FORWARD, ctypes.c_void_p(x.data_ptr()),
                                        ctypes.c_void_p(y.data_ptr()), None, st), "fwd")
        g = torch.from_numpy(fi).cuda()
        b = torch.empty(ff.size, dtype=torch.complex128, device="cuda")
        check(lib, lib.bfsht_alt_orders(h, INVERSE, ctypes.c_void_p(g.data_ptr()),
                                        ctypes.c_void_p(b.data_ptr()),
                                        ctypes.c_void_p(dp.weights.data_ptr()), st), "inv")
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want_f)
        assert np.array_equal(b.cpu().numpy(), want_i)
    finally:
        lib.bfsht_plan_free(h)
        dp.close()
