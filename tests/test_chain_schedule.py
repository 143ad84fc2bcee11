"""Chain schedule (bfsht_chain_schedule, csrc/packer.cpp: 32-byte records in
cost-balanced bundles, folded index adds) on CPU: structural invariants, and
the numpy interpreter running the chain stages from their records gives the
same arena, bit for bit, as running the tasks — the GPU twin of this check
is tests/test_gpu_chain.py."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt
from paper_2004_11346_b200.pack import NRHS, chain_schedule, pack_plans

import oracle.apply as OA
import packed_emulator as EMU

# multi-factor butterflies (gather / scatter tasks) start at N = 256; N = 512
# orders 0, 1 also carry index adds that fold into tile ops
CASES = [(64, [0, 3, 64, 126, 127], 16), (256, [0, 1, 300], 32), (512, [0, 1], 512)]


def _plans(n, ms, n0):
    q = gauss_legendre(2 * n)
    return q, [plan_alt(n, m, SamplingConfig(tolerance=1e-10), n0=n0, quadrature=q) for m in ms]


@pytest.mark.parametrize("n,ms,n0", CASES)
@pytest.mark.parametrize("mode,per_warp,warps", [(1, 8, 24), (2, 1, 7), (2, 64, 1776)])
def test_schedule_covers_every_op_once(n, ms, n0, mode, per_warp, warps):
    _, plans = _plans(n, ms, n0)
    pk = pack_plans(plans)
    for d, bounds in ((0, pk.stages_fwd), (1, pk.stages_inv)):
        recs, bund, stage = chain_schedule(pk, d, warps=warps, mode=mode, per_warp=per_warp)
        covered = 0
        for s in range(len(bounds) - 1):
            b0, nb, nrec, nfold = (int(v) for v in stage[s])
            tasks = pk.tasks[bounds[s]:bounds[s + 1]]
            nops = int(tasks["op_count"].sum())
            flags = np.concatenate([pk.ops["flags"][t["op_begin"]:t["op_begin"] + t["op_count"]]
                                    for t in tasks]) if len(tasks) else np.zeros(0, np.uint8)
            small = bool(((flags & 3) != 0).any())
            if nb == 0:
                assert mode == 1 and not small or len(tasks) == 0
                continue
            assert mode == 2 or small
            assert nb == min(len(tasks), warps * per_warp)
            bs = bund[b0:b0 + nb + 1]
            assert np.all(np.diff(bs) > 0) and bs[-1] - bs[0] == nrec
            r = recs[bs[0]:bs[-1]]
            assert nrec + nfold == nops
            # a fold of more than 32 entries is two index adds on one record
            fl = (r["flags"] & EMU.CF_ADD) != 0
            assert int(fl.sum()) + int((r["addR"][fl] > 32).sum()) == nfold
            last = (r["flags"] & EMU.CF_LAST) != 0
            assert int(last.sum()) == len(tasks)
            # every bundle ends on a task end; every task's outputs appear once
            assert np.all(last[bs[1:] - bs[0] - 1])
            got = sorted(zip(r["out"][last].tolist(), r["nout"][last].tolist()))
            assert got == sorted(zip(tasks["out"].tolist(), tasks["nout"].tolist()))
            # folded adds sit on tile ops whose slot tail is free
            f = r[(r["flags"] & EMU.CF_ADD) != 0]
            assert np.all(f["kind"] != EMU.OP_ADD)
            blk = ((f["R"].astype(int) + 3) // 4) * ((f["C"].astype(int) + 3) // 4) * 16
            assert np.all(f["addR"] <= 64)
            assert np.all(blk <= np.where(f["addR"] > 32, 768, 896))
            covered += 1
        assert covered > 0 or (mode == 1 and n < 256)
        if n == 512:
            assert int(stage[:, 3].sum()) > 0   # folded adds are exercised


@pytest.mark.parametrize("n,ms,n0", [(256, [0, 300], 32), (512, [1], 512)])
def test_chain_records_emulate_bitwise_like_tasks(n, ms, n0):
    q, plans = _plans(n, ms, n0)
    pk = pack_plans(plans)
    rng = np.random.default_rng(n)
    for d in (0, 1):
        base = rng.standard_normal((pk.stats["arena"], NRHS))
        a0 = base.copy()
        EMU.run_direction(pk, a0, d)
        for mode, per_warp in ((1, 8), (2, 3)):
            a1 = base.copy()
            EMU.run_direction(pk, a1, d, chain=chain_schedule(pk, d, warps=24, mode=mode,
                                                              per_warp=per_warp))
            assert np.array_equal(a0, a1)


def test_chain_schedule_through_alt_orders_matches_oracle():
    n, ms, n0 = 256, [0, 1], 32
    q, plans = _plans(n, ms, n0)
    pk = pack_plans(plans)
    rng = np.random.default_rng(1)
    vecs = [rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m) for m in ms]
    sched = chain_schedule(pk, 0, warps=24, mode=2)
    orig = EMU.run_direction
    try:
        EMU.run_direction = lambda pk_, arena, d: orig(pk_, arena, d, chain=sched if d == 0 else None)
        got = EMU.alt_orders(pk, plans, 0, vecs)
    finally:
        EMU.run_direction = orig
    for g, p, v in zip(got, plans, vecs):
        want = OA.alt_forward(p, v)
        assert np.linalg.norm(g - want) <= 1e-14 * np.linalg.norm(want)


def test_chain_schedule_rejects_bad_arguments():
    _, plans = _plans(32, [20], 16)
    pk = pack_plans(plans)
    with pytest.raises(RuntimeError):
        chain_schedule(pk, 0, warps=0)
