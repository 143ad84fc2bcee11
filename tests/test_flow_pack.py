"""Dataflow schedule emitted by the packer (packer.cpp build_flow): per
direction the claim order is a permutation of the direction's tasks, every
task with a dependency comes after every task of the stage it waits for,
chain stages wait for their predecessor, and the group tasks that wait are
exactly those reading an arena entry written on the GPU."""
import numpy as np
import pytest

from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_alt
from paper_2004_11346_b200.pack import pack_plans


@pytest.mark.parametrize("n,ms,n0", [(256, [0, 3, 100, 300, 511], 64), (128, [1, 64, 200, 255], 32)])
def test_flow_order_valid(n, ms, n0):
    q = gauss_legendre(2 * n)
    plans = [plan_alt(n, m, SamplingConfig(tolerance=1e-12), n0=n0, quadrature=q) for m in ms]
    pk = pack_plans(plans)
    assert pk.flow.size == pk.stats["tasks"]
    stage = pk.tinfo & 0xff
    dep = (pk.tinfo >> 8) - 1
    pos = 0
    for bounds in (pk.stages_fwd, pk.stages_inv):
        lo, hi = int(bounds[0]), int(bounds[-1])
        order = pk.flow[pos:pos + hi - lo]
        pos += hi - lo
        assert sorted(order.tolist()) == list(range(lo, hi))
        where = np.empty(hi - lo, np.int64)
        where[order - lo] = np.arange(hi - lo)
        for t in range(lo, hi):
            d = dep[t]
            if d < 0:
                continue
            members = np.arange(bounds[d], bounds[d + 1])
            assert members.size > 0
            assert where[members - lo].max() < where[t - lo], (t, d)
        # chain stages (below the group stage) depend on the previous non-empty stage
        nonempty = [s for s in range(len(bounds) - 1) if bounds[s + 1] > bounds[s]]
        for s in nonempty[1:]:
            t = int(bounds[s])
            if stage[t] == s and dep[t] >= 0:
                assert dep[t] < s
    # some group tasks are dependency-free (they read only inputs)
    assert (dep < 0).sum() > len(pk.stages_fwd)
