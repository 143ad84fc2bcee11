"""GPU: a whole forward + inverse SHT captured as a CUDA graph
(dist.SingleRunner.capture_step, what bench.py times) replays to the same
bits as the direct calls, and matches the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_graph_replay_is_bitwise_direct():
    import torch
    import oracle.apply as OA
    from bench import synthetic_coeffs
    from paper_2004_11346_b200 import SamplingConfig, plan_orders
    from paper_2004_11346_b200 import dist as D
    from paper_2004_11346_b200.api import DevicePlan, ShtDevice

    n = 32
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), n0=16)
    eng = ShtDevice.__new__(ShtDevice)
    eng.n = n
    eng.plan = DevicePlan(plans, weights=plans[0].quadrature.weights)
    run = D.SingleRunner(eng)
    flat = synthetic_coeffs(n)
    c, g, b = run.make_buffers(flat)
    run.forward(c, g)
    run.inverse(g, b)
    torch.cuda.synchronize()
    g0, b0 = g.cpu().numpy(), b.cpu().numpy()
    graph, per_step = run.capture_step(c, g, b)
    assert per_step >= 4
    g.zero_()
    b.zero_()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), g0)
    assert np.array_equal(b.cpu().numpy(), b0)
    want = OA.sht_forward(plans, n, flat)
    assert np.linalg.norm(g0 - want) <= 1e-12 * np.linalg.norm(want)
