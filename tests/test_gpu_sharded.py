"""GPU: the order-sharded SHT path (ShardedSht) through NCCL, world size 1.

Exercises the multi-GPU code path end to end on one B200 — shard packing,
the gather / all-to-all / row-layout DFT / scatter sequence and the
row-pair grid layout — with a one-rank NCCL group (no ranks waiting on
each other).  The two-rank exchange itself is covered on CPU over gloo
(tests/test_dist_gloo.py).
"""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [16, 64])
def test_sharded_world1_matches_oracle(n):
    import torch
    import torch.distributed as dist

    import oracle.apply as OA
    from paper_2004_11346_b200 import plan_orders
    from paper_2004_11346_b200.dist import ShardedSht, lpt_orders

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}",
                            rank=0, world_size=1)
    try:
        orders = lpt_orders(n, 1)[0]
        plans = plan_orders(n, orders, n0=16, processes=1)
        run = ShardedSht(n, plans, orders, 0, 1)
        rng = np.random.default_rng(n)
        parts = []
        for m in range(-(2 * n - 1), 2 * n):
            ln = 2 * n - abs(m)
            parts.append(rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
        flat = np.concatenate(parts)
        c, g, b = run.make_buffers(flat)
        run.forward(c, g)
        run.inverse(g, b)
        torch.cuda.synchronize()
        want = OA.sht_forward(plans, n, flat)
        got = g.cpu().numpy()   # one rank: rows n-n..n-1 then n..2n-1 = full grid
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
        back = b.cpu().numpy()
        want_b = run.shard_coeffs(OA.sht_inverse(plans, n, got))
        assert np.linalg.norm(back - want_b) <= 1e-12 * np.linalg.norm(want_b)
        assert run.roundtrip_error(c, g, b) < 1e-12
    finally:
        dist.destroy_process_group()
