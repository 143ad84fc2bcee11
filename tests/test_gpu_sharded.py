"""GPU: the order-sharded SHT path through the C ABI's NCCL communicator
(bfsht_comm_init + bfsht_sharded_forward / _inverse, csrc/comm.cu), world
size 1.

Exercises the multi-GPU code path end to end on one B200 — shard packing,
the ALT, the grouped ncclSend/ncclRecv straight from the row-major node
array, the row-layout DFT, the Yr -> node-half move and the row-pair grid
layout — with a one-rank communicator (no ranks waiting on each other).
The two-rank exchange layout is covered on CPU over gloo
(tests/test_dist_gloo.py), with the same C ABI layout function.
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
        run.close()
    finally:
        dist.destroy_process_group()


def test_alltoall_transpose_world1():
    # bfsht_alltoall_transpose on its own: a one-rank grouped send/recv is a
    # device copy of the whole run
    import ctypes
    import torch
    from paper_2004_11346_b200 import native
    from paper_2004_11346_b200._capi import check
    lib = native.cuda()
    torch.cuda.set_device(0)
    uid = ctypes.create_string_buffer(128)
    check(lib, lib.bfsht_comm_unique_id(uid), "id")
    comm = ctypes.c_void_p()
    check(lib, lib.bfsht_comm_init(uid, 0, 1, ctypes.byref(comm)), "init")
    x = torch.randn(1000, 4, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    cnt = (ctypes.c_int64 * 1)(1000)
    check(lib, lib.bfsht_alltoall_transpose(comm, ctypes.c_void_p(x.data_ptr()), cnt,
                                            ctypes.c_void_p(y.data_ptr()), cnt, 4,
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
          "a2a")
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    lib.bfsht_comm_free(comm)
