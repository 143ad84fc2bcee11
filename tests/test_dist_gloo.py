"""Order-sharded SHT host logic on CPU: world_size 2 over gloo.

Each rank plans and packs only its LPT share of the orders, runs the ALT
through the numpy interpreter of the packed format (packed_emulator), and
exchanges node-half entries exactly as the native sharded transform does
(csrc/comm.cu bfsht_sharded_forward / _inverse): the send buffer is the
rank's row-major node array Yr itself (each peer's rows one contiguous
run), the receive layout and per-peer counts come from the C ABI's host
function bfsht_exchange_layout (through dist.ExchangePlan), and the inverse
lands in the Yr region before the Yr -> m-major node-half move.  The
transport is a gloo all_to_all_single with the same counts as the grouped
ncclSend/ncclRecv.  The DFT stage is numpy on the rank's row pairs.  Results
must match the CPU oracle's full transform on every rank's shard.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import packed_emulator as EMU

N = 16
WORLD = 2


def _flat(n, seed):
    rng = np.random.default_rng(seed)
    parts = []
    for m in range(-(2 * n - 1), 2 * n):
        ln = 2 * n - abs(m)
        parts.append(rng.standard_normal(ln) + 1j * rng.standard_normal(ln))
    return np.concatenate(parts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _check_rank(rank, world)
    finally:
        dist.destroy_process_group()


def _check_rank(rank, world):
    import oracle.apply as OA
    from paper_2004_11346_b200 import gauss_legendre, plan_orders, plan_sht
    from paper_2004_11346_b200.dist import ExchangePlan, _flat_offset, lpt_orders
    from paper_2004_11346_b200.pack import pack_plans

    n = N
    L = 4 * n - 1
    q = gauss_legendre(2 * n)
    orders = lpt_orders(n, world)[rank]
    plans = plan_orders(n, orders, n0=8, processes=1, quadrature=q)
    pk = pack_plans(plans)
    xp = ExchangePlan(n, world, rank, pk.halves, int(pk.info[10]))
    flat = _flat(n, 11)
    full = plan_sht(n, n0=8)
    want_grid = OA.sht_forward(full.alt_plans, n, flat)
    want_back = OA.sht_inverse(full.alt_plans, n, want_grid)

    # ---- forward: shard pack -> ALT -> all-to-all -> row-pair DFT
    arena = np.zeros((pk.stats["arena"], 4))
    h = pk.halves
    for o, m in enumerate(orders):
        cp = flat[_flat_offset(n, m):_flat_offset(n, m) + 2 * n - m]
        cm = flat[_flat_offset(n, -m):_flat_offset(n, -m) + 2 * n - m] if m \
            else np.zeros(2 * n)
        for par in range(2):
            hf = h[2 * o + par]
            if hf["ncols"]:
                k = slice(1 if par == 0 else 0, None, 2)
                a, b = cp[k][:hf["ncols"]], cm[k][:hf["ncols"]]
                arena[hf["x"]:hf["x"] + hf["ncols"]] = np.stack(
                    [a.real, a.imag, b.real, b.imag], 1)
    EMU.run_direction(pk, arena, 0)
    yr, wy = xp.yr, xp.w
    assert sum(xp.send_counts) == n * wy
    send = torch.from_numpy(arena[yr:yr + n * wy].copy())   # Yr rows, peer after peer
    recv = torch.zeros((xp.recv_entries, 4), dtype=torch.float64)
    dist.all_to_all_single(recv.view(-1), send.view(-1),
                           [c * 4 for c in xp.recv_counts],
                           [c * 4 for c in xp.send_counts])
    rv = recv.numpy()
    phi0 = np.pi / L
    local = np.zeros((2 * xp.rc, L), dtype=np.complex128)
    for rr in range(xp.rc):
        r = xp.r0 + rr
        up = np.zeros(L, complex)
        lo = np.zeros(L, complex)
        for b in range(L):
            m = b if b <= 2 * n - 1 else b - L
            sel = 0 if m >= 0 else 2
            g = {}
            for par in range(2):
                hf = xp.recv_layout[2 * abs(m) + par]
                e = rv[hf["y"] + rr * hf["x"]] if hf["ncols"] else np.zeros(4)
                g[par] = e[sel] + 1j * e[sel + 1]
            t = np.exp(1j * m * phi0)
            up[b] = (g[1] + g[0]) * t
            lo[b] = (g[1] - g[0]) * t
        local[xp.rc + rr] = L * np.fft.ifft(up)
        local[xp.rc - 1 - rr] = L * np.fft.ifft(lo)
    r0, r1 = xp.r0, xp.r0 + xp.rc
    want_local = np.concatenate([want_grid[n - r1:n - r0], want_grid[n + r0:n + r1]])
    assert np.linalg.norm(local - want_local) <= 1e-13 * np.linalg.norm(want_local)

    # ---- inverse: row-pair DFT + fold -> all-to-all back -> ALT^T -> unpack
    ubuf = np.zeros((xp.recv_entries, 4))
    w = q.weights
    for rr in range(xp.rc):
        r = xp.r0 + rr
        su = np.fft.fft(want_local[xp.rc + rr]) / L
        sl = np.fft.fft(want_local[xp.rc - 1 - rr]) / L
        for b in range(L):
            m = b if b <= 2 * n - 1 else b - L
            sel = 0 if m >= 0 else 2
            t = np.exp(-1j * m * phi0)
            a, c = su[b] * t, sl[b] * t
            for par, v in ((0, w[n + r] * (a - c)), (1, w[n + r] * (a + c))):
                hf = xp.recv_layout[2 * abs(m) + par]
                if hf["ncols"]:
                    ubuf[hf["y"] + rr * hf["x"], sel:sel + 2] = (v.real, v.imag)
    back_send = torch.zeros((sum(xp.send_counts), 4), dtype=torch.float64)
    dist.all_to_all_single(back_send.view(-1), torch.from_numpy(ubuf).view(-1),
                           [c * 4 for c in xp.send_counts],
                           [c * 4 for c in xp.recv_counts])
    arena[:] = 0.0
    arena[yr:yr + n * wy] = back_send.numpy()       # back into the Yr region
    dst = xp.yr_to_halves()                          # yr_to_halves_kernel
    keep = dst >= 0
    arena[dst[keep]] = arena[yr:yr + n * wy][keep]
    EMU.run_direction(pk, arena, 1)
    for o, m in enumerate(orders):
        for sign in ((1, -1) if m else (1,)):
            mm = sign * m
            got = np.zeros(2 * n - m, complex)
            sel = 0 if sign > 0 else 2
            for par in range(2):
                hf = h[2 * o + par]
                if hf["ncols"]:
                    e = arena[hf["x"]:hf["x"] + hf["ncols"]]
                    got[(1 if par == 0 else 0)::2] = e[:, sel] + 1j * e[:, sel + 1]
            start = _flat_offset(n, mm)
            ref = want_back[start:start + 2 * n - m]
            assert np.linalg.norm(got - ref) <= 1e-12 * max(np.linalg.norm(ref), 1e-300)


def test_sharded_sht_gloo_world2():
    mp.spawn(_worker, args=(WORLD, _free_port()), nprocs=WORLD, join=True)


def test_lpt_and_rows_cover():
    from paper_2004_11346_b200.dist import lpt_orders, row_split
    for n, world in ((16, 2), (1024, 8), (4096, 8), (64, 3)):
        parts = lpt_orders(n, world)
        assert sorted(m for p in parts for m in p) == list(range(2 * n))
        loads = [sum(2 * n - m for m in p) for p in parts]
        assert max(loads) / (sum(loads) / world) < 1.01
        rows = row_split(n, world)
        assert rows[0][0] == 0 and rows[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))


def test_native_lpt_and_layout_match_host():
    # the C ABI's host-side shard / layout functions (used by the native
    # sharded transform) against the Python restatement
    import ctypes
    from paper_2004_11346_b200 import native
    from paper_2004_11346_b200.dist import half_cols, lpt_orders, row_split
    from paper_2004_11346_b200.pack import HALF_DTYPE
    lib = native.cuda()
    for n, world in ((16, 2), (64, 3), (1024, 8), (4096, 8), (8, 1)):
        parts = lpt_orders(n, world)
        for rank in range(world):
            buf = np.zeros(2 * n, dtype=np.int32)
            cnt = ctypes.c_int32()
            assert lib.bfsht_shard_orders(n, world, rank, buf.ctypes.data,
                                          ctypes.addressof(cnt)) == 0
            assert list(buf[:cnt.value]) == parts[rank]
        rank = world - 1
        lay = np.zeros(4 * n, dtype=HALF_DTYPE)
        sc = np.zeros(world, dtype=np.int64)
        rc = np.zeros(world, dtype=np.int64)
        assert lib.bfsht_exchange_layout(n, world, rank, lay.ctypes.data, sc.ctypes.data,
                                         rc.ctypes.data) == 0
        rows = row_split(n, world)
        w = 2 * len(parts[rank])
        assert list(sc) == [(b - a) * w for a, b in rows]
        mine = rows[rank][1] - rows[rank][0]
        assert list(rc) == [mine * 2 * len(p) for p in parts]
        pos = 0
        for s_, p in enumerate(parts):
            for i, m in enumerate(p):
                for par in range(2):
                    hf = lay[2 * m + par]
                    assert (hf["m"], hf["ncols"], hf["x"], hf["y"]) == \
                        (m, half_cols(n, m, par), 2 * len(p), pos + 2 * i + par)
            pos += rc[s_]


def test_exchange_plan_rejects_wrong_halves():
    from paper_2004_11346_b200 import plan_orders
    from paper_2004_11346_b200.dist import ExchangePlan, lpt_orders
    from paper_2004_11346_b200.pack import pack_plans
    orders = lpt_orders(8, 2)[0]
    pk = pack_plans(plan_orders(8, orders, n0=8, processes=1))
    ExchangePlan(8, 2, 0, pk.halves, int(pk.info[10]))
    with pytest.raises(ValueError):
        ExchangePlan(8, 2, 1, pk.halves, int(pk.info[10]))
