"""SHT runners: one GPU, or orders sharded over the GPUs of one node.

Sharding: the independent unit is the order |m| — its plan
serves +m and -m (pkg/src/bfsht/sht.py:146,165) — so each rank plans,
packs and applies the ALT for its own orders only (greedy LPT on the
per-order cost proxy 2N-|m|).  The phi DFT needs every order of a
colatitude row (sht.py:148,161), so each direction has exactly one exchange:
an NCCL all-to-all that transposes node-half entries between the m-major
ALT layout (owner of m) and the theta-major DFT layout (owner of row pairs
r, n+r / n-1-r).  The forward sends straight from the row-major node array
(each peer's rows are one contiguous run); the inverse sends them back and
one kernel moves each entry to its m-major node half.

The exchange runs in the C ABI (csrc/comm.cu: bfsht_comm_init,
bfsht_alltoall_transpose, bfsht_sharded_forward / _inverse) over its own
NCCL communicator; torch.distributed only carries the NCCL unique id and
the max-over-ranks timing.

Both runners expose the same interface to bench.py / smoke():
forward(coeffs, grid), inverse(grid, coeffs), time_alt, time_e2e, ...
"""
import ctypes

import numpy as np

from ._capi import check
from .pack import HALF_DTYPE

FORWARD, INVERSE = 0, 1


def lpt_orders(n, world):
    """Greedy LPT assignment of orders 0..2N-1 to ``world`` ranks on the
    proxy cost 2N - m (corr. 0.99 with payload bytes)."""
    loads = [0.0] * world
    out = [[] for _ in range(world)]
    for m in range(2 * n):  # descending cost order
        r = min(range(world), key=lambda i: (loads[i], i))
        out[r].append(m)
        loads[r] += 2 * n - m
    return [sorted(o) for o in out]


def row_split(n, world):
    """Row pairs r in [0, n) split into contiguous near-equal ranges."""
    return [(q * n // world, (q + 1) * n // world) for q in range(world)]


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream(torch, device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class ExchangePlan:
    """Host view of one rank's exchange (the layout the C ABI computes,
    bfsht_exchange_layout in csrc/comm.cu; no device code).

    Forward: the entries for peer q are this rank's Yr rows [a_q, b_q) —
    one contiguous run of the row-major node array Yr[r][order][parity]
    (arena entries yr + r * w + h, w = 2 x len(orders)) — sent back to back
    in peer order (send_counts).  The receiver keeps the sources' runs back
    to back: entry (m, parity, r) sits at recv_layout[2m+parity].y +
    (r - r0) * recv_layout[2m+parity].x, the addressing the DFT kernels
    take.  Inverse: the same runs travel back into the Yr region, and entry
    yr + r * w + h moves to the m-major node half halves[h].y + r that the
    inverse ALT reads (yr_to_halves).
    """

    def __init__(self, n, world, rank, halves, yr):
        from . import native
        lib = native.cuda()
        self.n, self.world, self.rank = n, world, rank
        self.all_orders = lpt_orders(n, world)
        self.orders = self.all_orders[rank]
        self.rows = row_split(n, world)
        self.r0 = self.rows[rank][0]
        self.rc = self.rows[rank][1] - self.r0
        h = np.asarray(halves)
        if len(h) != 2 * len(self.orders) or \
                list(h["m"][0::2]) != list(self.orders):
            raise ValueError("halves do not match this rank's orders")
        self.yr, self.w = int(yr), 2 * len(self.orders)
        self.halves = h
        self.recv_layout = np.zeros(4 * n, dtype=HALF_DTYPE)
        sc = np.zeros(world, dtype=np.int64)
        rcnt = np.zeros(world, dtype=np.int64)
        check(lib, lib.bfsht_exchange_layout(n, world, rank, self.recv_layout.ctypes.data,
                                             sc.ctypes.data, rcnt.ctypes.data),
              "bfsht_exchange_layout")
        self.send_counts = [int(v) for v in sc]
        self.recv_counts = [int(v) for v in rcnt]
        self.recv_entries = int(rcnt.sum())
        offs, at = [], 0
        for m in self.orders:
            offs.append(at)
            at += (2 * n - m) * (2 if m else 1)
        self.coeff_offsets = np.array(offs + [at], dtype=np.int64)
        self.coeff_len = at

    def yr_to_halves(self):
        """For every Yr entry (row-major, r then h) of this rank: the arena
        entry of its m-major node half (-1 for an absent half)."""
        ys = np.where(self.halves["ncols"] > 0, self.halves["y"], -1).astype(np.int64)
        r = np.arange(self.n, dtype=np.int64)[:, None]
        return np.where(ys[None, :] >= 0, ys[None, :] + r, -1).ravel()


def half_cols(n, m, par):
    """Columns of the (m, parity) half; 0 when absent (alt.py:102-107)."""
    half = (m + 1) // 2 if par == 0 else m // 2
    return max(n - half, 0)


class _Common:
    def launches_total(self):
        return int(self.dp.lib.bfsht_plan_launches(self.dp.handle))

    def alt_bytes(self):
        """Algorithmic ALT bytes per direction on this rank: every stored
        payload value once (8 B) + coefficient-half and node-half entries
        once (4 x 8 B each)."""
        h = self.dp.packed.halves
        present = h["ncols"] > 0
        entries = int(h["ncols"][present].sum()) + int(present.sum()) * self.n
        return 8 * self.dp.packed.stats["payload_values"] + 32 * entries

    def hbm_bytes(self):
        """Bytes the ALT stages actually stream per direction: like
        alt_bytes, but regenerated tiles count their seed blocks instead
        of their values (B_ALT with and without them)."""
        pk = self.dp.packed
        return self.alt_bytes() - 8 * pk.stats["regen_values"] + pk.seed_bytes()

    def time_alt(self, reps=3):
        import torch
        out = {}
        for name, d in (("fwd_ms", FORWARD), ("inv_ms", INVERSE)):
            self.dp.alt_apply(d)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                self.dp.alt_apply(d)
            e1.record()
            torch.cuda.synchronize()
            out[name] = e0.elapsed_time(e1) / reps
        return out

    def time_e2e(self, flat, steps, warmup, barrier, lag=3, depth=4):
        """Host API end to end: pinned host coefficients -> host grid ->
        host coefficients for every step, through api.HostPipeline (copies
        on their own streams, overlapped with other steps' transforms).

        Step j = forward(h_c[j]) into h_g[j], then inverse(h_g[j]) into
        h_b[j]; forwards run `lag` steps ahead of inverses so the compute
        stream has work while a grid travels device -> host -> device.
        Every step's copies are inside the timed region (pipeline fill and
        drain included)."""
        import torch
        from .api import HostPipeline
        c, g, _ = self.make_buffers(flat)
        coeff_shape, grid_shape = tuple(c.shape), tuple(g.shape)
        if hasattr(self, "shard_coeffs"):
            host0 = torch.from_numpy(np.ascontiguousarray(self.shard_coeffs(flat)))
        else:
            host0 = torch.from_numpy(np.ascontiguousarray(self.host_coeffs(flat)))
        nbuf = lag + 2
        h_c = [host0.clone().pin_memory() for _ in range(nbuf)]
        h_g = [torch.empty(grid_shape, dtype=torch.complex128).pin_memory()
               for _ in range(nbuf)]
        h_b = [torch.empty(coeff_shape, dtype=torch.complex128).pin_memory()
               for _ in range(nbuf)]
        del c, g
        pipe = HostPipeline(self.forward, self.inverse, self.dp.device,
                            coeff_shape, grid_shape, depth)

        def run(count):
            for i in range(count + lag):
                if i < count:
                    k = i % nbuf
                    pipe.forward(h_c[k], h_g[k])
                j = i - lag
                if j >= 0:
                    k = j % nbuf
                    pipe.inverse(h_g[k], h_b[k])

        run(warmup)
        pipe.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for s in (pipe.s_in, pipe.s_run, pipe.s_out):
            s.wait_stream(torch.cuda.current_stream())
        run(steps)
        for s in (pipe.s_in, pipe.s_run, pipe.s_out):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        barrier()
        nb_c = h_c[0].numel() * 16
        nb_g = h_g[0].numel() * 16
        self.last_e2e_output = h_b[(steps - 1) % nbuf]
        return {"ms": e0.elapsed_time(e1) / steps, "h2d": nb_c + nb_g,
                "d2h": nb_g + nb_c, "pipelined": {"lag": lag, "depth": depth}}


class SingleRunner(_Common):
    """Whole SHT on one GPU (plan holds every order)."""

    def __init__(self, sht_device, batch=1):
        self.dev = sht_device
        self.dp = sht_device.plan
        self.n = sht_device.n
        self.batch = int(batch)
        self._pinned = None

    def make_buffers(self, flat):
        """Device coefficients / grid / result; with batch B > 1 the same
        coefficient set is stacked B times (independent transforms)."""
        import torch
        dev = self.dp.device
        n = self.n
        c = torch.from_numpy(np.ascontiguousarray(flat)).to(dev)
        if self.batch > 1:
            c = c.unsqueeze(0).repeat(self.batch, 1).contiguous()
            g = torch.empty((self.batch, 2 * n, 4 * n - 1), dtype=torch.complex128, device=dev)
        else:
            g = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128, device=dev)
        return c, g, torch.empty_like(c)

    def host_coeffs(self, flat):
        if self.batch > 1:
            return np.ascontiguousarray(np.broadcast_to(flat, (self.batch, flat.size)))
        return flat

    def forward(self, coeffs, grid):
        if self.batch > 1:
            self.dp.sht_batch(FORWARD, coeffs, grid)
        else:
            self.dp.sht_forward(coeffs, grid)

    def inverse(self, grid, coeffs):
        if self.batch > 1:
            self.dp.sht_batch(INVERSE, grid, coeffs)
        else:
            self.dp.sht_inverse(grid, coeffs)

    def capture_step(self, coeffs, grid, back):
        """One forward + inverse on fixed device buffers as a CUDA graph:
        the ~35 launches and counter resets of a step replay without
        per-launch host work or stream gaps.  Returns (graph, launches
        per step).  The step is run once outside capture first, so every
        lazily built table and kernel attribute exists before capture."""
        import torch
        side = torch.cuda.Stream(self.dp.device)
        side.wait_stream(torch.cuda.current_stream(self.dp.device))
        with torch.cuda.stream(side):
            self.forward(coeffs, grid)
            self.inverse(grid, back)
        torch.cuda.current_stream(self.dp.device).wait_stream(side)
        torch.cuda.synchronize(self.dp.device)
        graph = torch.cuda.CUDAGraph()
        l0 = self.launches_total()
        with torch.cuda.graph(graph):
            self.forward(coeffs, grid)
            self.inverse(grid, back)
        return graph, self.launches_total() - l0

    def alt_bytes(self):
        if self.batch == 1:
            return _Common.alt_bytes(self)
        h = self.dp.packed.halves
        present = h["ncols"] > 0
        entries = int(h["ncols"][present].sum()) + int(present.sum()) * self.n
        return 8 * self.dp.packed.stats["payload_values"] + 128 * entries

    def time_alt(self, reps=3):
        if self.batch == 1:
            return _Common.time_alt(self, reps)
        import torch
        out = {}
        for name, d in (("fwd_ms", FORWARD), ("inv_ms", INVERSE)):
            self.dp.alt_apply_wide(d)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                self.dp.alt_apply_wide(d)
            e1.record()
            torch.cuda.synchronize()
            out[name] = e0.elapsed_time(e1) / reps
        return out

    def roundtrip_error(self, coeffs, grid, back):
        self.forward(coeffs, grid)
        self.inverse(grid, back)
        import torch
        return float(torch.linalg.norm(back - coeffs) / torch.linalg.norm(coeffs))

class ShardedSht(_Common):
    """Orders sharded over ranks, one NCCL exchange per direction — the
    native sharded transform of the C ABI (bfsht_sharded_forward /
    _inverse, csrc/comm.cu): its own NCCL communicator (bfsht_comm_init;
    torch.distributed only ships the unique id), grouped ncclSend/ncclRecv
    straight from the row-major node array.

    Data layout per rank: coefficients of its own orders (shard layout, see
    bfsht_shard_pack), and grid rows of its row pairs
    [r0, r1): rows n-r1..n-r0-1 then n+r0..n+r1-1.
    """

    def __init__(self, n, plans, orders, rank, world, group=None, regen=0.0, packed=None,
                 weights=None):
        import torch
        import torch.distributed as dist
        from .api import DevicePlan
        from .legendre import gauss_legendre
        self.torch, self.dist = torch, dist
        self.n, self.rank, self.world = n, rank, world
        self.group = group
        self.orders = list(orders)
        if weights is None:
            weights = plans[0].quadrature.weights if plans else gauss_legendre(2 * n).weights
        self.dp = DevicePlan(plans, weights=weights, regen=regen, packed=packed)
        lib = self.dp.lib
        self.lib = lib
        xp = ExchangePlan(n, world, rank, self.dp.packed.halves,
                          int(self.dp.packed.info[10]))
        self.xp = xp
        self.all_orders, self.rows = xp.all_orders, xp.rows
        self.r0, self.rc = xp.r0, xp.rc
        self.send_counts, self.recv_counts = xp.send_counts, xp.recv_counts
        self.recv_entries = xp.recv_entries
        self.coeff_len = xp.coeff_len
        self.weights = self.dp.weights
        # NCCL communicator of the C ABI: rank 0's unique id travels over
        # the torch process group, nothing else does
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            check(lib, lib.bfsht_comm_unique_id(uid), "bfsht_comm_unique_id")
        box = [uid.raw]
        if world > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        self.comm = ctypes.c_void_p()
        with torch.cuda.device(self.dp.device):
            check(lib, lib.bfsht_comm_init(uid, rank, world, ctypes.byref(self.comm)),
                  "bfsht_comm_init")
            self.handle = ctypes.c_void_p()
            check(lib, lib.bfsht_sharded_create(self.dp.handle, self.comm,
                                                ctypes.byref(self.handle)),
                  "bfsht_sharded_create")
        info = (ctypes.c_int64 * 4)()
        lib.bfsht_sharded_info(self.handle, info)
        if (info[0], info[1], info[2], info[3]) != (xp.r0, xp.rc, xp.coeff_len, xp.recv_entries):
            raise RuntimeError("native and host exchange layouts disagree")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.bfsht_sharded_free(self.handle)
            self.handle = None
        if getattr(self, "comm", None):
            self.lib.bfsht_comm_free(self.comm)
            self.comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def make_buffers(self, flat):
        torch = self.torch
        dev = self.dp.device
        c = torch.from_numpy(self.shard_coeffs(flat)).to(dev)
        g = torch.empty((2 * self.rc, 4 * self.n - 1), dtype=torch.complex128, device=dev)
        return c, g, torch.empty_like(c)

    # --------------------------------------------------------- transforms
    def forward(self, coeffs, grid):
        st = _stream(self.torch, self.dp.device)
        check(self.lib, self.lib.bfsht_sharded_forward(self.handle, _ptr(coeffs), _ptr(grid), st),
              "bfsht_sharded_forward")

    def inverse(self, grid, coeffs):
        st = _stream(self.torch, self.dp.device)
        check(self.lib, self.lib.bfsht_sharded_inverse(self.handle, _ptr(grid), _ptr(coeffs),
                                                       _ptr(self.weights), st),
              "bfsht_sharded_inverse")

    def shard_coeffs(self, flat):
        """This rank's coefficient shard from the full flat layout."""
        n = self.n
        parts = []
        for m in self.orders:
            for mm in ((m, -m) if m else (m,)):
                start = _flat_offset(n, mm)
                parts.append(flat[start:start + 2 * n - abs(mm)])
        return np.concatenate(parts)

    def unshard_coeffs(self, shard, total):
        """Shard-layout coefficients back into a flat ShtCoeffs.pack() array
        (orders of other ranks left zero)."""
        n = self.n
        out = np.zeros(total, dtype=np.complex128)
        at = 0
        for m in self.orders:
            for mm in ((m, -m) if m else (m,)):
                ln = 2 * n - abs(mm)
                start = _flat_offset(n, mm)
                out[start:start + ln] = shard[at:at + ln]
                at += ln
        return out

    def shard_grid(self, full):
        n = self.n
        r0, r1 = self.r0, self.r0 + self.rc
        return np.concatenate([full[n - r1:n - r0], full[n + r0:n + r1]])

    def roundtrip_error(self, coeffs, grid, back):
        torch = self.torch
        self.forward(coeffs, grid)
        self.inverse(grid, back)
        num = torch.linalg.norm(back - coeffs) ** 2
        den = torch.linalg.norm(coeffs) ** 2
        t = torch.stack([num, den])
        self.dist.all_reduce(t, group=self.group)
        return float((t[0] / t[1]).sqrt())


def _flat_offset(n, m):
    """Start of order m in ShtCoeffs.pack() (m ascending from -(2N-1))."""
    k = 2 * n
    if m <= 0:
        return (k + m - 1) * (k + m) // 2
    return (k - 1) * k // 2 + m * k - m * (m - 1) // 2
