"""Whole SHT on one GPU when the plan exceeds HBM: orders in chunks.

At N=4096 (BASELINE config 3) the packed payload is ~370 GB and even with
every turning tile regenerated (§8 f1) ~215 GB: more than one B200's
180 GB, and more than the GPU host's RAM.  Every order is an independent
unit, though (its plan serves +m and -m only, pkg/src/bfsht/sht.py:146,165),
so the transform can run chunk by chunk on one GPU: plan a chunk of orders
on the host (parallel processes), pack, upload, apply its ALT, copy its
node halves into a θ-major buffer that holds every order, release the
chunk.  The φ DFT stage then runs once over all rows (the same row-layout
kernels the sharded path uses, dist.py).  The inverse reverses the order:
analysis DFT into the θ-major buffer, then per chunk scatter → inverse ALT
→ unpack.

This is the sharded path of dist.py with the NCCL all-to-all replaced by
a local copy: chunk c plays the role of rank c (orders dealt by LPT on
2N-|m|), the single GPU owns every row pair.  Chunks that still fit when
the forward ends stay resident for the inverse; the others are planned
again (planning is deterministic, so the factors are the same).

Timing: every device step (shard pack, ALT stages, node-half copy, DFT
stages, unpack) is bracketed by CUDA events on the launching stream; the
sum is the device time of one transform direction with each chunk's
payload streamed from HBM — what a GPU holding the whole plan would
spend, up to per-stage tail effects of the smaller chunks.  Planning,
packing and upload are host work and reported separately.
"""
import sys
import time

import numpy as np

from ._capi import check
from .dist import FORWARD, INVERSE, _flat_offset, half_cols, lpt_orders
from .pack import HALF_DTYPE, NRHS


def _ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def chunk_layout(n, nchunks):
    """Chunks of orders (LPT on 2N-|m|) and the θ-major node-half layout.

    Chunk c's block of the buffer holds, for every row pair r, its
    2*len(orders) entries (order, parity) — exactly the chunk's forward
    node array Yr[r][order][parity], so moving it is one contiguous copy.
    Returns (chunks, layout, blocks, entries): layout[2m + parity] gives
    the entry of (m, parity, r) at y + r * x (the addressing of the DFT
    kernels' row path, bfsht_synth_rows / bfsht_anal_rows), blocks[c] =
    (first entry, count)."""
    chunks = [o for o in lpt_orders(n, nchunks) if o]
    layout = np.zeros(4 * n, dtype=HALF_DTYPE)
    blocks = []
    pos = 0
    for orders in chunks:
        w = 2 * len(orders)
        for i, m in enumerate(orders):
            for par in range(2):
                hf = layout[2 * m + par]
                hf["m"], hf["ncols"] = m, half_cols(n, m, par)
                hf["x"], hf["y"] = w, pos + 2 * i + par
        blocks.append((pos, n * w))
        pos += n * w
    return chunks, layout, blocks, pos


def scatter_index(halves, n):
    """Arena entry of every θ-major entry of a chunk (row-major over row
    pairs, (order, parity) within a row; -1 for an absent half): where the
    inverse ALT reads its node halves (the halves' y bases, row r at y + r)."""
    ys = np.where(halves["ncols"] > 0, halves["y"], -1).astype(np.int64)
    r = np.arange(n, dtype=np.int64)[:, None]
    return np.where(ys[None, :] >= 0, ys[None, :] + r, -1).ravel().astype(np.int32)


class _PackedSummary:
    """What a DevicePlan still reads from its packed plan after upload."""

    def __init__(self, pk):
        self.info = np.array(pk.info, copy=True)
        self.stats = dict(pk.stats)
        self.halves = np.array(pk.halves, copy=True)
        self.tile_bytes = int(pk.tiles.nbytes)
        self.n = pk.n

    def payload_bytes(self):
        return 8 * self.stats["payload_values"]


class ChunkedSht:
    """Forward / inverse SHT of size N on one GPU, orders in ``nchunks``
    chunks.  ``planner(orders) -> list[AltPlan]`` builds the factors of a
    chunk (default: ``plan_orders`` in ``processes`` host processes)."""

    def __init__(self, n, nchunks, params=None, tau=None, n0=None, processes=0,
                 planner=None, reserve_bytes=24 << 30, device=None, verbose=False,
                 only=None, regen=0.0):
        import torch
        from .api import DevicePlan
        from .legendre import gauss_legendre
        from .plan import TAU_DEFAULT, plan_orders
        self.torch = torch
        self.n = n
        self.nchunks = int(nchunks)
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        self.quadrature = gauss_legendre(2 * n)
        tau = TAU_DEFAULT if tau is None else tau
        if planner is None:
            def planner(orders):
                return plan_orders(n, orders, params, n0=n0, tau=tau,
                                   processes=processes, quadrature=self.quadrature)
        self.planner = planner
        self.reserve_bytes = int(reserve_bytes)
        # regen: fraction of full-height turning tiles stored as recurrence
        # seeds and regenerated on the GPU (§8 f1): ~4.7x fewer bytes for
        # those tiles, so more chunks stay resident between directions
        self.regen = float(regen)
        self.verbose = verbose
        # only: chunk indices to process (None = all).  A subset runs the
        # full-size grid and DFT stage with the other orders' node halves
        # zero: the transform of coefficients supported on those orders
        # (a sampled run when the whole plan is out of reach, e.g. N=8192).
        self.only = None if only is None else sorted(set(int(c) for c in only))
        self.chunks, self.layout, self.block, entries = chunk_layout(n, self.nchunks)
        dev = self.device
        self.ybuf = torch.zeros((entries, NRHS), dtype=torch.float64, device=dev)
        self.layout_dev = torch.from_numpy(self.layout.view(np.int32).copy()).to(dev)
        self.weights = torch.as_tensor(self.quadrature.weights, dtype=torch.float64,
                                       device=dev)
        # DFT-stage context: the plan of the single order 2N-1 (its handle
        # carries N and the DFT tables; its payload is one tiny block)
        self.ctx = DevicePlan(planner([2 * n - 1]), weights=self.quadrature.weights)
        self.lib = self.ctx.lib
        # build the DFT tables now (a zero-row call only prepares them), so
        # the first timed DFT stage does not include their setup
        check(self.lib, self.lib.bfsht_synth_rows(
            self.ctx.handle, _ptr(self.layout_dev), _ptr(self.ybuf), 0, 0,
            _ptr(self.ybuf), self._stream()), "bfsht_synth_rows")
        self.resident = {}

    # ------------------------------------------------------------ helpers
    def _stream(self):
        import ctypes
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def _chunk_plan(self, c):
        """DevicePlan of chunk c (resident, or planned + packed + uploaded)."""
        from .api import DevicePlan
        dp = self.resident.get(c)
        if dp is not None:
            return dp, 0.0, 0.0
        t0 = time.perf_counter()
        plans = self.planner(self.chunks[c])
        t1 = time.perf_counter()
        dp = DevicePlan(plans, weights=self.quadrature.weights, regen=self.regen)
        del plans
        self.torch.cuda.synchronize()
        # the device copy is all that is needed from here: drop the host
        # packed arrays (hundreds of GB over all chunks at N=4096)
        pk = dp.packed
        dp.packed = _PackedSummary(pk)
        pk.close()
        return dp, t1 - t0, time.perf_counter() - t1

    def _keep(self, c, dp):
        torch = self.torch
        free, _ = torch.cuda.mem_get_info(self.device)
        if free > self.reserve_bytes + 2 * dp.packed.tile_bytes:
            self.resident[c] = dp
            return True
        return False

    def _coeff_offsets(self, orders):
        offs, at = [], 0
        for m in orders:
            offs.append(at)
            at += (2 * self.n - m) * (2 if m else 1)
        return np.array(offs + [at], dtype=np.int64)

    def _shard(self, flat, orders):
        n = self.n
        parts = []
        for m in orders:
            for mm in ((m, -m) if m else (m,)):
                s = _flat_offset(n, mm)
                parts.append(flat[s:s + 2 * n - abs(mm)])
        return np.concatenate(parts)

    def _timed(self, key, fn):
        torch = self.torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        self._events.append((key, e0, e1))

    def _warm_dft(self, key, fn):
        """First launch of a DFT-stage kernel in this process, on one row
        pair and outside the timed events: the runtime loads the kernel's
        code lazily, and that host-side pause (about 25 ms for the analysis
        kernel, seen as a 34 ms analysis stage at N=4096 against 8.5 ms
        alone) otherwise sits between the stage's two events.  The timed call
        that follows writes the same rows again."""
        done = self.__dict__.setdefault("_dft_warm", set())
        if key in done:
            return
        fn()
        self.torch.cuda.synchronize()
        done.add(key)

    def _collect(self):
        self.torch.cuda.synchronize()
        out = {}
        for key, e0, e1 in self._events:
            out[key] = out.get(key, 0.0) + e0.elapsed_time(e1)
        self._events = []
        return out

    @staticmethod
    def alt_bytes(dp, n):
        h = dp.packed.halves
        present = h["ncols"] > 0
        entries = int(h["ncols"][present].sum()) + int(present.sum()) * n
        return 8 * dp.packed.stats["payload_values"] + 32 * entries

    # ---------------------------------------------------------- transforms
    def forward(self, flat, grid):
        """flat: host complex128 coefficients (ShtCoeffs.pack() layout);
        grid: device (2N, 4N-1) complex128.  Returns a report dict."""
        torch, lib = self.torch, self.lib
        n = self.n
        if self.only is not None:
            self.ybuf.zero_()   # orders outside the subset contribute nothing
        self._events = []
        rep = {"plan_s": 0.0, "pack_upload_s": 0.0, "alt_bytes": 0, "payload_values": 0,
               "chunks": []}
        for c, orders in enumerate(self.chunks):
            if self.only is not None and c not in self.only:
                continue
            dp, tp, tu = self._chunk_plan(c)
            rep["plan_s"] += tp
            rep["pack_upload_s"] += tu
            off = torch.from_numpy(self._coeff_offsets(orders)).to(self.device)
            coeffs = torch.from_numpy(self._shard(flat, orders)).to(self.device)
            st = self._stream()
            self._timed("pack", lambda: check(lib, lib.bfsht_shard_pack(
                dp.handle, _ptr(off), _ptr(coeffs), st), "bfsht_shard_pack"))
            self._timed(f"alt{c}", lambda: dp.alt_apply(FORWARD))
            yr = int(dp.packed.info[10])
            pos, cnt = self.block[c]
            self._timed("copy", lambda: self.ybuf[pos:pos + cnt].copy_(dp.arena[yr:yr + cnt]))
            ab = self.alt_bytes(dp, n)
            rep["alt_bytes"] += ab
            rep["payload_values"] += dp.packed.stats["payload_values"]
            rep["chunks"].append({"orders": len(orders), "alt_bytes": ab, "plan_s": tp,
                                  "pack_upload_s": tu, "resident": False})
            torch.cuda.synchronize()
            rep["chunks"][-1]["resident"] = self._keep(c, dp)
            rep["chunks"][-1]["tile_gb"] = dp.packed.tile_bytes / 1e9
            if self.verbose:
                free, total = torch.cuda.mem_get_info(self.device)
                print(f"[ooc] fwd chunk {c}: {len(orders)} orders, tiles "
                      f"{dp.packed.tile_bytes / 1e9:.1f} GB, arena "
                      f"{dp.arena.numel() * 8 / 1e9:.2f} GB, plan {tp:.1f} s, pack+upload "
                      f"{tu:.1f} s, resident {rep['chunks'][-1]['resident']}, device used "
                      f"{(total - free) / 1e9:.1f} GB", file=sys.stderr, flush=True)
            del dp, coeffs
            torch.cuda.empty_cache()
        free, total = torch.cuda.mem_get_info(self.device)
        rep["gpu_mem_used_gb"] = (total - free) / 1e9
        st = self._stream()
        self._warm_dft("synth", lambda: check(lib, lib.bfsht_synth_rows(
            self.ctx.handle, _ptr(self.layout_dev), _ptr(self.ybuf), 0, 1, _ptr(grid), st),
            "bfsht_synth_rows"))
        self._timed("dft", lambda: check(lib, lib.bfsht_synth_rows(
            self.ctx.handle, _ptr(self.layout_dev), _ptr(self.ybuf), 0, n, _ptr(grid), st),
            "bfsht_synth_rows"))
        t = self._collect()
        self._finish(rep, t)
        return rep

    def inverse(self, grid):
        """grid: device (2N, 4N-1) complex128 -> host flat coefficients
        (returned as rep["coeffs"])."""
        torch, lib = self.torch, self.lib
        n = self.n
        self._events = []
        st = self._stream()
        self._warm_dft("anal", lambda: check(lib, lib.bfsht_anal_rows(
            self.ctx.handle, _ptr(self.layout_dev), _ptr(self.ybuf), 0, 1, _ptr(grid),
            _ptr(self.weights), st), "bfsht_anal_rows"))
        self._timed("dft", lambda: check(lib, lib.bfsht_anal_rows(
            self.ctx.handle, _ptr(self.layout_dev), _ptr(self.ybuf), 0, n, _ptr(grid),
            _ptr(self.weights), st), "bfsht_anal_rows"))
        out = np.zeros(4 * n * n, dtype=np.complex128)
        rep = {"plan_s": 0.0, "pack_upload_s": 0.0, "alt_bytes": 0, "payload_values": 0,
               "chunks": [], "replanned": 0}
        order = sorted((c for c in range(len(self.chunks))
                        if self.only is None or c in self.only),
                       key=lambda c: c not in self.resident)
        for c in order:
            orders = self.chunks[c]
            replan = c not in self.resident
            dp, tp, tu = self._chunk_plan(c)
            rep["replanned"] += int(replan)
            rep["plan_s"] += tp
            rep["pack_upload_s"] += tu
            idx = torch.from_numpy(scatter_index(dp.packed.halves, n)).to(self.device)
            offs = self._coeff_offsets(orders)
            off = torch.from_numpy(offs).to(self.device)
            coeffs = torch.empty(int(offs[-1]), dtype=torch.complex128, device=self.device)
            pos, cnt = self.block[c]
            src = self.ybuf[pos:pos + cnt]
            st = self._stream()
            self._timed("copy", lambda: check(lib, lib.bfsht_scatter_entries(
                dp.handle, _ptr(idx), idx.numel(), _ptr(src), st), "bfsht_scatter_entries"))
            self._timed(f"alt{c}", lambda: dp.alt_apply(INVERSE))
            self._timed("pack", lambda: check(lib, lib.bfsht_shard_unpack(
                dp.handle, _ptr(off), _ptr(coeffs), st), "bfsht_shard_unpack"))
            ab = self.alt_bytes(dp, n)
            rep["alt_bytes"] += ab
            rep["payload_values"] += dp.packed.stats["payload_values"]
            host = coeffs.cpu().numpy()
            for i, m in enumerate(orders):
                a = int(offs[i])
                for mm in ((m, -m) if m else (m,)):
                    s = _flat_offset(n, mm)
                    ln = 2 * n - abs(mm)
                    out[s:s + ln] = host[a:a + ln]
                    a += ln
            rep["chunks"].append({"orders": len(orders), "alt_bytes": ab, "plan_s": tp,
                                  "pack_upload_s": tu, "replanned": replan})
            self.resident.pop(c, None)
            del dp, coeffs
            torch.cuda.empty_cache()
        t = self._collect()
        self._finish(rep, t)
        rep["coeffs"] = out
        return rep

    def _finish(self, rep, t):
        alt = sum(v for k, v in t.items() if k.startswith("alt"))
        rep["alt_ms"] = alt
        rep["dft_ms"] = t.get("dft", 0.0)
        rep["pack_ms"] = t.get("pack", 0.0)
        rep["copy_ms"] = t.get("copy", 0.0)
        rep["device_ms"] = alt + rep["dft_ms"] + rep["pack_ms"] + rep["copy_ms"]
        rep["alt_gbs"] = rep["alt_bytes"] / (alt * 1e-3) / 1e9 if alt > 0 else 0.0
        per = sorted((int(k[3:]), v) for k, v in t.items() if k.startswith("alt"))
        rep["alt_ms_per_chunk"] = [round(v, 3) for _, v in per]   # by chunk index

    def node_entries(self, m):
        """Host copy of order m's node-half entries in the θ-major buffer:
        (2 parities, N rows, 4 doubles) — Re/Im of +m then -m."""
        out = np.zeros((2, self.n, NRHS))
        for par in range(2):
            hf = self.layout[2 * m + par]
            if hf["ncols"] <= 0:
                continue
            y, x = int(hf["y"]), int(hf["x"])
            idx = y + x * np.arange(self.n)
            out[par] = self.ybuf[self.torch.from_numpy(idx).to(self.device)].cpu().numpy()
        return out

    def close(self):
        self.resident.clear()
        self.ctx.close()
