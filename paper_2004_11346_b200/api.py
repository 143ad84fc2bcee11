"""Apply path on the B200: the reference's apply API over the C ABI.

Same names, argument meaning and ValueError messages as the reference
(pkg/src/bfsht/alt.py:264-282, sht.py:137-166):

    alt_forward(plan, coeffs)        -> GridFunctionColumn
    alt_inverse(plan, column)        -> CoeffVector
    idbf_apply(fac, x), idbf_apply_transpose(fac, y)   (butterfly.py:275-292)
    sht_forward(plan, coeffs)        -> ShtGridValues
    sht_inverse(plan, grid_values)   -> ShtCoeffs

``plan`` is an ``AltPlan`` / ``ShtPlan`` in the reference layout (from
``plan_alt`` / ``plan_sht`` of this package, or from ``bfsht``).  On first
use the plan is packed (csrc/packer.cpp) and uploaded once; the device
plan is cached on the plan object.  Host numpy inputs return host numpy
outputs like the reference; CUDA torch tensors stay on the device.

``DevicePlan`` is the lower-level handle (device arrays owned by torch, the
C ABI borrows them); ``ShtDevice`` runs whole transforms on device tensors.
There is no CPU fallback: without the CUDA library or a GPU every call
raises.
"""
import ctypes
from dataclasses import dataclass

import numpy as np

from . import native
from ._capi import check
from .pack import INFO_LEN, NRHS, pack_plans
from .sht import ShtCoeffs, ShtGridValues

FORWARD, INVERSE = 0, 1
WIDE_NRHS = 16   # BFSHT_WIDE_NRHS
FIELDS_NRHS = 64   # BFSHT_FIELDS_NRHS


@dataclass
class CoeffVector:
    """Coefficients for degrees k = m .. 2N-1, ascending; length 2N - m."""

    m: int
    values: np.ndarray


@dataclass
class GridFunctionColumn:
    """One order's profile at the 2N quadrature angles, node-ascending."""

    m: int
    values: np.ndarray


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2004_11346_b200 needs a CUDA device "
                           "(no CPU fallback)")
    return torch


def _stream_ptr(torch, stream=None, device=None):
    """The given stream, else the current stream OF THE PLAN'S DEVICE (the
    C ABI switches to the plan's device for the call)."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class DevicePlan:
    """A packed plan resident on one GPU.

    Device arrays (tile store, ops, indices, lane maps, tasks, halves, and
    the vector arena) are torch tensors; the native handle borrows them.
    """

    def __init__(self, plans, device=None, packed=None, weights=None, regen=0.0):
        torch = _torch()
        self.lib = native.cuda()
        plans = list(plans)
        self.packed = pack_plans(plans, regen=regen) if packed is None else packed
        pk = self.packed
        self.n = pk.n
        self.orders = [int(m) for m in pk.orders]
        self.device = torch.device("cuda", torch.cuda.current_device()
                                   if device is None else device)
        with torch.cuda.device(self.device):
            def up(a, dtype=None):
                t = torch.from_numpy(np.ascontiguousarray(a))
                if dtype is not None:
                    t = t.view(dtype)
                return t.to(self.device)

            self._dev = [
                up(pk.tiles if pk.tiles.size else np.zeros(2)),
                up(pk.ops.view(np.uint8) if pk.ops.size else np.zeros(24, np.uint8)),
                up(pk.idx if pk.idx.size else np.zeros(1, np.int32)),
                up(pk.maps if pk.maps.size else np.zeros(32, np.int8)),
                up(pk.tasks.view(np.int32) if pk.tasks.size else np.zeros(4, np.int32)),
                up(pk.halves.view(np.int32)),
                up(pk.rec if pk.rec.size else np.zeros(2)),
                up(pk.xpos if pk.xpos.size else np.zeros(2)),
            ]
            self.arena = torch.zeros((max(pk.stats["arena"], 1), NRHS),
                                     dtype=torch.float64, device=self.device)
            if weights is None and plans and hasattr(plans[0], "quadrature"):
                weights = plans[0].quadrature.weights
            self.weights = None if weights is None else \
                torch.as_tensor(np.asarray(weights, dtype=np.float64),
                                device=self.device)
            self._host_halves = np.ascontiguousarray(pk.halves)
            self._sf = np.ascontiguousarray(pk.stages_fwd)
            self._si = np.ascontiguousarray(pk.stages_inv)
            info = (ctypes.c_int64 * INFO_LEN)(*[int(v) for v in pk.info])
            host = (ctypes.c_void_p * 8)()
            if pk.ops.size and pk.tasks.size:
                # host copies of ops / tasks: the chain-stage schedule
                host[1] = pk.ops.ctypes.data
                host[4] = pk.tasks.ctypes.data
            host[5] = self._host_halves.ctypes.data
            host[6] = self._sf.ctypes.data
            host[7] = self._si.ctypes.data
            dev = (ctypes.c_void_p * 12)()
            for i, t in enumerate(self._dev[:6]):
                dev[i] = t.data_ptr()
            dev[6] = self.arena.data_ptr()
            dev[7] = self._dev[6].data_ptr()
            dev[8] = self._dev[7].data_ptr()
            h = ctypes.c_void_p()
            check(self.lib, self.lib.bfsht_plan_wrap(info, host, dev,
                                                     ctypes.byref(h)),
                  "bfsht_plan_wrap")
            self.handle = h
        self.coeff_len = sum(2 * self.n - m for m in self.orders)

    # ---------------------------------------------------------------- stats
    @property
    def stats(self):
        return self.packed.stats

    def payload_bytes(self):
        return self.packed.payload_bytes()

    def launches(self):
        return int(self.lib.bfsht_plan_launches(self.handle))

    def chain_info(self, direction, stage):
        """(bundles, op records, folded index adds) of one stage's chain
        schedule; bundles == 0: the stage runs on the stage kernel."""
        out = (ctypes.c_int64 * 3)()
        check(self.lib, self.lib.bfsht_plan_chain_info(self.handle, direction, stage, out),
              "bfsht_plan_chain_info")
        return tuple(int(v) for v in out)

    # -------------------------------------------------------------- apply
    def alt_apply(self, direction, stream=None):
        """All ALT stages over the arena (inputs already in place)."""
        torch = _torch()
        check(self.lib, self.lib.bfsht_alt_apply(
            self.handle, direction, _stream_ptr(torch, stream, self.device)), "bfsht_alt_apply")

    def alt_apply_wide(self, direction, stream=None):
        """All ALT stages over the wide (16-RHS) arena, inputs in place."""
        torch = _torch()
        check(self.lib, self.lib.bfsht_alt_apply_wide(
            self.handle, direction, ctypes.c_void_p(self.wide_arena().data_ptr()),
            _stream_ptr(torch, stream, self.device)), "bfsht_alt_apply_wide")

    def alt_orders(self, direction, inp, out=None, stream=None):
        """Per-order ALT on device complex128 tensors laid out plan after
        plan: forward in = coefficients (2N-m each), out = 2N node values;
        inverse the reverse."""
        torch = _torch()
        n2 = 2 * self.n
        inp = inp.contiguous()
        if out is None:
            size = len(self.orders) * n2 if direction == FORWARD else self.coeff_len
            out = torch.empty(size, dtype=torch.complex128, device=self.device)
        w = self.weights.data_ptr() if self.weights is not None else None
        check(self.lib, self.lib.bfsht_alt_orders(
            self.handle, direction, ctypes.c_void_p(inp.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(w),
            _stream_ptr(torch, stream, self.device)), "bfsht_alt_orders")
        return out

    def wide_arena(self):
        """Work arena of the batched calls (BFSHT_WIDE_NRHS doubles per
        entry), allocated on first use."""
        if getattr(self, "_wide", None) is None:
            torch = _torch()
            self._wide = torch.zeros((max(self.packed.stats["arena"], 1), WIDE_NRHS),
                                     dtype=torch.float64, device=self.device)
        return self._wide

    def fields_arena(self):
        """Work arena of alt_fields (BFSHT_FIELDS_NRHS doubles per entry),
        allocated on first use."""
        if getattr(self, "_fields", None) is None:
            torch = _torch()
            self._fields = torch.zeros((max(self.packed.stats["arena"], 1), FIELDS_NRHS),
                                       dtype=torch.float64, device=self.device)
        return self._fields

    def alt_fields(self, direction, inp, out=None, stream=None):
        """Batched-fields ALT: inp is a device complex128 (rows, F) tensor,
        rows laid out plan after plan (2N-m coefficient rows forward, 2N
        node rows inverse); one payload pass per 32 fields (8 when F <= 8
        or the plan regenerates tiles)."""
        torch = _torch()
        inp = inp.contiguous()
        if inp.dim() != 2:
            raise ValueError("alt_fields expects a (rows, fields) tensor")
        nf = inp.shape[1]
        rows = len(self.orders) * 2 * self.n if direction == FORWARD else self.coeff_len
        if out is None:
            out = torch.empty((rows, nf), dtype=torch.complex128, device=self.device)
        w = self.weights.data_ptr() if self.weights is not None else None
        check(self.lib, self.lib.bfsht_alt_fields(
            self.handle, direction, nf, ctypes.c_void_p(inp.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(w),
            ctypes.c_void_p(self.fields_arena().data_ptr()),
            _stream_ptr(torch, stream, self.device)), "bfsht_alt_fields")
        return out

    def sht_batch(self, direction, inp, out=None, stream=None):
        """B <= 4 independent whole transforms in one payload pass.
        FORWARD: inp (B, 4N^2) coefficients -> (B, 2N, 4N-1) grids;
        INVERSE: grids -> coefficients.  Bitwise equal to B single calls."""
        torch = _torch()
        n = self.n
        inp = inp.contiguous()
        nb = inp.shape[0]
        if out is None:
            shape = (nb, 2 * n, 4 * n - 1) if direction == FORWARD else (nb, 4 * n * n)
            out = torch.empty(shape, dtype=torch.complex128, device=self.device)
        w = self.weights.data_ptr() if self.weights is not None else None
        check(self.lib, self.lib.bfsht_sht_batch(
            self.handle, direction, int(nb), ctypes.c_void_p(inp.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(w),
            ctypes.c_void_p(self.wide_arena().data_ptr()),
            _stream_ptr(torch, stream, self.device)), "bfsht_sht_batch")
        return out

    def half_apply(self, direction, half, x, stream=None):
        """Matrix of one (order, parity) half on a device real (len, k)
        tensor: forward K x (len = half columns -> N rows), inverse K^T y."""
        torch = _torch()
        x = x.contiguous()
        h = self.packed.halves[half]
        n_out = self.n if direction == FORWARD else int(h["ncols"])
        out = torch.empty((n_out, x.shape[1]), dtype=torch.float64, device=self.device)
        check(self.lib, self.lib.bfsht_half_apply(
            self.handle, direction, int(half), int(x.shape[1]),
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(self.wide_arena().data_ptr()),
            _stream_ptr(torch, stream, self.device)), "bfsht_half_apply")
        return out

    def sht_forward(self, coeffs, out=None, stream=None):
        torch = _torch()
        n = self.n
        if out is None:
            out = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128,
                              device=self.device)
        check(self.lib, self.lib.bfsht_sht_forward(
            self.handle, ctypes.c_void_p(coeffs.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), _stream_ptr(torch, stream, self.device)),
            "bfsht_sht_forward")
        return out

    def sht_inverse(self, grid, out=None, stream=None):
        torch = _torch()
        n = self.n
        if out is None:
            out = torch.empty(4 * n * n, dtype=torch.complex128, device=self.device)
        check(self.lib, self.lib.bfsht_sht_inverse(
            self.handle, ctypes.c_void_p(grid.data_ptr()),
            ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(self.weights.data_ptr()),
            _stream_ptr(torch, stream, self.device)), "bfsht_sht_inverse")
        return out

    def close(self):
        if getattr(self, "handle", None):
            self.lib.bfsht_plan_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _device_plan(plan):
    dp = getattr(plan, "_b200_device_plan", None)
    if dp is None:
        dp = DevicePlan([plan])
        try:
            plan._b200_device_plan = dp
        except AttributeError:
            pass
    return dp


def _as_device(torch, values, dp):
    is_tensor = isinstance(values, torch.Tensor)
    if is_tensor:
        return values.to(dp.device, torch.complex128), True, values.is_complex()
    arr = np.asarray(values)
    cplx = np.iscomplexobj(arr)
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.complex128)) \
        .to(dp.device), False, cplx


def _shape_of(values):
    return tuple(values.shape)


def _finish(y, on_dev, cplx):
    if not on_dev:
        y = y.cpu().numpy()
        if not cplx:
            y = y.real.copy()
    elif not cplx:
        y = y.real.contiguous()
    return y


def _run_orders(plan, values, direction, want_rows):
    torch = _torch()
    dp = _device_plan(plan)
    x, on_dev, cplx = _as_device(torch, values, dp)
    if x.dim() == 1:
        y = dp.alt_orders(direction, x)
    else:
        y = dp.alt_fields(direction, x)
    return _finish(y, on_dev, cplx)


def alt_forward(plan, coeffs):
    """Coefficients beta_k (k = m..2N-1) to values at the 2N nodes
    (reference alt.py:264-272).  Extension: a
    (2N-m, F) array applies F fields at once."""
    values = coeffs.values if isinstance(coeffs, CoeffVector) else coeffs
    if not hasattr(values, "shape"):
        values = np.asarray(values)
    shape = _shape_of(values)
    if not (shape == (2 * plan.n - plan.m,)
            or (len(shape) == 2 and shape[0] == 2 * plan.n - plan.m)):
        raise ValueError(f"expected {2 * plan.n - plan.m} coefficients, "
                         f"got shape {shape}")
    return GridFunctionColumn(m=plan.m, values=_run_orders(plan, values, FORWARD, 2 * plan.n))


def alt_inverse(plan, column):
    """Values at the 2N nodes back to coefficients via the weighted
    transpose (reference alt.py:275-282); (2N, F) arrays batch F fields."""
    values = column.values if isinstance(column, GridFunctionColumn) else column
    if not hasattr(values, "shape"):
        values = np.asarray(values)
    shape = _shape_of(values)
    if not (shape == (2 * plan.n,) or (len(shape) == 2 and shape[0] == 2 * plan.n)):
        raise ValueError(f"expected {2 * plan.n} node values, "
                         f"got shape {shape}")
    return CoeffVector(m=plan.m, values=_run_orders(plan, values, INVERSE, 2 * plan.n - plan.m))


class _FactorSpec:
    def __init__(self, num_cols):
        self.num_cols = num_cols


class _FactorBlock:
    def __init__(self, trim, payload):
        self.trim = trim
        self.payload = payload


class _FactorPlan:
    """A ButterflyFactorization dressed as a one-half plan for the packer:
    K (h x w) is the odd half of order 0 with N = h rows and w columns."""

    def __init__(self, fac):
        h, w = (int(v) for v in fac.shape)
        self.n, self.m = h, 0
        self.spec_odd, self.spec_even = _FactorSpec(w), None
        self.blocks_odd, self.blocks_even = [_FactorBlock((0, h, 0, w), fac)], []


def _factor_device(fac):
    dp = getattr(fac, "_b200_device_plan", None)
    if dp is None:
        dp = DevicePlan([_FactorPlan(fac)])
        try:
            fac._b200_device_plan = dp
        except AttributeError:
            pass
    return dp


def _factor_apply(fac, v, direction):
    torch = _torch()
    dp = _factor_device(fac)
    is_tensor = isinstance(v, torch.Tensor)
    if is_tensor:
        cplx = v.is_complex()
        t = v.to(dp.device)
    else:
        arr = np.asarray(v)
        cplx = np.iscomplexobj(arr)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dp.device)
    vec = t.dim() == 1
    t = t.reshape(t.shape[0], -1)
    k = t.shape[1]
    if cplx:
        t = torch.view_as_real(t.to(torch.complex128).contiguous()).reshape(t.shape[0], 2 * k)
    else:
        t = t.to(torch.float64)
    y = dp.half_apply(direction, 0, t)
    if cplx:
        y = torch.view_as_complex(y.reshape(y.shape[0], k, 2).contiguous())
    if vec:
        y = y.reshape(-1)
    return y if is_tensor else y.cpu().numpy()


def idbf_apply(fac, x):
    """y = K x through the butterfly factor chain on the GPU
    (reference butterfly.py:275-282); x is (w,) or (w, k)."""
    shape = tuple(x.shape) if hasattr(x, "shape") else np.asarray(x).shape
    if shape[0] != fac.shape[1]:
        raise ValueError(f"length {shape[0]} against shape {fac.shape}")
    return _factor_apply(fac, x, FORWARD)


def idbf_apply_transpose(fac, y):
    """x = K^T y (reference butterfly.py:285-292); y is (h,) or (h, k)."""
    shape = tuple(y.shape) if hasattr(y, "shape") else np.asarray(y).shape
    if shape[0] != fac.shape[0]:
        raise ValueError(f"length {shape[0]} against shape {fac.shape}")
    return _factor_apply(fac, y, INVERSE)


class ShtDevice:
    """Whole-transform handle: every order's plan resident on one GPU."""

    def __init__(self, sht_plan, device=None):
        self.n = sht_plan.n
        ms = [p.m for p in sht_plan.alt_plans]
        if ms != list(range(2 * self.n)):
            raise ValueError("ShtPlan must hold plans for m = 0..2N-1")
        self.plan = DevicePlan(sht_plan.alt_plans, device=device,
                               weights=sht_plan.quadrature.weights)

    def forward(self, coeffs, out=None, stream=None):
        return self.plan.sht_forward(coeffs, out, stream)

    def inverse(self, grid, out=None, stream=None):
        return self.plan.sht_inverse(grid, out, stream)

    def forward_batch(self, coeffs, out=None, stream=None):
        """(B, 4N^2) device coefficients, B <= 4 -> (B, 2N, 4N-1) grids."""
        return self.plan.sht_batch(FORWARD, coeffs, out, stream)

    def inverse_batch(self, grids, out=None, stream=None):
        """(B, 2N, 4N-1) device grids, B <= 4 -> (B, 4N^2) coefficients."""
        return self.plan.sht_batch(INVERSE, grids, out, stream)

    def pipeline(self, depth=3):
        """Host-buffer streaming handle (see HostPipeline)."""
        n = self.n
        return HostPipeline(
            lambda c, g: self.plan.sht_forward(c, g),
            lambda g, c: self.plan.sht_inverse(g, c),
            self.plan.device, (4 * n * n,), (2 * n, 4 * n - 1), depth)


class HostPipeline:
    """Whole transforms on pinned HOST buffers, streamed.

    ``forward(h_coeffs, h_grid)`` / ``inverse(h_grid, h_coeffs)`` enqueue
    one transform each and return an event that completes when the host
    output is written.  Every call copies its input host->device, runs the
    transform, and copies the result device->host, on three streams:

        h2d stream:     copy-in of job j+1 ...
        compute stream: transform of job j (the plan's one work arena, so
                        transforms are serialized in submission order)
        d2h stream:     copy-out of job j-1 ...

    so with several jobs in flight the PCIe traffic hides under the
    transforms.  Dependencies are CUDA events only: device buffers rotate
    through a ring of ``depth`` per shape and are reused after their last
    reader/writer finished, and host buffers are tracked by address (a
    copy-in waits for the copy-out that last wrote that host buffer, a
    copy-out waits for the copy-in that last read it), so chaining
    ``forward`` into ``inverse`` through the same host grid is safe without
    a host synchronization.  Host buffers must be pinned torch tensors
    (pageable memory would serialize the copies).
    """

    def __init__(self, run_forward, run_inverse, device, coeff_shape,
                 grid_shape, depth=3):
        torch = _torch()
        self.torch = torch
        self.run = {FORWARD: run_forward, INVERSE: run_inverse}
        self.device = device
        self.depth = int(depth)
        if self.depth < 1:
            raise ValueError("depth must be >= 1")
        with torch.cuda.device(device):
            self.s_in = torch.cuda.Stream(device)
            self.s_run = torch.cuda.Stream(device)
            self.s_out = torch.cuda.Stream(device)
            shapes = {"c": tuple(coeff_shape), "g": tuple(grid_shape)}
            self.pool = {k: [[torch.empty(s, dtype=torch.complex128, device=device),
                              None] for _ in range(self.depth)]
                         for k, s in shapes.items()}
        self.next = {"c": 0, "g": 0}
        self.shapes = shapes
        self.host_write = {}   # host address -> event of the copy-out writing it
        self.host_read = {}    # host address -> event of the copy-in reading it

    def _slot(self, kind):
        i = self.next[kind]
        self.next[kind] = (i + 1) % self.depth
        return self.pool[kind][i]

    def _check(self, t, kind, name):
        torch = self.torch
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise ValueError(f"{name} must be a host torch tensor")
        if not t.is_pinned():
            raise ValueError(f"{name} must be pinned (tensor.pin_memory())")
        if t.dtype != torch.complex128 or not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous complex128")
        if t.numel() != int(np.prod(self.shapes[kind])):
            raise ValueError(f"{name} has {t.numel()} values, expected "
                             f"{int(np.prod(self.shapes[kind]))}")

    def _submit(self, direction, h_in, h_out):
        torch = self.torch
        kin, kout = ("c", "g") if direction == FORWARD else ("g", "c")
        self._check(h_in, kin, "input")
        self._check(h_out, kout, "output")
        sin, sout = self._slot(kin), self._slot(kout)
        ev = lambda: torch.cuda.Event()   # noqa: E731
        # copy-in: after the last writer of the host buffer and the last
        # user of the device slot
        w = self.host_write.get(h_in.data_ptr())
        if w is not None:
            self.s_in.wait_event(w)
        if sin[1] is not None:
            self.s_in.wait_event(sin[1])
        with torch.cuda.stream(self.s_in):
            sin[0].view(-1).copy_(h_in.view(-1), non_blocking=True)
            e_in = ev()
            e_in.record(self.s_in)
        self.host_read[h_in.data_ptr()] = e_in
        # transform
        self.s_run.wait_event(e_in)
        if sout[1] is not None:
            self.s_run.wait_event(sout[1])
        with torch.cuda.stream(self.s_run):
            self.run[direction](sin[0], sout[0])
            e_run = ev()
            e_run.record(self.s_run)
        sin[1] = e_run
        # copy-out: after the last reader of the host buffer
        self.s_out.wait_event(e_run)
        r = self.host_read.get(h_out.data_ptr())
        if r is not None and h_out.data_ptr() != h_in.data_ptr():
            self.s_out.wait_event(r)
        with torch.cuda.stream(self.s_out):
            h_out.view(-1).copy_(sout[0].view(-1), non_blocking=True)
            e_out = ev()
            e_out.record(self.s_out)
        sout[1] = e_out
        self.host_write[h_out.data_ptr()] = e_out
        return e_out

    def forward(self, h_coeffs, h_grid):
        return self._submit(FORWARD, h_coeffs, h_grid)

    def inverse(self, h_grid, h_coeffs):
        return self._submit(INVERSE, h_grid, h_coeffs)

    def synchronize(self):
        for s in (self.s_in, self.s_run, self.s_out):
            s.synchronize()


def _sht_device(plan):
    dev = getattr(plan, "_b200_sht_device", None)
    if dev is None:
        dev = ShtDevice(plan)
        try:
            plan._b200_sht_device = dev
        except AttributeError:
            pass
    return dev


def sht_forward(plan, coeffs):
    """Coefficients to grid values f(theta_l, phi_j), shape 2N x (4N-1)
    (reference sht.py:137-148)."""
    n = plan.n
    if coeffs.n != n:
        raise ValueError(f"coefficient set is for N={coeffs.n}, plan N={n}")
    torch = _torch()
    dev = _sht_device(plan)
    flat = torch.from_numpy(np.ascontiguousarray(coeffs.pack(),
                                                 dtype=np.complex128))
    grid = dev.forward(flat.to(dev.plan.device))
    return ShtGridValues(n=n, values=grid.cpu().numpy())


def sht_inverse(plan, grid_values):
    """Grid values to coefficients (reference sht.py:151-166)."""
    n = plan.n
    values = grid_values.values if isinstance(grid_values, ShtGridValues) \
        else np.asarray(grid_values)
    if values.shape != (2 * n, 4 * n - 1):
        raise ValueError(f"expected grid shape {(2 * n, 4 * n - 1)}, "
                         f"got {values.shape}")
    torch = _torch()
    dev = _sht_device(plan)
    g = torch.from_numpy(np.ascontiguousarray(values, dtype=np.complex128))
    flat = dev.inverse(g.to(dev.plan.device))
    return ShtCoeffs.unpack(n, flat.cpu().numpy())


def dft_rows(x, inverse=False, stream=None):
    """Batched length-L DFT of the rows of a complex128 CUDA tensor:
    numpy fft(axis=1) (forward) or L*ifft(axis=1) (inverse)."""
    torch = _torch()
    lib = native.cuda()
    x = x.contiguous()
    out = torch.empty_like(x)
    rows, L = x.shape
    with torch.cuda.device(x.device):
        check(lib, lib.bfsht_dft_rows(L, rows, INVERSE if inverse else FORWARD,
                                      ctypes.c_void_p(x.data_ptr()),
                                      ctypes.c_void_p(out.data_ptr()),
                                      _stream_ptr(torch, stream, x.device)), "bfsht_dft_rows")
    return out
