"""Time the SHT's phi-DFT stage (synthesis / analysis kernels over all row
pairs, dft.cu) at N = 1024, 2048 (Bluestein), 4096, 8192 on random node
halves / grids, with CUDA events; one JSON line per (N, kernel) with the
algorithmic bytes (node-half entries read or written once, grid rows
written or read once) and the fraction of the measured HBM copy peak.
Also times N=1024's stage inside the whole-SHT path (Yr addressing) when
--sht is given (plans every order: ~10 s)."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_11346_b200.ooc import ChunkedSht  # noqa: E402


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


ap = argparse.ArgumentParser()
ap.add_argument("--n", default="1024,2048,4096,8192")
ap.add_argument("--sht", action="store_true")
args = ap.parse_args()
pk = peak()
for n in [int(v) for v in args.n.split(",")]:
    run = ChunkedSht(n, min(96, n), processes=1, only=[])
    L = 4 * n - 1
    lib, st = run.lib, run._stream()
    run.ybuf.normal_()
    grid = torch.randn((2 * n, L), dtype=torch.complex128, device="cuda")
    # node halves: every present (order, parity) half, n rows x 32 B
    lay = run.layout
    halves = int((lay["ncols"] > 0).sum())
    nbytes = halves * n * 32 + 2 * n * L * 16
    reps = 20 if n <= 2048 else 5
    for name, fn in (("synth", lambda: lib.bfsht_synth_rows(run.ctx.handle, _ptr(run.layout_dev),
                                                            _ptr(run.ybuf), 0, n, _ptr(grid), st)),
                     ("anal", lambda: lib.bfsht_anal_rows(run.ctx.handle, _ptr(run.layout_dev),
                                                          _ptr(run.ybuf), 0, n, _ptr(grid),
                                                          _ptr(run.weights), st))):
        ms = timed(fn, reps)
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"n": n, "L": L, "kernel": name, "ms": ms, "alg_bytes": nbytes,
                          "GBps": gbs, "frac_of_peak": gbs / pk}), flush=True)
    run.close()
    del grid, run
    torch.cuda.empty_cache()

if args.sht:
    from bench import synthetic_coeffs
    from paper_2004_11346_b200 import SamplingConfig, plan_orders
    from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE
    n = 1024
    L = 4 * n - 1
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
    dp = DevicePlan(plans)
    c = torch.from_numpy(synthetic_coeffs(n)).cuda()
    g = torch.empty((2 * n, L), dtype=torch.complex128, device="cuda")
    b = torch.empty_like(c)
    t_f = timed(lambda: dp.sht_forward(c, g), 10)
    t_i = timed(lambda: dp.sht_inverse(g, b), 10)
    a_f = timed(lambda: dp.alt_apply(FORWARD), 10)
    a_i = timed(lambda: dp.alt_apply(INVERSE), 10)
    print(json.dumps({"n": n, "sht_fwd_ms": t_f, "sht_inv_ms": t_i, "alt_fwd_ms": a_f,
                      "alt_inv_ms": a_i, "synth_plus_pack_ms": t_f - a_f,
                      "anal_plus_unpack_ms": t_i - a_i}), flush=True)
