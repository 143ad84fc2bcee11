"""DFT-stage timing at N=1024 (CUDA events, no profiler): standalone batched
DFT (2048 rows x 4095) and the SHT synthesis / analysis kernels, obtained as
sht_forward/inverse minus the ALT stages."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, dft_rows, FORWARD, INVERSE  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


n = 1024
L = 4 * n - 1
x = torch.randn(2 * n, L, dtype=torch.complex128, device="cuda")
out = {"tag": os.environ.get("BFSHT_NVCC_FLAGS", "")}
out["dft_rows_fwd_ms"] = timed(lambda: dft_rows(x))
out["dft_rows_inv_ms"] = timed(lambda: dft_rows(x, inverse=True))
del x
for LL, rows in ((16383, 16384), (32767, 2048)):
    xl = torch.randn(rows, LL, dtype=torch.complex128, device="cuda")
    out[f"dft_rows_L{LL}_x{rows}_ms"] = timed(lambda: dft_rows(xl), reps=3)
    del xl
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
dp = DevicePlan(plans)
c = torch.from_numpy(synthetic_coeffs(n)).cuda()
g = torch.empty((2 * n, L), dtype=torch.complex128, device="cuda")
b = torch.empty_like(c)
t_f = timed(lambda: dp.sht_forward(c, g))
t_i = timed(lambda: dp.sht_inverse(g, b))
a_f = timed(lambda: dp.alt_apply(FORWARD))
a_i = timed(lambda: dp.alt_apply(INVERSE))
out.update({"sht_fwd_ms": t_f, "sht_inv_ms": t_i, "alt_fwd_ms": a_f, "alt_inv_ms": a_i,
            "synth_plus_pack_ms": t_f - a_f, "anal_plus_unpack_ms": t_i - a_i})
print(json.dumps(out), flush=True)
