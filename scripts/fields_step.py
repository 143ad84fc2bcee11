"""One batched-fields forward ALT (all orders, F fields) at N=1024 for ncu.
With CACHE=dir the packed plan is loaded from / saved to a BFPK file, so a
run under ncu does not start the planner's process pool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, FORWARD  # noqa: E402
from paper_2004_11346_b200.pack import load_packed, pack_plans, save_packed  # noqa: E402

n = int(os.environ.get("N", "1024"))
nf = int(os.environ.get("F", "8"))
cache = os.environ.get("CACHE")
path = os.path.join(cache, f"fields_n{n}.bfpk") if cache else None
if path and os.path.exists(path):
    packed = load_packed(path)
else:
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
    packed = pack_plans(plans)
    if path:
        os.makedirs(cache, exist_ok=True)
        save_packed(packed, path)
dp = DevicePlan([], packed=packed)
x = torch.randn(dp.coeff_len, nf, dtype=torch.complex128, device="cuda")
out = dp.alt_fields(FORWARD, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    dp.alt_fields(FORWARD, x, out)
e1.record()
e1.synchronize()
print(f"F={nf} ms_per_call={e0.elapsed_time(e1) / 3:.3f}", flush=True)
