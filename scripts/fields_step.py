"""One batched-fields forward pass (F=8, 16-RHS engine) at N=1024 for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, FORWARD  # noqa: E402

n = int(os.environ.get("N", "1024"))
nf = int(os.environ.get("F", "8"))
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
dp = DevicePlan(plans)
x = torch.randn(dp.coeff_len, nf, dtype=torch.complex128, device="cuda")
out = dp.alt_fields(FORWARD, x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    dp.alt_fields(FORWARD, x, out)
e1.record()
e1.synchronize()
print(f"F={nf} pass_ms={e0.elapsed_time(e1) / 3 / ((nf + 7) // 8):.3f}", flush=True)
