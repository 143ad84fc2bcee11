"""One forward + one inverse N=1024 SHT for ncu (no timing printed as a number
to trust: run the same command without ncu for that).  Launch order per
direction: coef pack, ALT stages (7 at N=1024), DFT kernel."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--tol", type=float, default=1e-12)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--regen", type=float, default=0.0)
a = ap.parse_args()
n = a.n
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=a.tol), processes=0)
dp = DevicePlan(plans, regen=a.regen)
print("stages fwd/inv", dp.stats["stages_fwd"], dp.stats["stages_inv"], flush=True)
c = torch.from_numpy(synthetic_coeffs(n)).cuda()
g = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128, device="cuda")
b = torch.empty_like(c)
for _ in range(a.reps):
    dp.sht_forward(c, g)
    dp.sht_inverse(g, b)
torch.cuda.synchronize()
err = float(torch.linalg.norm(b - c) / torch.linalg.norm(c))
print(f"roundtrip {err:.3e} launches {dp.launches()}", flush=True)
