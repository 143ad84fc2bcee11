"""e2e (HostPipeline) throughput vs number of timed steps: separates the
pipeline fill/drain from the steady state."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, ShtDevice  # noqa: E402
from paper_2004_11346_b200 import dist as D  # noqa: E402

n = 1024
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
eng = ShtDevice.__new__(ShtDevice)
eng.n = n
eng.plan = DevicePlan(plans, weights=plans[0].quadrature.weights)
run = D.SingleRunner(eng)
flat = synthetic_coeffs(n)
for lag, depth in ((2, 3), (1, 2), (3, 4)):
    for k in (10, 30):
        r = run.time_e2e(flat, k, 3, torch.cuda.synchronize, lag=lag, depth=depth)
        print(json.dumps({"lag": lag, "depth": depth, "steps": k, "ms": r["ms"],
                          "sht_per_s": 1e3 / r["ms"]}), flush=True)
