"""e2e (HostPipeline) throughput vs pipeline lag / depth and step count,
next to the device-resident step time of the same engine.  Plans come from
a BFPK cache when CACHE=dir is set."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, ShtDevice  # noqa: E402
from paper_2004_11346_b200.legendre import gauss_legendre  # noqa: E402
from paper_2004_11346_b200.pack import load_packed, pack_plans, save_packed  # noqa: E402
from paper_2004_11346_b200 import dist as D  # noqa: E402

n = 1024
cache = os.environ.get("CACHE")
path = os.path.join(cache, f"e2e_n{n}.bfpk") if cache else None
if path and os.path.exists(path):
    packed = load_packed(path)
else:
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
    packed = pack_plans(plans)
    if path:
        os.makedirs(cache, exist_ok=True)
        save_packed(packed, path)
eng = ShtDevice.__new__(ShtDevice)
eng.n = n
eng.plan = DevicePlan([], packed=packed, weights=gauss_legendre(2 * n).weights)
run = D.SingleRunner(eng)
flat = synthetic_coeffs(n)
c, g, b = run.make_buffers(flat)
for _ in range(3):
    run.forward(c, g)
    run.inverse(g, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    run.forward(c, g)
    run.inverse(g, b)
e1.record()
e1.synchronize()
print(json.dumps({"device_ms": e0.elapsed_time(e1) / 50}), flush=True)
for lag, depth in ((3, 4), (4, 5), (6, 7), (2, 3)):
    for k in (50, 100):
        r = run.time_e2e(flat, k, 3, torch.cuda.synchronize, lag=lag, depth=depth)
        print(json.dumps({"lag": lag, "depth": depth, "steps": k, "ms": r["ms"],
                          "sht_per_s": 1e3 / r["ms"]}), flush=True)
