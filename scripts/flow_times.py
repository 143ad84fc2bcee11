"""ALT time per direction, staged vs dataflow schedule, for several dataflow
gap lengths (BFSHT_FLOW_GAP, packing time); bitwise check between them."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan, FORWARD, INVERSE  # noqa: E402
from paper_2004_11346_b200.pack import pack_plans  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


n = int(os.environ.get("N", "1024"))
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
c = torch.from_numpy(synthetic_coeffs(n)).cuda()
ref = None
for gap in [int(g) for g in os.environ.get("GAPS", "3552").split(",")]:
    os.environ["BFSHT_FLOW_GAP"] = str(gap)
    dp = DevicePlan(plans, packed=pack_plans(plans), weights=plans[0].quadrature.weights)
    g = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128, device="cuda")
    b = torch.empty_like(c)
    for flow in (False, True):
        dp.set_schedule(flow)
        dp.sht_forward(c, g)
        dp.sht_inverse(g, b)
        torch.cuda.synchronize()
        if ref is None:
            ref = (g.clone(), b.clone())
        same = bool(torch.equal(ref[0], g) and torch.equal(ref[1], b))
        r = {"gap": gap, "flow": flow, "alt_fwd_ms": timed(lambda: dp.alt_apply(FORWARD)),
             "alt_inv_ms": timed(lambda: dp.alt_apply(INVERSE)),
             "step_ms": timed(lambda: (dp.sht_forward(c, g), dp.sht_inverse(g, b))),
             "bitwise_same": same}
        print(json.dumps(r), flush=True)
    del dp
    torch.cuda.empty_cache()
