"""Sweep the chain/free SM split of the overlapped ALT schedule (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan  # noqa: E402
from paper_2004_11346_b200.dist import SingleRunner  # noqa: E402
from paper_2004_11346_b200.api import ShtDevice  # noqa: E402

n = int(os.environ.get("N", "1024"))
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
eng = ShtDevice.__new__(ShtDevice)
eng.n = n
eng.plan = DevicePlan(plans, weights=plans[0].quadrature.weights)
run = SingleRunner(eng)
dp = eng.plan
c, g, b = run.make_buffers(synthetic_coeffs(n))
ref = None
for overlap, chain in [(0, 0), (1, 30), (1, 40), (1, 50), (1, 59), (1, 70), (1, 85)]:
    dp.lib.bfsht_plan_tune(dp.handle, overlap, chain)
    run.forward(c, g)
    run.inverse(g, b)
    torch.cuda.synchronize()
    if ref is None:
        ref = (g.clone(), b.clone())
    same = bool(torch.equal(ref[0], g) and torch.equal(ref[1], b))
    t = run.time_alt(reps=5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run.forward(c, g)
        run.inverse(g, b)
    e1.record()
    torch.cuda.synchronize()
    print(f"overlap={overlap} chain={chain} alt_fwd={t['fwd_ms']:.3f} alt_inv={t['inv_ms']:.3f} "
          f"step={e0.elapsed_time(e1)/5:.3f} ms bitwise_same={same}", flush=True)
