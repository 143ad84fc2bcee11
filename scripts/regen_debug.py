"""Debug: regenerated-tile engine vs stored-tile engine, per order."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2004_11346_b200 import SamplingConfig, gauss_legendre, plan_orders
from paper_2004_11346_b200.api import DevicePlan, FORWARD
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
q = gauss_legendre(2 * n)
orders = list(range(0, 2 * n, 3)) + [2 * n - 1]
plans = plan_orders(n, orders, SamplingConfig(tolerance=1e-12), processes=0, quadrature=q)
base = DevicePlan(plans)
dp = DevicePlan(plans, regen=1.0)
print("mode", os.environ.get("BFSHT_REGEN_COLS"), "regen tiles", dp.packed.regen_tiles)
rng = np.random.default_rng(n)
vec = np.concatenate([rng.standard_normal(2 * n - m) + 1j * rng.standard_normal(2 * n - m) for m in orders])
x = torch.from_numpy(vec).cuda()
a = dp.alt_orders(FORWARD, x).cpu().numpy().reshape(len(orders), 2 * n)
b = base.alt_orders(FORWARD, x).cpu().numpy().reshape(len(orders), 2 * n)
bad = [(o, m) for o, m in enumerate(orders) if not np.array_equal(a[o], b[o])]
print("bad orders", len(bad), bad[:10])
if bad:
    o, m = bad[0]
    d = np.nonzero(a[o] != b[o])[0]
    print("order", m, "rows", d[:10], a[o][d[:3]], b[o][d[:3]])
