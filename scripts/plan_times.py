"""Planning wall time with host vs device (f3) entry tabulation on a
sample of orders (default N=4096, 64 orders evenly spaced over 0..2N-1),
all host cores; digests of the two runs compared.  One JSON line."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from plan_digest import plan_digest  # noqa: E402

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--orders", type=int, default=64)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--processes", type=int, default=0)
    a = ap.parse_args()
    orders = np.linspace(0, 2 * a.n - 1, a.orders).round().astype(int).tolist()
    cfg = SamplingConfig(tolerance=a.tol)
    out = {"n": a.n, "orders": len(orders), "tol": a.tol, "cores": os.cpu_count()}
    digests = {}
    for name, dev in (("device", 0), ("host", None)):
        t0 = time.perf_counter()
        plans = plan_orders(a.n, orders, cfg, processes=a.processes, device=dev)
        out[f"{name}_s"] = time.perf_counter() - t0
        digests[name] = [plan_digest(p) for p in plans]
        out["total_nnz"] = int(sum(p.stats["total_nnz"] for p in plans))
        del plans
    out["digests_equal"] = digests["device"] == digests["host"]
    out["speedup"] = out["host_s"] / out["device_s"]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
