"""Per-stage ALT timing (CUDA events) with each stage's algorithmic bytes."""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--tol", type=float, default=1e-12)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--chunk", type=int, default=0,
                help="plan only chunk 0 of this many LPT chunks (N=4096-style runs)")
a = ap.parse_args()
if a.chunk:
    from paper_2004_11346_b200.dist import lpt_orders
    orders = lpt_orders(a.n, a.chunk)[0]
else:
    orders = range(2 * a.n)
plans = plan_orders(a.n, orders, SamplingConfig(tolerance=a.tol), processes=0)
dp = DevicePlan(plans)
pk = dp.packed
ops, tasks = pk.ops, pk.tasks
tile_b = np.where(ops["kind"] == 2, 0, ((ops["R"].astype(np.int64) * ops["C"] * 8 + 15) // 16) * 16)
vec_n = np.where(ops["kind"] == 0, ops["C"], np.where(ops["kind"] == 1, ops["R"], ops["R"]))
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
out = []
for d, bounds in ((0, pk.stages_fwd), (1, pk.stages_inv)):
    for s in range(len(bounds) - 1):
        t0, t1 = int(bounds[s]), int(bounds[s + 1])
        tk = tasks[t0:t1]
        sel = np.concatenate([np.arange(t["op_begin"], t["op_begin"] + t["op_count"]) for t in tk]) \
            if t1 > t0 else np.zeros(0, np.int64)
        tb = int(tile_b[sel].sum())
        vb = int(vec_n[sel].sum()) * 32
        gathers = int(((ops["flags"][sel] & 1) != 0).sum())
        for _ in range(2):
            dp.lib.bfsht_alt_stage(dp.handle, d, s, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            dp.lib.bfsht_alt_stage(dp.handle, d, s, st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        nb, nrec, nfold = dp.chain_info(d, s)
        rec = {"dir": d, "stage": s, "tasks": t1 - t0, "ops": int(sel.size), "gather_ops": gathers,
               "chain_bundles": nb, "chain_records": nrec, "folded_adds": nfold,
               "tile_MB": tb / 1e6, "vec_MB": vb / 1e6, "avg_tile_KB": tb / max(sel.size, 1) / 1e3,
               "ms": ms, "tile_GBps": tb / ms / 1e6}
        out.append(rec)
        print(json.dumps(rec), flush=True)
