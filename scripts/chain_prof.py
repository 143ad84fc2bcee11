"""One forward SHT at N=1024, then every forward ALT stage once more on its
own (bfsht_alt_stage) — the workload for an ncu capture of the butterfly
chain stages:
  ncu --set full --import-source on -k regex:alt_stage_kernel \
      --launch-skip 7 --launch-count 5 python scripts/chain_prof.py
(the first 7 alt_stage launches belong to the warm-up sht_forward).  With
CACHE=dir the packed plan comes from / goes to a BFPK file, so a run under
ncu does not start the planner's process pool."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan  # noqa: E402
from paper_2004_11346_b200.pack import load_packed, pack_plans, save_packed  # noqa: E402

n = int(os.environ.get("N", "1024"))
cache = os.environ.get("CACHE")
path = os.path.join(cache, f"chain_n{n}.bfpk") if cache else None
if path and os.path.exists(path):
    packed = load_packed(path)
else:
    plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
    packed = pack_plans(plans)
    if path:
        os.makedirs(cache, exist_ok=True)
        save_packed(packed, path)
dp = DevicePlan([], packed=packed)
c = torch.from_numpy(synthetic_coeffs(n)).cuda()
g = dp.sht_forward(c)
torch.cuda.synchronize()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
nst = len(dp.packed.stages_fwd) - 1
for s in range(nst):
    assert dp.lib.bfsht_alt_stage(dp.handle, 0, s, st) == 0
torch.cuda.synchronize()
print("stages", nst)
