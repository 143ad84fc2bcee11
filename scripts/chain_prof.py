"""One forward SHT at N=1024, then every forward ALT stage once more on its
own (bfsht_alt_stage) — the workload for an ncu capture of the butterfly
chain stages:
  ncu --set full --import-source on -k regex:alt_stage_kernel \
      --launch-skip 7 --launch-count 5 python scripts/chain_prof.py
(the first 7 alt_stage launches belong to the warm-up sht_forward)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import synthetic_coeffs  # noqa: E402
from paper_2004_11346_b200 import SamplingConfig, plan_orders  # noqa: E402
from paper_2004_11346_b200.api import DevicePlan  # noqa: E402

n = int(os.environ.get("N", "1024"))
plans = plan_orders(n, range(2 * n), SamplingConfig(tolerance=1e-12), processes=0)
dp = DevicePlan(plans)
c = torch.from_numpy(synthetic_coeffs(n)).cuda()
g = dp.sht_forward(c)
torch.cuda.synchronize()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
nst = len(dp.packed.stages_fwd) - 1
for s in range(nst):
    assert dp.lib.bfsht_alt_stage(dp.handle, 0, s, st) == 0
torch.cuda.synchronize()
print("stages", nst)
