"""One SHT synthesis launch at N=8192 (L = 32767) for ncu."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_11346_b200.ooc import ChunkedSht  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
run = ChunkedSht(n, 96, processes=1, only=[])
L = 4 * n - 1
run.ybuf.normal_()
grid = torch.empty((2 * n, L), dtype=torch.complex128, device="cuda")
p = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
rc = run.lib.bfsht_synth_rows(run.ctx.handle, p(run.layout_dev), p(run.ybuf), 0, n, p(grid),
                              run._stream())
torch.cuda.synchronize()
print("rc", rc)
