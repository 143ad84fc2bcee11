"""Time the SHT DFT stage (synthesis / analysis kernels over all row pairs)
at N=4096 and N=8192 on random node halves / grids (CUDA events)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2004_11346_b200.ooc import ChunkedSht  # noqa: E402


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


out = {}
for n, ch in ((4096, 48), (8192, 96)):
    run = ChunkedSht(n, ch, processes=1, only=[])
    L = 4 * n - 1
    lib, st = run.lib, run._stream()
    run.ybuf.normal_()
    grid = torch.randn((2 * n, L), dtype=torch.complex128, device="cuda")
    for name, fn in (("synth", lambda: lib.bfsht_synth_rows(run.ctx.handle, _ptr(run.layout_dev),
                                                            _ptr(run.ybuf), 0, n, _ptr(grid), st)),
                     ("anal", lambda: lib.bfsht_anal_rows(run.ctx.handle, _ptr(run.layout_dev),
                                                          _ptr(run.ybuf), 0, n, _ptr(grid),
                                                          _ptr(run.weights), st))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            fn()
        e1.record()
        e1.synchronize()
        out[f"{name}_n{n}_ms"] = e0.elapsed_time(e1) / 3
    run.close()
    del run, grid
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
