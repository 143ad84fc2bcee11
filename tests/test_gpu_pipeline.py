"""HostPipeline (api.py): streamed host-buffer transforms give the same bits
as the synchronous device calls, including forward -> inverse chained
through one host grid buffer with no host synchronization in between, and
host buffers reused while earlier jobs are still in flight."""
import numpy as np
import pytest

from paper_2004_11346_b200 import plan_sht

pytestmark = pytest.mark.gpu


def _flat(n, seed):
    rng = np.random.default_rng(seed)
    size = 4 * n * n
    return rng.standard_normal(size) + 1j * rng.standard_normal(size)


@pytest.mark.parametrize("depth,lag", [(1, 0), (2, 1), (3, 2)])
def test_pipeline_bitwise_vs_device_calls(depth, lag):
    import torch
    from paper_2004_11346_b200.api import ShtDevice
    n = 32
    dev = ShtDevice(plan_sht(n))
    jobs = 7
    flats = [_flat(n, s) for s in range(jobs)]
    want_g, want_b = [], []
    for f in flats:
        g = dev.forward(torch.from_numpy(f).cuda())
        want_g.append(g.cpu().numpy())
        want_b.append(dev.inverse(g).cpu().numpy())
    pipe = dev.pipeline(depth=depth)
    nbuf = lag + 2
    h_c = [torch.empty(4 * n * n, dtype=torch.complex128).pin_memory() for _ in range(nbuf)]
    h_g = [torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128).pin_memory()
           for _ in range(nbuf)]
    h_b = [torch.empty(4 * n * n, dtype=torch.complex128).pin_memory() for _ in range(nbuf)]
    got_g, got_b = [None] * jobs, [None] * jobs
    ev_g, ev_b = [None] * jobs, [None] * jobs
    for i in range(jobs + lag):
        if i < jobs:
            k = i % nbuf
            if i >= nbuf:   # host buffers are reused: harvest the old job first
                ev_b[i - nbuf].synchronize()
                got_b[i - nbuf] = h_b[k].numpy().copy()
            h_c[k].copy_(torch.from_numpy(flats[i]))
            ev_g[i] = pipe.forward(h_c[k], h_g[k])
        j = i - lag
        if j >= 0:
            k = j % nbuf
            ev_g[j].synchronize()
            got_g[j] = h_g[k].numpy().copy()
            ev_b[j] = pipe.inverse(h_g[k], h_b[k])
    pipe.synchronize()
    for j in range(jobs):
        if got_b[j] is None:
            got_b[j] = h_b[j % nbuf].numpy().copy()
    for j in range(jobs):
        assert np.array_equal(got_g[j], want_g[j]), j
        assert np.array_equal(got_b[j], want_b[j]), j


def test_pipeline_rejects_bad_buffers():
    import torch
    from paper_2004_11346_b200.api import ShtDevice
    n = 8
    pipe = ShtDevice(plan_sht(n)).pipeline()
    g = torch.empty((2 * n, 4 * n - 1), dtype=torch.complex128).pin_memory()
    with pytest.raises(ValueError, match="pinned"):
        pipe.forward(torch.zeros(4 * n * n, dtype=torch.complex128), g)
    with pytest.raises(ValueError, match="values"):
        pipe.forward(torch.zeros(5, dtype=torch.complex128).pin_memory(), g)
    with pytest.raises(ValueError, match="host"):
        pipe.forward(torch.zeros(4 * n * n, dtype=torch.complex128, device="cuda"), g)
