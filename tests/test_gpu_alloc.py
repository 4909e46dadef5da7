"""Handle memory on the e2e path: X, radii and the window ring come from the
engine's private stream-ordered pool and are reused by the next handle (up to
SCMWU_POOL_GB, default 12 GiB, stays mapped; sc_pool_trim releases it); larger buffers use
cudaMalloc.  Creating and destroying handles must not leak device memory, and a handle on
reused memory computes exactly what a fresh one does.
"""
import numpy as np
import pytest
import torch

from paper_2405_09157_b200 import instances, ses
from paper_2405_09157_b200.devgen import gen_ses_device

pytestmark = pytest.mark.gpu

SLACK = 64 << 20


def _free():
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info(0)[0]


def test_handles_reuse_pool_memory_without_leaking():
    inst = instances.gen_ses(200_000, 100, 3, "uniform-ball")   # 160 MB of X
    y = np.linspace(-0.1, 0.1, 100)
    dev = ses.ses_device(inst)
    f0 = dev.progress(y)
    dev.close()
    free0 = _free()
    for _ in range(8):
        dev = ses.ses_device(inst)
        assert dev.progress(y) == f0           # bitwise: reused memory, same rows
        dev.close()
    assert _free() >= free0 - SLACK
    # a full solve on a pooled handle equals a solve on a second pooled handle
    r1, s1 = ses.solve_ses(inst, 1e-2)
    r2, s2 = ses.solve_ses(inst, 1e-2)
    assert r1.total_iterations == r2.total_iterations and s1.radius == s2.radius
    assert _free() >= free0 - SLACK


def test_pool_retains_then_trims():
    from paper_2405_09157_b200 import _native as nat
    eng = nat.cuda_engine()
    eng.trim_pool(0)
    free0 = _free()
    for _ in range(2):   # 7e6 x 100 fp64 = 5.6 GB: pooled, reused by the second handle
        dev = gen_ses_device(7_000_000, 100, 1, "uniform-ball")
        dev.close()
        kept = free0 - _free()
        assert kept <= (12 << 30) + SLACK      # at most the retained size stays mapped
    eng.trim_pool(0)
    assert _free() >= free0 - SLACK          # and sc_pool_trim returns it
