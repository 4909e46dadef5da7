"""sc_row_range on the device: the range D of the resident rows equals the reference's
numpy expression bit for bit (R/ses.py:65-72, R/svm.py:62-66), and building a handle no
longer scans X on the host.
"""
import numpy as np
import pytest

from paper_2405_09157_b200 import instances, ses, svm

pytestmark = pytest.mark.gpu

DIMS = [1, 5, 8, 9, 13, 64, 100, 128, 129, 200, 256, 257, 384, 512]


@pytest.mark.parametrize("d", DIMS)
def test_ses_row_range_bitwise(d):
    rng = np.random.default_rng(100 + d)
    n = 20_000
    c = rng.standard_normal((n, d)) * rng.uniform(0.1, 10.0, size=(n, 1)) + 3.0
    r = rng.uniform(0.0, 0.5, size=n)
    inst = ses.SesInstance(c, r)
    ref = float((np.linalg.norm(c[1:] - c[0], axis=1) + r[0] + r[1:]).max())
    dev = ses.ses_device(inst)
    try:
        assert dev.handle.prob.D == ref
    finally:
        dev.close()


@pytest.mark.parametrize("d", DIMS)
def test_svm_row_range_bitwise(d):
    inst, _ = instances.gen_svm(7_000, 5_000, d, d, 0.5)
    ref = float(max(np.linalg.norm(inst.P, axis=1).max(), np.linalg.norm(inst.Q, axis=1).max()))
    dev = svm.svm_device(inst)
    try:
        assert dev.handle.prob.D == ref
    finally:
        dev.close()


def test_headline_shapes_and_no_host_scan(monkeypatch):
    """configs[1]-shaped rows (uniform ball, d = 100): the device range equals ses_range,
    and solve_ses builds its handle without calling it."""
    inst = instances.gen_ses(1_000_000, 100, 0, "uniform-ball")
    D = ses.ses_range(inst)[0]
    dev = ses.ses_device(inst)
    try:
        assert dev.handle.prob.D == D
    finally:
        dev.close()

    def no_scan(_inst):
        raise AssertionError("host scan of X")
    monkeypatch.setattr(ses, "ses_range", no_scan)
    small = instances.gen_ses(2_000, 10, 0, "uniform-ball")
    rep, sol = ses.solve_ses(small, 1e-2)
    assert sol.radius > 0 and rep.total_iterations > 0


def test_every_row_can_be_the_maximum():
    """Per-row norms, not just one maximum: make each sampled row the farthest in turn."""
    rng = np.random.default_rng(11)
    d = 100
    c = rng.standard_normal((4096, d))
    nrm = np.linalg.norm(c, axis=1)
    for i in range(0, 4096, 257):
        P = c.copy()
        P[i] *= 1e3 / nrm[i]
        inst = svm.SvmInstance(P, c[:3] * 1e-3)
        dev = svm.svm_device(inst)
        try:
            assert dev.handle.prob.D == float(np.linalg.norm(P[i:i + 1], axis=1)[0])
        finally:
            dev.close()
