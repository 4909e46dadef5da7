"""The range D from the resident rows (sc_row_range) equals the reference's numpy
expression bit for bit (R/ses.py:65-72, R/svm.py:62-66).  The row norms restate numpy's
pairwise summation (csrc/np_rownorm.h); here the restatement runs through the CPU emulator
(same header, host compiler) and tests/test_gpu_range.py runs it on the device.
"""
import numpy as np
import pytest

from paper_2405_09157_b200 import instances, ses, svm
from paper_2405_09157_b200 import _native as nat


def _ref_ses_range(c, r):
    """R/ses.py:69-70, verbatim numpy."""
    v1 = c[0]
    return float((np.linalg.norm(c[1:] - v1, axis=1) + r[0] + r[1:]).max())


def _ref_max_norm(P, Q):
    """R/svm.py:64-66, verbatim numpy."""
    return float(max(np.linalg.norm(P, axis=1).max(), np.linalg.norm(Q, axis=1).max()))


# every branch of numpy's pairwise sum: n < 8, 8 <= n <= 128 with and without a tail,
# one and two recursive splits
DIMS = [1, 2, 5, 7, 8, 9, 13, 16, 31, 64, 100, 127, 128, 129, 136, 200, 255, 256, 257,
        300, 384, 511, 512]


@pytest.mark.parametrize("d", DIMS)
def test_ses_row_range_matches_numpy(emu_engine, d):
    rng = np.random.default_rng(d)
    n = 400
    c = rng.standard_normal((n, d)) * rng.uniform(0.1, 10.0, size=(n, 1))
    r = rng.uniform(0.0, 0.5, size=n)
    inst = ses.SesInstance(c, r)
    dev = ses.ses_device(inst, engine=emu_engine)
    try:
        assert dev.handle.prob.D == _ref_ses_range(c, r)
        assert dev.handle.prob.D == ses.ses_range(inst)[0]
        assert dev.handle.row_range() == dev.handle.prob.D
    finally:
        dev.close()


@pytest.mark.parametrize("d", DIMS)
def test_svm_row_range_matches_numpy(emu_engine, d):
    inst, _ = instances.gen_svm(150, 90, d, d, 0.7)
    ref = _ref_max_norm(inst.P, inst.Q)
    dev = svm.svm_device(inst, engine=emu_engine)
    try:
        assert dev.handle.prob.D == ref
        assert inst.max_norm == ref          # the cached value the device filled in
    finally:
        dev.close()


def test_row_norms_restatement_on_many_rows(emu_engine):
    """Per-row terms, not only the maximum: shift the rows so each one in turn is the
    farthest; every row's norm must equal numpy's."""
    rng = np.random.default_rng(7)
    d = 100
    c = rng.standard_normal((64, d))
    norms = np.linalg.norm(c, axis=1)
    for i in range(0, 64, 9):
        P = c.copy()
        P[i] *= 1e3 / norms[i]                     # row i dominates
        Q = c[:2] * 1e-3
        inst = svm.SvmInstance(P, Q)
        dev = svm.svm_device(inst, engine=emu_engine)
        try:
            assert dev.handle.prob.D == float(np.linalg.norm(P[i:i + 1], axis=1)[0])
        finally:
            dev.close()


def test_degenerate_range_is_zero(emu_engine):
    c = np.ones((5, 3))
    inst = ses.SesInstance(c, np.zeros(5))
    rep, sol = ses.solve_ses(inst, 1e-2, engine=emu_engine)
    assert sol.radius == 0.0 and rep.total_iterations == 0


def test_constants_follow_the_range(emu_engine):
    """sc_set_range derives rho, R, rank and ln_r as the solvers do (R/ses.py:161,169)."""
    inst = instances.gen_ses(300, 10, 0, "gaussian")
    dev = ses.ses_device(inst, engine=emu_engine)
    try:
        D = ses.ses_range(inst)[0]
        p = dev.handle.prob
        assert p.D == D and p.rho == 3.0 * D / np.sqrt(2.0) and p.rank == 2 * 299
    finally:
        dev.close()
    assert nat.SC_SES == 0
