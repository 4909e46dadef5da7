"""Width violations on the GPU (R/mwu.py:57-66 -> R/meta.py:323-327, :509-512).

A handle created with a width rho below the true residual bound makes Scmwu.observe's
check fire.  The device must raise WidthViolationError at the same iteration and with
the same residual norm as the oracle restatement of the reference, through both the
bound-certified SES path (exact residuals computed only when the bound fails,
DESIGN.md §4.4) and the SVM path, in refine_run and solve_ftp; and a width that the
residuals respect must not raise.
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2405_09157_b200 import instances, meta, ses, svm

pytestmark = pytest.mark.gpu


def _ses(engine, inst, rho):
    D, _, _ = ses.ses_range(inst)
    n, d = inst.centers.shape
    h = engine.create(0, inst.centers, None, inst.radii, D=D, rho=rho, R=math.sqrt(2),
                      rank=2 * (n - 1))
    dev = meta.DeviceProblem(h, ses.ses_cone(n, d), 0)
    spec = meta.OracleSpec(dev.cone, rho, d + 1, dev, math.sqrt(2), meta.Orientation.MAX)
    return D, dev, spec


def _svm(engine, inst, rho):
    D = inst.max_norm
    h = engine.create(1, inst.P, inst.Q, None, D=D, rho=rho, R=2.0, rank=inst.n1 + inst.n2, n1=inst.n1)
    dev = meta.DeviceProblem(h, svm.svm_cone(inst.n1 + inst.n2), 1)
    spec = meta.OracleSpec(dev.cone, rho, inst.d + 2, dev, 2.0, meta.Orientation.MIN,
                           counter_progress=True)
    return D, dev, spec


def _oracle_outcome(run):
    try:
        r = run()
        return ("ok", r.iterations, None)
    except O.WidthViolation as e:
        return ("width", e.iteration, e.norm)


def _device_outcome(run):
    try:
        r = run()
        return ("ok", r.iterations, None)
    except meta.WidthViolationError as e:
        return ("width", e.iteration, e.norm)


def _same(dev_out, ora_out):
    assert dev_out[0] == ora_out[0], (dev_out, ora_out)
    assert dev_out[1] == ora_out[1], (dev_out, ora_out)
    if ora_out[0] == "width":
        assert math.isclose(dev_out[2], ora_out[2], rel_tol=1e-9), (dev_out, ora_out)


# (n, d, seed, rho / D, alpha / D): violations at iterations 4 and 5 of a refine run, a
# width that holds, and a d = 100 instance streamed from HBM (not shared-memory resident)
SES_CASES = [(300, 5, 3, 1.6, 0.9), (300, 5, 3, 1.65, 0.7), (300, 5, 3, 1.95, 0.7),
             (300, 5, 3, 1.2, 0.7), (20000, 100, 1, 1.6, 0.9), (20000, 100, 1, 2.0, 0.9)]


@pytest.mark.parametrize("n,d,seed,c,a", SES_CASES)
def test_ses_width_violation_matches_oracle(cuda_engine, n, d, seed, c, a):
    inst = instances.gen_ses(n, d, seed, "uniform-ball")
    D, _, _ = ses.ses_range(inst)
    rho = c * D
    D, dev, spec = _ses(cuda_engine, inst, rho)
    pr = O.SesProblem(inst.centers, inst.radii)
    ospec = pr.spec(rho)
    prog = (lambda y: pr.progress(y[:d]))
    st = meta.EarlyStopConfig(enabled=False)
    ora = _oracle_outcome(lambda: O.refine(ospec, a * D, 512, 1e-4, 10, False, prog))
    got = _device_outcome(lambda: meta.refine_run(spec, a * D, 512, st, dev.progress))
    _same(got, ora)
    # solve_ftp: the same check inside the rung ladder (iteration counted over rungs)
    ora = _oracle_outcome(lambda: O.ftp(ospec, a * D, 0.01, progress=prog, cap=512))
    got = _device_outcome(lambda: meta.solve_ftp(spec, a * D, 0.01, meta.EarlyStopConfig(),
                                                 dev.progress, 512))
    _same(got, ora)
    dev.close()


SVM_CASES = [(150, 150, 5, 2, 0.9, 0.1), (150, 150, 5, 2, 0.92, 0.1), (150, 150, 5, 2, 0.92, 0.3),
             (150, 150, 5, 2, 0.6, 0.05), (4000, 4000, 100, 0, 0.8, 0.3)]


@pytest.mark.parametrize("n1,n2,d,seed,c,a", SVM_CASES)
def test_svm_width_violation_matches_oracle(cuda_engine, n1, n2, d, seed, c, a):
    inst, _ = instances.gen_svm(n1, n2, d, seed, 1.0)
    D = inst.max_norm
    rho = c * 2.0 * D
    _, dev, spec = _svm(cuda_engine, inst, rho)
    sp = O.SvmProblem(inst.P, inst.Q)
    ospec = sp.spec()
    ospec.rho = rho
    prog = (lambda y: sp.progress(y[:d]))
    st = meta.EarlyStopConfig(enabled=False)
    ora = _oracle_outcome(lambda: O.refine(ospec, a * D, 512, 1e-4, 10, False, prog))
    got = _device_outcome(lambda: meta.refine_run(spec, a * D, 512, st, dev.progress))
    _same(got, ora)
    dev.close()


def test_width_violation_error_carries_the_reference_fields(cuda_engine):
    inst = instances.gen_ses(300, 5, 3, "uniform-ball")
    D, _, _ = ses.ses_range(inst)
    _, dev, spec = _ses(cuda_engine, inst, 1.6 * D)
    with pytest.raises(meta.WidthViolationError) as ei:
        meta.refine_run(spec, 0.9 * D, 512, meta.EarlyStopConfig(enabled=False), dev.progress)
    e = ei.value
    assert e.alpha == 0.9 * D and e.rho == 1.6 * D and e.iteration == 4 and e.norm > e.rho
    # the handle stays usable after the error
    r = meta.refine_run(spec, 0.6 * D, 64, meta.EarlyStopConfig(enabled=False), dev.progress)
    assert r.iterations == 64
    dev.close()
