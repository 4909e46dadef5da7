"""The device-resident adaptive search (sc_solve, one launch per solve) against the
host-driven one (SCMWU_HOST_SEARCH=1, one sc_ftp launch per test) on the GPU.

SVM decisions are robust to the last bit (SURVEY finding 5): identical search steps,
iteration counts and termination, values to 1e-12.  SES trajectories are chaotic; the
seed's progress is evaluated by a different kernel in the two paths (a progress pass of
the persistent kernel vs progress_kernel), so SES is compared on a known answer and by the
certified result."""
import math

import numpy as np
import pytest

from paper_2405_09157_b200 import instances, ses, svm

pytestmark = pytest.mark.gpu


def _both(monkeypatch, fn):
    monkeypatch.setenv("SCMWU_HOST_SEARCH", "1")
    a = fn()
    monkeypatch.delenv("SCMWU_HOST_SEARCH")
    b = fn()
    return a, b


def _steps(rep):
    return [(s.iterations, s.reason) for s in rep.steps]


@pytest.mark.parametrize("args,eps", [((150, 150, 5, 2, 1.0), 1e-2),
                                      ((1000, 1000, 10, 0, 1.0), 1e-2),
                                      ((2000, 3000, 100, 4, 0.5), 1e-2),
                                      ((20000, 20000, 512, 1, 1.0), 3e-2)])
def test_svm_resident_equals_host_search(monkeypatch, args, eps):
    inst, _ = instances.gen_svm(*args)
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: svm.solve_svm(inst, eps))
    assert _steps(r1) == _steps(r2)
    assert r1.total_iterations == r2.total_iterations and r1.termination == r2.termination
    for a, b in zip(r1.steps, r2.steps):
        assert math.isclose(a.alpha, b.alpha, rel_tol=1e-12)
    assert math.isclose(s1.margin, s2.margin, rel_tol=1e-12)
    assert math.isclose(s1.pd_distance, s2.pd_distance, rel_tol=1e-12)
    assert np.allclose(s1.pd_point[0], s2.pd_point[0], rtol=1e-9, atol=1e-15)


def test_ses_resident_search_known_answer(monkeypatch):
    th = np.linspace(0, 2 * np.pi, 32, endpoint=False)
    inst = ses.SesInstance(np.stack([np.cos(th), np.sin(th)], 1), np.zeros(32))
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: ses.solve_ses(inst, 0.05))
    assert r1.total_iterations == r2.total_iterations == 18
    assert s1.radius == pytest.approx(s2.radius, rel=1e-12)


@pytest.mark.parametrize("args,eps", [((3000, 17, 1, "uniform-ball"), 1e-2),
                                      ((20000, 100, 2, "gaussian"), 3e-3)])
def test_ses_resident_search_certified(monkeypatch, args, eps):
    inst = instances.gen_ses(*args)
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: ses.solve_ses(inst, eps))
    for r, s in ((r1, s1), (r2, s2)):
        f = float((np.sqrt(((inst.centers - s.center) ** 2).sum(axis=1)) + inst.radii).max())
        assert f <= s.radius * (1 + 1e-9) and abs(s.enclosure_slack) <= 1e-9 * s.radius
        assert r.primal_value <= s.radius
    assert r1.termination == r2.termination
    assert abs(s1.radius - s2.radius) <= 3 * eps * s1.radius


@pytest.mark.parametrize("cfg", [dict(iteration_cap_override=64), dict(early_stop=False),
                                 dict(delta=1e-3, patience=3)])
def test_svm_resident_search_configs(monkeypatch, cfg):
    """RunConfig knobs reach the device search: an iteration cap, early stop off, other
    delta / patience — the same decisions as the host-driven search."""
    from paper_2405_09157_b200 import RunConfig
    inst, _ = instances.gen_svm(500, 600, 12, 3, 0.7)
    c = RunConfig(**cfg)
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: svm.solve_svm(inst, 1e-2, c))
    assert _steps(r1) == _steps(r2) and r1.termination == r2.termination
    assert math.isclose(s1.margin, s2.margin, rel_tol=1e-12)


def test_resident_search_tiny_instances():
    """Smallest shapes through sc_solve: the SPEC two-point SVM and collinear SES."""
    r, s = svm.solve_svm(svm.SvmInstance(np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]])), 0.01)
    assert s.margin == 2.0 and s.pd_distance == 2.0
    r, s = ses.solve_ses(ses.SesInstance(np.array([[0.0], [1.0], [2.0]]), np.zeros(3)), 0.05)
    assert 1.0 <= s.radius <= 1.05


@pytest.mark.parametrize("n1,n2,d,seed,gap", [(60, 70, 1, 1, 0.8), (40, 90, 3, 2, 0.5),
                                              (60, 70, 33, 5, 0.8), (60, 70, 129, 5, 0.8),
                                              (50, 45, 257, 6, 1.0), (60, 70, 512, 5, 0.8)])
def test_svm_full_solve_matches_oracle_across_d(n1, n2, d, seed, gap):
    """The whole device solve (sc_solve) vs the oracle's restatement of the reference's
    solve_svm (bit-exact with the reference) across the kernel configurations (lanes per
    row 2..32, odd d with padded rows, d = 512): identical search steps, iteration counts
    and termination; margin and pd distance to 1e-6 (SVM decisions are robust)."""
    import oracle as O
    inst, _ = instances.gen_svm(n1, n2, d, seed, gap)
    rep, sol = svm.solve_svm(inst, 1e-2)
    ref = O.solve_svm(inst.P, inst.Q, 1e-2)
    assert rep.total_iterations == ref["iterations"] and rep.search_steps == ref["steps"]
    assert rep.termination.value == ref["termination"]
    assert [(s.iterations, s.reason) for s in rep.steps] == \
        [(s.iterations, s.reason) for s in ref["search"]]
    assert math.isclose(sol.margin, ref["margin"], rel_tol=1e-6)
    assert math.isclose(sol.pd_distance, ref["pd_distance"], rel_tol=1e-6)
