"""Whole-solve residency (sc_solve) checked on the CPU emulator: the
device-resident adaptive search (scmwu_control.h Search, the code the kernel runs between
passes) must reproduce the host-driven restatement of adaptive_search / _Bracket
(meta.adaptive_search, R/meta.py:576-781) decision for decision: same search steps,
iteration counts, termination and results, bit for bit (the emulator evaluates the seed and
final progress passes in the same order as sc_progress)."""
import math

import numpy as np
import pytest

from paper_2405_09157_b200 import RunConfig, instances, meta, ses, svm


def _both(monkeypatch, fn):
    monkeypatch.setenv("SCMWU_HOST_SEARCH", "1")
    a = fn()
    monkeypatch.delenv("SCMWU_HOST_SEARCH")
    b = fn()
    return a, b


def _steps(rep):
    return [(s.alpha, s.eps, s.iteration_bound, s.iterations, s.separated, s.reason)
            for s in rep.steps]


@pytest.mark.parametrize("args,eps", [((300, 4, 5, "gaussian"), 1e-2),
                                      ((64, 3, 3, "gaussian"), 1e-2),
                                      ((200, 6, 1, "uniform-ball"), 3e-3),
                                      ((32, 2, 0, "sphere-surface"), 1e-2)])
def test_ses_resident_search_equals_host_search(emu_engine, monkeypatch, args, eps):
    inst = instances.gen_ses(*args)
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: ses.solve_ses(inst, eps, engine=emu_engine))
    assert _steps(r1) == _steps(r2)
    assert r1.total_iterations == r2.total_iterations and r1.search_steps == r2.search_steps
    assert r1.termination == r2.termination
    assert s1.radius == s2.radius and np.array_equal(s1.center, s2.center)
    assert s1.enclosure_slack == s2.enclosure_slack and r1.primal_value == r2.primal_value


@pytest.mark.parametrize("args,eps", [((150, 150, 5, 2, 1.0), 1e-2),
                                      ((50, 50, 4, 1, 1.0), 1e-2),
                                      ((37, 21, 6, 4, 0.5), 1e-2),
                                      ((100, 120, 8, 3, 0.3), 3e-3)])
def test_svm_resident_search_equals_host_search(emu_engine, monkeypatch, args, eps):
    inst, _ = instances.gen_svm(*args)
    (r1, s1), (r2, s2) = _both(monkeypatch, lambda: svm.solve_svm(inst, eps, engine=emu_engine))
    assert _steps(r1) == _steps(r2)
    assert r1.total_iterations == r2.total_iterations and r1.termination == r2.termination
    assert s1.margin == s2.margin and s1.pd_distance == s2.pd_distance
    assert np.array_equal(s1.w, s2.w)
    assert np.array_equal(s1.pd_point[0], s2.pd_point[0])
    assert np.array_equal(s1.pd_point[1], s2.pd_point[1])


def test_resident_search_honours_cap_and_early_stop(emu_engine, monkeypatch):
    inst = instances.gen_ses(300, 4, 5, "gaussian")
    for cfg in (RunConfig(iteration_cap_override=16), RunConfig(early_stop=False),
                RunConfig(delta=1e-3, patience=3)):
        (r1, s1), (r2, s2) = _both(monkeypatch, lambda: ses.solve_ses(inst, 1e-2, cfg,
                                                                      engine=emu_engine))
        assert _steps(r1) == _steps(r2) and r1.termination == r2.termination
        assert s1.radius == s2.radius
    (r, _), _ = _both(monkeypatch, lambda: ses.solve_ses(inst, 1e-2,
                                                         RunConfig(iteration_cap_override=16),
                                                         engine=emu_engine))
    assert r.termination == meta.Termination.ITERATION_CAP


def test_resident_search_matches_reference_record(emu_engine, golden):
    """The device search on the emulator reproduces the reference's recorded solve."""
    c = [c for c in golden["calls"] if c["kind"] == "svm"][0]
    inst, _ = instances.gen_svm(*c["inst"])
    rep, sol = svm.solve_svm(inst, c["eps"], engine=emu_engine)
    g = c["solve"]
    assert rep.total_iterations == g["iterations"] and rep.search_steps == g["steps"]
    assert math.isclose(sol.margin, g["margin"], rel_tol=1e-9)
    assert math.isclose(sol.pd_distance, g["pd_distance"], rel_tol=1e-9)


def test_resident_search_width_violation(emu_engine):
    """A too-small width inside the search raises WidthViolationError with the failing
    test's level (R/meta.py:323-327 propagated through adaptive_search)."""
    inst = instances.gen_ses(20, 3, 0)
    D, L0, U0 = ses.ses_range(inst)
    h = emu_engine.create(0, inst.centers, None, inst.radii, D=D, rho=0.1 * D,
                          R=math.sqrt(2), rank=2 * 19)
    dev = meta.DeviceProblem(h, ses.ses_cone(20, 3), 0)
    spec = meta.OracleSpec(dev.cone, 0.1 * D, 4, dev, math.sqrt(2), meta.Orientation.MAX)
    with pytest.raises(meta.WidthViolationError) as ei:
        meta.resident_search(spec, L0, U0, 1e-2, None, None, inst.centers[0])
    assert ei.value.iteration >= 1 and ei.value.norm > 0.1 * D and ei.value.alpha > 0
    dev.close()
