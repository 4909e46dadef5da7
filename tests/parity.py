"""Shared parity helpers: replay recorded reference calls through an engine
(the CUDA library on the GPU box, the CPU emulator in the CPU suite) and compare
with the reference / the oracle under the tiered contract of DESIGN.md §6:

  P1/P2  per-call results of one feasibility test, teacher-forced at the call
         boundary (same alpha, eps, caps, bounds as the reference's call);
  P3     SVM end-to-end: identical iteration counts and termination, values to 1e-6;
  P4     SES end-to-end: certified radius, inside the reference's own spread.
"""
from __future__ import annotations

import math

import numpy as np

from conftest import gf
from paper_2405_09157_b200 import instances, meta, ses, svm


def make_device(kind, inst_args, engine):
    if kind == "ses":
        inst = instances.gen_ses(*inst_args)
        dev = ses.ses_device(inst, engine=engine)
        D, _, _ = ses.ses_range(inst)
        spec = meta.OracleSpec(dev.cone, 3.0 * D / math.sqrt(2.0), inst.d + 1, dev,
                               math.sqrt(2.0), meta.Orientation.MAX)
    else:
        inst, _ = instances.gen_svm(*inst_args)
        dev = svm.svm_device(inst, engine=engine)
        D = inst.max_norm
        spec = meta.OracleSpec(dev.cone, 2.0 * D, inst.d + 2, dev, 2.0, meta.Orientation.MIN,
                               counter_progress=True)
    return inst, dev, spec


def replay(call, spec, dev):
    st = meta.EarlyStopConfig(delta=call["delta"], patience=call["patience"],
                              enabled=call["enabled"])
    if call["fn"] == "ftp":
        return meta.solve_ftp(spec, call["alpha"], call["eps"], st, dev.progress, call["cap"])
    lo, hi = (gf(b) for b in call["bounds"])
    return meta.refine_run(spec, call["alpha"], call["horizon"], st, dev.progress,
                           gain_rel=call["gain_rel"], bounds=(lo, hi), target=call["target"])


def close(a, b, rel, abs_=1e-12):
    if a is None or b is None:
        return a is None and b is None
    a, b = gf(a), gf(b)
    if math.isinf(a) or math.isinf(b):
        return a == b
    return math.isclose(a, b, rel_tol=rel, abs_tol=abs_)


def compare_call(res, ref, rel, progress=None):
    """Return a list of mismatch descriptions (empty = parity).

    Offers keep a candidate only on STRICT improvement, so two candidates whose
    certified values tie to rounding may be kept in either order: a differing
    best_y / affirmative y_tilde is accepted when ``progress`` certifies it at the
    reference's best value."""
    bad = []
    is_primal = isinstance(res, meta.PrimalCertificate)
    if is_primal != (ref["type"] == "primal"):
        return [f"type {type(res).__name__} vs {ref['type']}"]
    if res.iterations != ref["iterations"]:
        bad.append(f"iterations {res.iterations} vs {ref['iterations']}")
    if not is_primal and res.reason != ref["reason"]:
        bad.append(f"reason {res.reason} vs {ref['reason']}")
    if not close(res.best_progress, ref["best_progress"], rel):
        bad.append(f"best_progress {res.best_progress} vs {ref['best_progress']}")
    if not close(res.best_counter, ref["best_counter"], rel):
        bad.append(f"best_counter {res.best_counter} vs {ref['best_counter']}")
    def tie_ok(y):
        return progress is not None and ref["best_progress"] is not None and \
            close(progress(np.asarray(y)), ref["best_progress"], max(rel, 1e-12))

    if ref["best_y"] is not None and res.best_y is not None:
        if not np.allclose(res.best_y, ref["best_y"], rtol=rel, atol=1e-10) \
                and not tie_ok(res.best_y):
            bad.append("best_y")
    if is_primal:
        if not close(res.oracle_value, ref["oracle_value"], max(rel, 1e-9), 1e-9):
            bad.append(f"oracle_value {res.oracle_value} vs {ref['oracle_value']}")
    else:
        if not close(res.value, ref["value"], rel):
            bad.append(f"value {res.value} vs {ref['value']}")
        if not close(res.eps_eff, ref["eps_eff"], rel):
            bad.append(f"eps_eff {res.eps_eff} vs {ref['eps_eff']}")
        if not np.allclose(res.y_tilde, ref["y_tilde"], rtol=rel, atol=1e-10) and not (
                res.reason == "affirmative" and tie_ok(res.y_tilde)):
            bad.append("y_tilde")
    return bad


def solve(kind, inst_args, eps, engine):
    if kind == "ses":
        inst = instances.gen_ses(*inst_args)
        return inst, ses.solve_ses(inst, eps, engine=engine)
    inst, _ = instances.gen_svm(*inst_args)
    return inst, svm.solve_svm(inst, eps, engine=engine)


def check_svm_solve(inst, rep, sol, g, rel=1e-6):
    """P3: SVM end-to-end parity with the reference."""
    assert rep.total_iterations == g["iterations"], (rep.total_iterations, g["iterations"])
    assert rep.search_steps == g["steps"]
    assert rep.termination.value == g["termination"]
    assert math.isclose(sol.margin, g["margin"], rel_tol=rel)
    assert math.isclose(sol.pd_distance, g["pd_distance"], rel_tol=rel)
    assert np.allclose(sol.w, g["w"], rtol=1e-5, atol=1e-7)
    mu, gam = sol.pd_point
    assert math.isclose(mu.sum(), 1.0, rel_tol=1e-12) and math.isclose(gam.sum(), 1.0,
                                                                         rel_tol=1e-12)
    # the returned pair realises the reported distance
    z = inst.P.T @ mu - inst.Q.T @ gam
    assert math.isclose(float(np.linalg.norm(z)), sol.pd_distance, rel_tol=1e-6)
    # sandwich: margin <= optimum <= pd distance
    assert sol.margin <= sol.pd_distance * (1 + 1e-12)


def check_ses_solve(inst, rep, sol, refs, spread_floor=2e-3):
    """P4: certified enclosure, inside the reference's partition spread."""
    # the reported radius is a certified covering radius at the centre
    d = np.sqrt(((inst.centers - sol.center) ** 2).sum(axis=1)) + inst.radii
    assert d.max() <= sol.radius * (1 + 1e-9), (d.max(), sol.radius)
    assert abs(sol.enclosure_slack) <= 1e-9 * sol.radius
    assert rep.primal_value <= sol.radius
    radii = [r["radius"] for r in refs]
    lo, hi = min(radii), max(radii)
    spread = max((hi - lo) / lo, spread_floor)
    mid = 0.5 * (lo + hi)
    assert abs(sol.radius - mid) / mid <= spread, (sol.radius, radii)
    terms = {r["termination"] for r in refs}
    assert rep.termination.value in terms, (rep.termination.value, terms)
