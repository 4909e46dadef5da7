"""Pin the oracle (CPU restatement) against vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py, which imports the reference
from /root/reference in the build container.  The oracle restates the
reference's arithmetic order (numpy calls on the same shapes, C loops with glibc
exp for the numba kernels), so on the build machine it reproduces the reference
bit for bit; elsewhere (other CPU, other BLAS threading) to rounding.
"""
import hashlib
import math

import numpy as np
import pytest

import oracle as O
from conftest import gf
from paper_2405_09157_b200 import instances


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_generators_match_reference(golden):
    for g in golden["generators"]["ses"]:
        inst = instances.gen_ses(g["n"], g["d"], g["seed"], g["dist"])
        assert _digest(inst.centers) == g["centers"], g
        assert _digest(inst.radii) == g["radii"]
        c, r = O.gen_ses(g["n"], g["d"], g["seed"], g["dist"])
        assert _digest(c) == g["centers"]
    for g in golden["generators"]["svm"]:
        inst, direction = instances.gen_svm(g["n1"], g["n2"], g["d"], g["seed"], g["gap"])
        assert _digest(inst.P) == g["P"] and _digest(inst.Q) == g["Q"], g
        assert _digest(direction) == g["direction"]


def test_learner_kats(golden):
    k = golden["kats"]
    L = O.Learner(2, 1.0, None)
    L.observe(np.array([1.0, -1.0]), 1.0)
    assert np.allclose(L.current(), k["scmwu_orthant2_eta1"], rtol=0, atol=1e-15)
    assert np.allclose(L.current(), [0.11920292, 0.88079708], atol=1e-8)   # SPEC :188
    L = O.Learner(2, 0.5, None)
    for _ in range(200):
        L.observe(np.array([1.0, 0.0]), 1.0)
    p = L.current()
    assert p[1] > 0.999 and np.allclose(p, k["scmwu_orthant2_200steps"], atol=1e-15)
    p = O.Learner(4, 0.3, 4).current()
    assert np.allclose(p, k["init_soc3"], atol=0) and math.isclose(p[3], math.sqrt(2) / 2)


def test_loss_norm_contract():
    L = O.Learner(4, 0.5, 4)
    with pytest.raises(O.LossNormError):
        L.observe(np.array([3.0, 0.0, 0.0, 0.0]), 1.0)   # (0 + 3)/sqrt2 > 1 + 1e-9


def test_oracle_kats(golden):
    k = golden["kats"]["ses_oracle_n2"]
    prob = O.SesProblem(np.array([[0.0, 0.0], [1.0, 0.0]]), np.zeros(2))
    out = prob.query(np.array(k["p"]), 1.5)
    assert isinstance(out, O.Wit)
    assert out.value == k["value"] == pytest.approx(1.5 / math.sqrt(2))   # SPEC :335
    assert np.array_equal(out.y, k["y"])
    assert O.soc_inf_norm(out.residual, 3) == k["res_inf"]
    k = golden["kats"]["svm_oracle_2pt"]
    prob = O.SvmProblem(np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]]))
    out = prob.query(np.array([0.5, 0.5]), 1.0)
    assert out.value == k["value"] == 0.5 and list(out.y) == k["y"]           # SPEC :414
    assert list(out.residual) == k["res"] and out.candidate == k["cand"]


@pytest.mark.parametrize("name", ["ses64_hi", "ses64_mid", "ses33_lo"])
def test_ses_traces(golden, name):
    tr = golden["traces"][name]
    _, n, d, seed, dist = tr["inst"]
    c, r = O.gen_ses(n, d, seed, dist)
    prob = O.SesProblem(c, r)
    L = O.Learner((n - 1) * (d + 1), tr["eta"], d + 1)
    y_sum = np.zeros(d + 1)
    for rec in tr["records"]:
        out = prob.query(L.current(), tr["alpha"])
        if rec.get("separated"):
            assert isinstance(out, O.Sep) and out.value == gf(rec["value"])
            break
        assert out.value == rec["value"], rec["t"]
        assert np.array_equal(out.y[:-1], rec["u"])
        y_sum += out.y
        assert O.soc_inf_norm(out.residual, d + 1) / tr["rho"] == rec["width"]
        assert prob.progress((y_sum / rec["t"])[:d]) == rec["f"]
        L.observe(out.residual, 1.0 / tr["rho"])


@pytest.mark.parametrize("name", ["svm50_a", "svm50_b", "svm50_c"])
def test_svm_traces(golden, name):
    tr = golden["traces"][name]
    _, n1, n2, d, seed, gap = tr["inst"]
    P, Q, _ = O.gen_svm(n1, n2, d, seed, gap)
    prob = O.SvmProblem(P, Q)
    L = O.Learner(n1 + n2, tr["eta"], None)
    y_sum = np.zeros(d + 2)
    for rec in tr["records"]:
        p = L.current()
        out = prob.query(p, tr["alpha"])
        if rec.get("separated"):
            assert isinstance(out, O.Sep) and out.value == pytest.approx(gf(rec["value"]),
                                                                         rel=1e-12)
            break
        assert out.value == pytest.approx(rec["value"], rel=1e-12, abs=1e-14)
        assert np.allclose(out.y[:d], rec["w"], rtol=1e-12, atol=1e-14)
        assert out.candidate == pytest.approx(rec["cand"], rel=1e-12, abs=1e-14)
        y_sum += out.y
        assert prob.progress((y_sum / rec["t"])[:d]) == pytest.approx(rec["f"], rel=1e-12,
                                                                       abs=1e-14)
        L.observe(out.residual, 1.0 / tr["rho"])


def _case(golden, kind, inst):
    for c in golden["calls"]:
        if c["kind"] == kind and c["inst"] == list(inst):
            return c
    raise KeyError(inst)


@pytest.mark.parametrize("inst", [(300, 4, 5, "gaussian"), (64, 3, 3, "gaussian")])
def test_oracle_ses_solve_matches_reference(golden, inst):
    c = _case(golden, "ses", inst)
    cen, rad = O.gen_ses(*inst)
    r = O.solve_ses(cen, rad, c["eps"])
    g = c["solve"]
    assert r["iterations"] == g["iterations"] and r["steps"] == g["steps"]
    assert r["radius"] == pytest.approx(g["radius"], rel=1e-13)
    assert np.allclose(r["center"], g["center"], rtol=1e-12, atol=1e-13)
    assert r["termination"] == g["termination"]


@pytest.mark.parametrize("inst", [(37, 21, 6, 4, 0.5), (50, 50, 4, 1, 1.0)])
def test_oracle_svm_solve_matches_reference(golden, inst):
    c = _case(golden, "svm", inst)
    P, Q, _ = O.gen_svm(*inst)
    r = O.solve_svm(P, Q, c["eps"])
    g = c["solve"]
    assert r["iterations"] == g["iterations"] and r["steps"] == g["steps"]
    assert r["margin"] == pytest.approx(g["margin"], rel=1e-12)
    assert r["pd_distance"] == pytest.approx(g["pd_distance"], rel=1e-12)
    assert np.allclose(r["w"], g["w"], rtol=1e-10, atol=1e-12)


def test_oracle_spec_kats(golden):
    k = golden["kats"]
    th = np.linspace(0, 2 * np.pi, 32, endpoint=False)
    r = O.solve_ses(np.stack([np.cos(th), np.sin(th)], 1), np.zeros(32), 0.05)
    assert r["radius"] == k["ses_circle32"]["radius"] and r["iterations"] == 18
    r = O.solve_ses(np.array([[0.0], [1.0], [2.0]]), np.zeros(3), 0.05)
    assert r["radius"] == k["ses_collinear3"]["radius"]
    r = O.solve_svm(np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]]), 0.01)
    assert r["margin"] == 2.0 and r["pd_distance"] == 2.0          # SPEC :450
