"""Verification baselines: meb_baseline / gilbert_baseline.

CPU: the oracle restatement (oracle/baselines_oracle.py) reproduces the reference's
records in tests/golden/baselines.json bit for bit.  GPU: the device baselines
(sc_meb_baseline / sc_gilbert_baseline) agree with those records (same vertex choices,
values to 1e-9), and at the BASELINE sizes they cross-check the SCMWU solvers with an
independent algorithm: the SES certified bounds bracket the Badoiu-Clarkson radius, and the
SVM margin / pd distance bracket Gilbert's distance bounds.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import baselines_oracle as B
from paper_2405_09157_b200 import instances

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "baselines.json")))


def _case_inputs(c):
    if c["kind"] == "meb":
        inst = instances.gen_ses(*c["inst"])
        rad = (np.random.default_rng(c["radii_seed"]).uniform(0.0, 0.1, c["inst"][0])
               if c["radii_seed"] is not None else None)
        return inst.centers, rad
    inst, _ = instances.gen_svm(*c["inst"])
    return inst.P, inst.Q


@pytest.mark.parametrize("c", GOLD, ids=lambda c: f"{c['kind']}-{c['inst']}")
def test_oracle_baselines_match_reference(c):
    a, b = _case_inputs(c)
    if c["kind"] == "meb":
        v, cen, it = B.meb_baseline(a, b, **c["kw"])
        assert v == c["value"] and it == c["iterations"]
        assert np.array_equal(cen, np.array(c["center"]))
    else:
        v, gap, it, mu, gam = B.gilbert_baseline(a, b, **c["kw"])
        assert v == c["value"] and gap == c["gap"] and it == c["iterations"]
        assert np.array_equal(mu, np.array(c["mu"])) and np.array_equal(gam, np.array(c["gam"]))


@pytest.mark.gpu
@pytest.mark.parametrize("c", GOLD, ids=lambda c: f"{c['kind']}-{c['inst']}")
def test_device_baselines_match_reference(c):
    from paper_2405_09157_b200 import baselines
    a, b = _case_inputs(c)
    if c["kind"] == "meb":
        r = baselines.meb_baseline(a, b, **c["kw"])
        assert r.iterations == c["iterations"]
        assert abs(r.value - c["value"]) <= 1e-9 * c["value"]
        assert np.allclose(r.certificate, np.array(c["center"]), rtol=0, atol=1e-9)
    else:
        r = baselines.gilbert_baseline(a, b, **c["kw"])
        mu, gam = r.certificate
        assert r.iterations == c["iterations"]
        assert abs(r.value - c["value"]) <= 1e-9 * c["value"]
        assert np.allclose(mu, np.array(c["mu"]), rtol=0, atol=1e-9)
        assert np.allclose(gam, np.array(c["gam"]), rtol=0, atol=1e-9)
        assert abs(np.sum(mu) - 1.0) < 1e-12 and abs(np.sum(gam) - 1.0) < 1e-12


@pytest.mark.gpu
def test_full_size_ses_bracketed_by_independent_meb():
    """configs[1] shape (n = 10^6, d = 100, uniform ball): the SCMWU solve's certified
    bounds lower <= OPT <= radius must be consistent with the Badoiu-Clarkson radius
    R_bc, which satisfies OPT <= R_bc <= (1 + eps_base) OPT."""
    from paper_2405_09157_b200 import baselines, ses
    inst = instances.gen_ses(10 ** 6, 100, 0, "uniform-ball")
    dev = ses.ses_device(inst)
    try:
        rep, sol = ses.solve_ses(inst, 1e-2, device=dev)
        eps_base = 0.05
        r = baselines.meb_baseline(dev, eps_base=eps_base)
    finally:
        dev.close()
    assert rep.primal_value <= r.value * (1 + 1e-12)          # lower <= OPT <= R_bc
    assert r.value / (1 + eps_base) <= sol.radius * (1 + 1e-12)  # OPT <= radius
    assert sol.enclosure_slack <= 1e-12


@pytest.mark.gpu
def test_full_size_svm_bracketed_by_independent_gilbert():
    """configs[2] shape (n = 10^6, d = 100): the SVM margin is a certified lower bound of
    the polytope distance and the pd pair realises an upper bound; Gilbert gives
    |z| >= OPT >= sqrt(|z|^2 - gap)."""
    from paper_2405_09157_b200 import baselines, svm
    inst, _ = instances.gen_svm(500_000, 500_000, 100, 0, 1.0)
    dev = svm.svm_device(inst)
    try:
        r = baselines.gilbert_baseline(dev, gap_tol=1e-6, max_iters=2000)
        rep, sol = svm.solve_svm(inst, 1e-2, device=dev)
    finally:
        dev.close()
    lower_g = math.sqrt(max(0.0, r.value ** 2 - r.gap))
    assert sol.margin <= r.value * (1 + 1e-12)       # margin <= OPT <= |z|
    assert lower_g <= sol.pd_distance * (1 + 1e-12)  # OPT <= pd distance
