"""The drop-in, proved on the reference's own code.

The unmodified reference installed in baseline/_ref (pip --target) is
copied to a temporary directory, integration/_b200.py is dropped into it and
integration/symcone_b200.patch is applied with patch(1).  Then:

* CPU: the patched package with the device path off is the reference (same solves);
* GPU: with SYMCONE_DEVICE=b200 the reference's own solve_ses / solve_svm, adaptive
  search, _Bracket and result types run on libscmwu.so and reproduce the reference's
  recorded headline solves (tests/golden/headline/).
Skipped when baseline/_ref is not installed.
"""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "symcone")
LIB = os.path.join(ROOT, "paper_2405_09157_b200", "libscmwu.so")

needs_ref = pytest.mark.skipif(not os.path.isdir(REF),
                               reason="the reference is not installed in baseline/_ref")


@pytest.fixture(scope="module")
def patched(tmp_path_factory):
    base = tmp_path_factory.mktemp("patched")
    shutil.copytree(REF, base / "symcone", ignore=shutil.ignore_patterns("__pycache__"))
    shutil.copy(os.path.join(ROOT, "integration", "_b200.py"), base / "symcone" / "_b200.py")
    with open(os.path.join(ROOT, "integration", "symcone_b200.patch")) as fh:
        r = subprocess.run(["patch", "-p1", "-d", str(base)], stdin=fh, capture_output=True,
                           text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return str(base)


def _run(path, code, device):
    env = dict(os.environ, PYTHONPATH=path, NUMBA_CACHE_DIR="/tmp/numba_cache_dropin",
               SCMWU_LIB=LIB)
    env.pop("SYMCONE_DEVICE", None)
    if device:
        env["SYMCONE_DEVICE"] = "b200"
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout.strip().splitlines()[-1])




def _solve_code(kind, args, eps):
    return f"""
import json
import symcone
from symcone import instances, ses, svm
if {kind!r} == "ses":
    inst = instances.gen_ses(*{args!r})
    r, s = ses.solve_ses(inst, {eps!r})
    out = dict(value=s.radius, slack=s.enclosure_slack)
else:
    inst, _ = instances.gen_svm(*{args!r})
    r, s = svm.solve_svm(inst, {eps!r})
    out = dict(value=s.margin, pd=s.pd_distance, mu_sum=float(s.pd_point[0].sum()))
out.update(iterations=r.total_iterations, steps=r.search_steps,
           termination=r.termination.value,
           search=[[st.alpha, st.iterations, st.reason] for st in r.steps])
print(json.dumps(out))
"""


@needs_ref
def test_patched_reference_cpu_path_unchanged(patched):
    """Device path off: the patched package solves exactly like the reference."""
    code = _solve_code("svm", (50, 50, 4, 1, 1.0), 1e-2)
    got = _run(patched, code, device=False)
    base = os.path.dirname(REF)
    ref = _run(base, code, device=False)
    assert got == ref


def _golden(name):
    with open(os.path.join(ROOT, "tests", "golden", "headline", name)) as fh:
        return json.load(fh)["solve"]


@needs_ref
@pytest.mark.gpu
def test_patched_reference_svm_on_b200(patched):
    g = _golden("svm_n2000_t1.json")
    got = _run(patched, _solve_code("svm", (1000, 1000, 100, 0, 1.0), 1e-3), device=True)
    assert got["iterations"] == g["iterations"] and got["steps"] == g["steps"]
    assert got["termination"] == g["termination"]
    assert [(s[1], s[2]) for s in got["search"]] == [(s[3], s[5]) for s in g["search"]]
    assert abs(got["value"] - g["margin"]) <= 1e-6 * g["margin"]
    assert abs(got["pd"] - g["pd_distance"]) <= 1e-6 * g["pd_distance"]
    assert abs(got["mu_sum"] - 1.0) <= 1e-12


@needs_ref
@pytest.mark.gpu
def test_patched_reference_ses_on_b200(patched):
    g = _golden("ses_n1000_t1.json")
    got = _run(patched, _solve_code("ses", (1000, 100, 0, "uniform-ball"), 1e-3), device=True)
    assert got["iterations"] == g["iterations"] and got["steps"] == g["steps"]
    assert got["termination"] == g["termination"]
    assert [(s[1], s[2]) for s in got["search"]] == [(s[3], s[5]) for s in g["search"]]
    assert abs(got["value"] - g["radius"]) <= 1e-5 * g["radius"]
    assert abs(got["slack"]) <= 1e-9 * got["value"]
