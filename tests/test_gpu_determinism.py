"""Bitwise reproducibility across processes (R/_reduce.py:1-6 promises it for a fixed
partition; SPEC :612).  The row partition is the equal cyclic one by CTA index and every
reduction has a fixed order, so two processes solving the same instance must agree to the
last bit, iteration for iteration — on the SES trajectory, which is sensitive to the last
bit (SURVEY finding 5), and at a size large enough for the opt-in calibrated partition."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

CODE = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2405_09157_b200 import instances, ses, svm
inst = instances.gen_ses(300_000, 100, 5, "uniform-ball")
r, s = ses.solve_ses(inst, 3e-3)
inst2, _ = instances.gen_svm(150_000, 150_000, 100, 5, 1.0)
r2, s2 = svm.solve_svm(inst2, 1e-2)
print(json.dumps(dict(it=r.total_iterations, steps=[[st.alpha.hex(), st.iterations]
                                                   for st in r.steps],
                     radius=s.radius.hex(), center=[c.hex() for c in s.center[:8]],
                     it2=r2.total_iterations, margin=s2.margin.hex(),
                     pd=s2.pd_distance.hex())))
""" % ROOT


def _run():
    env = dict(os.environ)
    env.pop("SCMWU_BALANCE", None)
    r = subprocess.run([sys.executable, "-c", CODE], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_two_processes_bitwise_identical():
    a, b = _run(), _run()
    assert a == b
