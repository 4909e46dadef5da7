"""Failure path of the in-kernel rank exchange: a rank that never arrives.

Two emulated ranks on one GPU (SCMWU_VWORLD=2: CTA groups of one launch running the real
exchange code); fault injection (SCMWU_FAULT_DROP_RANK=1, test-only) makes rank 1 never
raise its arrival flags.  Rank 0 must give up after SCMWU_EXCHANGE_TIMEOUT_S, set the
launch-wide abort word so every CTA (both ranks, any barrier) leaves the pass loop, and
the call must return SC_ENCCL — not hang, not SC_ECUDA — after which the handle refuses
further calls with SC_ENCCL (its flag epochs no longer match the peers')."""
import json
import os
import subprocess
import sys
import time

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

CODE = r"""
import json, math, sys, time
sys.path.insert(0, %(root)r)
from paper_2405_09157_b200 import _native as nat, instances, meta, svm
inst, _ = instances.gen_svm(3000, 3000, 20, 0, 1.0)
dev = svm.svm_device(inst)
D = inst.max_norm
spec = meta.OracleSpec(dev.cone, 2 * D, 22, dev, 2.0, meta.Orientation.MIN,
                       counter_progress=True)
out = {}
t0 = time.time()
try:
    meta.refine_run(spec, 0.3 * D, 256, meta.EarlyStopConfig(enabled=False), dev.progress)
    out["first"] = "ok"
except nat.NativeError as e:
    out["first"] = e.status
out["first_s"] = time.time() - t0
t0 = time.time()
try:
    meta.refine_run(spec, 0.3 * D, 256, meta.EarlyStopConfig(enabled=False), dev.progress)
    out["second"] = "ok"
except nat.NativeError as e:
    out["second"] = e.status
out["second_s"] = time.time() - t0
dev.close()
print("RESULT " + json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ, SCMWU_VWORLD="2", SCMWU_EXCHANGE_TIMEOUT_S="1", **env_extra)
    r = subprocess.run([sys.executable, "-c", CODE % {"root": ROOT}], capture_output=True,
                       text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][0][7:])


def test_missing_rank_aborts_with_enccl():
    out = _run({"SCMWU_FAULT_DROP_RANK": "1"})
    assert out["first"] == 3, out           # SC_ENCCL
    assert out["first_s"] < 60, out         # gave up after the timeout, did not hang
    assert out["second"] == 3 and out["second_s"] < 1.0, out   # the handle stays unusable


def test_healthy_ranks_unaffected():
    out = _run({})
    assert out["first"] == "ok" and out["second"] == "ok", out
