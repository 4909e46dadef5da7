"""Small runs of every device entry point, for the bounds-checked library (compute-sanitizer
is not available on the GPU pool):

    SCMWU_LIB=paper_2405_09157_b200/libscmwu_checked.so python tools/sanitize.py [case ...]

Cases: ses, svm, refine, gen, balanced, baselines, vworld (default: all).  Each case goes through
the public API on small instances so the tool finishes in minutes; the kernels, grid
(148 CTAs) and code paths are the production ones.
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_09157_b200 import baselines, devgen, instances, ses, svm  # noqa: E402


def case_ses():
    inst = instances.gen_ses(3000, 17, 1, "uniform-ball")
    rep, sol = ses.solve_ses(inst, 1e-2)
    assert math.isfinite(sol.radius), sol


def case_svm():
    inst, _ = instances.gen_svm(1500, 1200, 10, 2, 1.0)
    rep, sol = svm.solve_svm(inst, 1e-2)
    assert math.isfinite(sol.margin), sol


def case_refine():
    # d = 100 (the BASELINE width) exercises the FULL kernels and the refine schedule
    inst = instances.gen_ses(2000, 100, 3, "gaussian")
    rep, sol = ses.solve_ses(inst, 1e-2)
    assert math.isfinite(sol.radius), sol


def case_gen():
    inst = devgen.gen_ses_device(4000, 33, 5, "uniform-ball")
    try:
        rep, sol = ses.solve_ses(inst, 3e-2)
        assert math.isfinite(sol.radius), sol
    finally:
        inst.close()
    inst = devgen.gen_svm_device(2000, 2000, 24, 6, 1.0)
    try:
        rep, sol = svm.solve_svm(inst, 3e-2)
        assert math.isfinite(sol.margin), sol
    finally:
        inst.close()


def case_balanced():
    # >= 64 warp tiles per SM: the calibrated per-SM contiguous partition (opt-in)
    os.environ["SCMWU_BALANCE"] = "1"
    inst = devgen.gen_ses_device(400000, 100, 4, "uniform-ball")
    try:
        rep, sol = ses.solve_ses(inst, 3e-2)
        assert math.isfinite(sol.radius), sol
    finally:
        inst.close()
    inst = devgen.gen_svm_device(200000, 200000, 100, 4, 1.0)
    try:
        rep, sol = svm.solve_svm(inst, 3e-2)
        assert math.isfinite(sol.margin), sol
    finally:
        inst.close()
    os.environ.pop("SCMWU_BALANCE")


def case_baselines():
    inst = instances.gen_ses(2000, 9, 7, "gaussian")
    r = baselines.meb_baseline(inst.centers, eps_base=0.05)
    assert math.isfinite(r.value)
    s, _ = instances.gen_svm(800, 700, 6, 8, 1.0)
    g = baselines.gilbert_baseline(s.P, s.Q, gap_tol=1e-4, max_iters=2000)
    assert math.isfinite(g.value)


def case_vworld():
    os.environ["SCMWU_VWORLD"] = "2"
    try:
        inst, _ = instances.gen_svm(1200, 1000, 12, 9, 1.0)
        rep, sol = svm.solve_svm(inst, 3e-2)
        assert math.isfinite(sol.margin), sol
    finally:
        del os.environ["SCMWU_VWORLD"]


CASES = {"ses": case_ses, "svm": case_svm, "refine": case_refine, "gen": case_gen,
         "balanced": case_balanced, "baselines": case_baselines, "vworld": case_vworld}


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"sanitize case {name}: ok", flush=True)
