"""Record every feasibility test of a device solve (host-driven search, one call per test):
arguments and outcome, so each call can be replayed on the oracle (the reference's
algorithm on the CPU) with identical inputs.

    SCMWU_HOST_SEARCH=1 python tools/record_calls.py ses 10000 out.json [d seed dist]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SCMWU_HOST_SEARCH"] = "1"
from paper_2405_09157_b200 import instances, meta, ses, svm  # noqa: E402


def _f(x):
    if x is None:
        return None
    x = float(x)
    return "inf" if x == math.inf else "-inf" if x == -math.inf else x


def main():
    kind, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    d = int(sys.argv[4]) if len(sys.argv) > 4 else 100
    seed = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    dist = sys.argv[6] if len(sys.argv) > 6 else "uniform-ball"
    calls = []
    orig_ftp, orig_ref = meta.solve_ftp, meta.refine_run

    def rec(res):
        d = {"type": type(res).__name__, "iterations": res.iterations,
             "best_progress": _f(res.best_progress), "best_counter": _f(res.best_counter)}
        if isinstance(res, meta.DualFeasible):
            d.update(reason=res.reason, value=_f(res.value), eps_eff=_f(res.eps_eff))
        else:
            d.update(oracle_value=_f(res.oracle_value))
        return d

    def ftp(oracle, alpha, eps, stopping=None, progress=None, cap=None):
        r = orig_ftp(oracle, alpha, eps, stopping, progress, cap)
        calls.append({"fn": "ftp", "alpha": alpha, "eps": eps, "cap": cap,
                      "delta": stopping.delta, "patience": stopping.patience,
                      "enabled": stopping.enabled, "result": rec(r)})
        return r

    def ref(oracle, alpha, horizon, stopping, progress, gain_rel=None, bounds=None,
            target=None):
        r = orig_ref(oracle, alpha, horizon, stopping, progress, gain_rel, bounds, target)
        calls.append({"fn": "refine", "alpha": alpha, "horizon": horizon,
                      "gain_rel": gain_rel, "bounds": [_f(b) for b in bounds],
                      "target": target, "delta": stopping.delta,
                      "patience": stopping.patience, "enabled": stopping.enabled,
                      "result": rec(r)})
        return r

    meta.solve_ftp, meta.refine_run = ftp, ref
    if kind == "ses":
        inst = instances.gen_ses(n, d, seed, dist)
        rep, sol = ses.solve_ses(inst, 1e-3)
        val = sol.radius
    else:
        inst, _ = instances.gen_svm(n // 2, n - n // 2, 100, 0, 1.0)
        rep, sol = svm.solve_svm(inst, 1e-3)
        val = sol.margin
    json.dump({"kind": kind, "n": n, "d": d, "seed": seed, "dist": dist, "iterations": rep.total_iterations,
               "value": val, "lower": rep.primal_value, "calls": calls}, open(out, "w"),
              indent=1)
    print(kind, n, rep.total_iterations, val, len(calls))


if __name__ == "__main__":
    main()
