"""One full time-to-eps solve of the C5 shape on one GPU (informational, not a bench line):
SVM n = 2e7 (1e7 + 1e7), d = 512, gap 1, eps = 1e-3, drawn in HBM (82 GB).

    python tools/c5_solve.py [--n1 N] [--eps E]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_09157_b200 import devgen, svm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n1", type=int, default=10 ** 7)
    ap.add_argument("--d", type=int, default=512)
    ap.add_argument("--eps", type=float, default=1e-3)
    a = ap.parse_args()
    t0 = time.perf_counter()
    inst = devgen.gen_svm_device(a.n1, a.n1, a.d, 0, 1.0)
    t1 = time.perf_counter()
    rep, sol = svm.solve_svm(inst, a.eps)
    t2 = time.perf_counter()
    bytes_pass = 8 * 2 * a.n1 * a.d
    out = {"workload": f"SVM n={2 * a.n1} d={a.d} gap 1 eps={a.eps}, generated in HBM, 1 GPU",
           "generate_s": t1 - t0, "solve_wall_s": t2 - t1, "kernel_s": rep.kernel_ms / 1e3,
           "iterations": rep.total_iterations, "search_steps": rep.search_steps,
           "passes": rep.passes, "termination": rep.termination.value,
           "us_per_pass": rep.kernel_ms * 1e3 / max(rep.passes, 1),
           "gbs": rep.passes * bytes_pass / (rep.kernel_ms * 1e-3) / 1e9,
           "margin": sol.margin, "pd_distance": sol.pd_distance}
    print(json.dumps(out), flush=True)
    inst.close()


if __name__ == "__main__":
    main()
