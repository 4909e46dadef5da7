"""Iteration counts of the configs[3] solve (SES n=10^7, d=100, eps=1e-3) under different
reduction orders (grid sizes): the spread of the chaotic trajectory (SURVEY finding 5).

    python tools/c4_variants.py [grid ...]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2405_09157_b200 import ses  # noqa: E402


def main():
    grids = [int(g) for g in sys.argv[1:]] or [0]
    w = dict(bench.WORKLOADS[os.environ.get("WORKLOAD", "ses_c4")])
    inst = bench.make_instance(w)
    for g in grids:
        dev = ses.ses_device(inst, grid=g) if w["kind"] == "ses" else None
        if dev is None:
            from paper_2405_09157_b200 import svm
            dev = svm.svm_device(inst, grid=g)
        t0 = time.time()
        rep, sol = bench.solve(w, inst, dev)
        val = sol.radius if w["kind"] == "ses" else sol.margin
        print(f"grid {dev.handle.info()['grid']}: {rep.total_iterations} its, "
              f"{rep.search_steps} steps, {rep.termination.value}, value {val:.12f}, "
              f"{time.time() - t0:.1f} s, {rep.kernel_ms / max(rep.passes, 1) * 1e3:.1f} "
              f"us/pass; steps " + " ".join(f"{s.iterations}{s.reason[0]}" for s in rep.steps),
              flush=True)
        dev.close()


if __name__ == "__main__":
    main()
