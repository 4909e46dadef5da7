"""Where the e2e time of the default bench step goes (dev tool): host range D, handle
creation + upload, the solve, per phase wall time.

    python tools/e2e_breakdown.py [--pinned]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_09157_b200 import ses  # noqa: E402


def main():
    w = bench.WORKLOADS["ses_c2"]
    inst = bench.make_instance(w, pinned="--pinned" in sys.argv)
    for rep in range(3):
        t0 = time.perf_counter()
        D, _, _ = ses.ses_range(inst)
        t1 = time.perf_counter()
        dev = ses.ses_device(inst, D)
        t2 = time.perf_counter()
        rep_, sol = ses.solve_ses(inst, w["eps"], device=dev)
        t3 = time.perf_counter()
        dev.close()
        t4 = time.perf_counter()
        print(f"rep {rep}: range {t1 - t0:.3f}s  create+upload {t2 - t1:.3f}s  "
              f"solve {t3 - t2:.3f}s (kernel {rep_.kernel_ms / 1e3:.3f}s)  close {t4 - t3:.3f}s  "
              f"total {t4 - t0:.3f}s", flush=True)


if __name__ == "__main__":
    main()
