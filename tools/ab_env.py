"""Interleaved A/B of a launch-time knob (an SCMWU_* environment variable read by every
launch) on one resident instance: refine runs of H passes, rounds of all values in turn.

    python tools/ab_env.py ses_c4 SCMWU_L2_AHEAD 0,1,2,4 [--horizon 256] [--rounds 4]
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_09157_b200 import meta, ses, svm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("var")
    ap.add_argument("values")
    ap.add_argument("--horizon", type=int, default=256)
    ap.add_argument("--rounds", type=int, default=4)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    inst = bench.make_instance(w)
    if w["kind"] == "ses":
        dev = ses.ses_device(inst)
        D, L0, U0 = ses.ses_range(inst)
        spec = meta.OracleSpec(dev.cone, 3 * D / math.sqrt(2), w["d"] + 1, dev, math.sqrt(2),
                               meta.Orientation.MAX)
        alpha = 0.5 * (L0 + U0)
    else:
        dev = svm.svm_device(inst)
        spec = meta.OracleSpec(dev.cone, 2 * inst.max_norm, w["d"] + 2, dev, 2.0,
                               meta.Orientation.MIN, counter_progress=True)
        alpha = 0.3
    st = meta.EarlyStopConfig(enabled=False)
    bytes_pass = bench.alg_bytes_per_pass(w)
    vals = a.values.split(",")
    res = {v: [] for v in vals}
    ref = None
    meta.refine_run(spec, alpha, 16, st, dev.progress)   # warm-up
    for rnd in range(a.rounds):
        for v in vals:
            os.environ[a.var] = v
            r = meta.refine_run(spec, alpha, a.horizon, st, dev.progress)
            us = r.kernel_ms * 1e3 / max(r.passes, 1)
            res[v].append(us)
            key = (r.iterations, getattr(r, "value", None), getattr(r, "best_progress", None))
            ref = ref or key
            print(f"round {rnd} {a.var}={v}: {us:.2f} us/pass "
                  f"{bytes_pass / us / 1e3:.1f} GB/s iters {r.iterations}"
                  + ("" if key == ref else " (RESULT DIFFERS)"), flush=True)
    for v in vals:
        x = np.array(res[v])
        print(f"{a.var}={v}: median {np.median(x):.2f} us/pass, min {x.min():.2f}, "
              f"max {x.max():.2f}", flush=True)


if __name__ == "__main__":
    main()
