"""Per-pass throughput of the persistent kernel on the BASELINE workloads (dev tool).

    python tools/gpu_perf.py [ses_c2|svm_c3|ses_c1|...] [--full] [--grid G]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_09157_b200 import meta, ses, svm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="ses_c2")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--horizon", type=int, default=2048)
    ap.add_argument("--ftp", action="store_true", help="solve_ftp (rung ladder) instead of refine")
    ap.add_argument("--alpha", type=float, default=None)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    t0 = time.time()
    inst = bench.make_instance(w)
    print(f"gen {time.time()-t0:.1f}s", flush=True)
    t0 = time.time()
    if w["kind"] == "ses":
        dev = ses.ses_device(inst, grid=a.grid)
        D, L0, U0 = ses.ses_range(inst)
        spec = meta.OracleSpec(dev.cone, 3 * D / math.sqrt(2), w["d"] + 1, dev, math.sqrt(2),
                               meta.Orientation.MAX)
        alpha = 0.5 * (L0 + U0)
    else:
        dev = svm.svm_device(inst, grid=a.grid)
        D = inst.max_norm
        spec = meta.OracleSpec(dev.cone, 2 * D, w["d"] + 2, dev, 2.0, meta.Orientation.MIN,
                               counter_progress=True)
        alpha = 0.3
    print(f"upload {time.time()-t0:.2f}s info {json.dumps(dev.handle.info())}", flush=True)
    st = meta.EarlyStopConfig(enabled=False)
    bytes_pass = bench.alg_bytes_per_pass(w)
    if a.alpha is not None:
        alpha = a.alpha
    for rep in range(3):
        if a.ftp:
            r = meta.solve_ftp(spec, alpha, 1e-9, st, dev.progress, a.horizon)
        else:
            r = meta.refine_run(spec, alpha, a.horizon, st, dev.progress)
        us = r.kernel_ms * 1e3 / max(r.passes, 1)
        print(f"refine h={a.horizon}: {type(r).__name__} iters {r.iterations} passes {r.passes} "
              f"kernel {r.kernel_ms:.1f} ms -> {us:.2f} us/pass, "
              f"{bytes_pass / us / 1e3:.1f} GB/s", flush=True)
        if os.environ.get("SCMWU_TIMING"):
            full = dev.handle.debug_timing()
            G = dev.handle.info()["grid"]
            per = full[9:9 + G] / max(r.passes, 1)
            sm = full[169:169 + G]
            if os.environ.get("SCMWU_DUMP"):
                with open(os.environ["SCMWU_DUMP"], "w") as fh:
                    json.dump({"cycles_per_pass": per.tolist(), "smid": sm.tolist()}, fh)
            if per.max() > 0:
                order = np.argsort(per)
                print(f"  per-CTA streaming cycles/pass: min {per.min():.0f} median "
                      f"{np.median(per):.0f} max {per.max():.0f}; slowest CTAs (cta:sm) "
                      + " ".join(f"{i}:{int(sm[i])}" for i in order[-6:])
                      + "; fastest " + " ".join(f"{i}:{int(sm[i])}" for i in order[:4]),
                      flush=True)
                h = G // 2
                print("  mean cycles/pass first half %.0f second half %.0f; by decile: %s"
                      % (per[:h].mean(), per[h:].mean(),
                         " ".join("%.0f" % per[i * G // 10:(i + 1) * G // 10].mean()
                                  for i in range(10))), flush=True)
            gs, ge = full[329:329 + G], full[489:489 + G]
            if gs.max() > 0:
                base = gs.min()
                print(f"  last pass, global ns: start spread {gs.max() - gs.min():.0f}, end "
                      f"spread {ge.max() - ge.min():.0f}, CTA0 start +{gs[0] - base:.0f} end "
                      f"+{ge[0] - base:.0f}, latest start CTA {int(np.argmax(gs))}, latest end "
                      f"CTA {int(np.argmax(ge))} (+{ge.max() - base:.0f})", flush=True)
            ga, gr = full[649:649 + G], full[809:809 + G]
            if ga.max() > 0:
                la = ga.max()
                print(f"  last pass, first barrier: arrival spread {ga.max() - ga.min():.0f} ns, "
                      f"CTA0 arrives {la - ga[0]:.0f} ns before the last; release after the "
                      f"last arrival: min {(gr - la).min():.0f} median {np.median(gr - la):.0f} "
                      f"max {(gr - la).max():.0f} ns; last arriver CTA {int(np.argmax(ga))}",
                      flush=True)
            ts = full[969:976] / max(r.passes, 1)
            if ts.sum() > 0:
                print("  tail sections cycles/pass: finish_iteration %.0f, oracle epilogue %.0f,"
                      " update loops %.0f, window %.0f, checks+shift %.0f, write_pass %.0f"
                      % tuple(ts[1:7]), flush=True)
            t = full[:9] / max(r.passes, 1)
            names = ["pass", "join", "cta_part", "bar1", "fold", "bar2", "red_read", "tail",
                     "tail_join"]
            tot = t.sum()
            print("  cycles/pass (CTA0 thread0): " + ", ".join(
                f"{n}={v:.0f}" for n, v in zip(names, t)) + f"  total={tot:.0f} "
                f"(~{tot / 1.9e3:.2f} us at 1.9 GHz)", flush=True)
    if a.full:
        dev.close()
        t0 = time.time()
        rep, sol = bench.solve(w, inst, None)
        print(f"full solve {time.time()-t0:.1f}s iters {rep.total_iterations} steps "
              f"{rep.search_steps} {rep.termination.value} kernel {rep.kernel_ms/1e3:.1f}s "
              f"passes {rep.passes} result "
              f"{sol.radius if w['kind']=='ses' else sol.margin}", flush=True)
        for s in rep.steps:
            print("  ", s, flush=True)


if __name__ == "__main__":
    main()
