"""Where the non-kernel wall time of one solve goes (dev tool): every native call made
by solve_ses / solve_svm (sc_create, sc_solve or sc_ftp, sc_progress, sc_pd_pair, ...) is
timed on the host; prints per call wall vs kernel time and the host gaps between calls.

    python tools/solve_gaps.py [--reps 3] [--resident] [--workload ses_c2|svm_c3|...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_09157_b200 import ses, _native as nat  # noqa: E402

LOG = []


def wrap(name):
    fn = getattr(nat.Handle, name)

    def timed(self, *a, **k):
        t0 = time.perf_counter()
        out = fn(self, *a, **k)
        t1 = time.perf_counter()
        res = out[1] if isinstance(out, tuple) and len(out) == 4 else out   # sc_solve
        LOG.append((name, t0, t1, getattr(res, "kernel_ms", 0.0) / 1e3,
                    getattr(res, "passes", 0)))
        return out
    setattr(nat.Handle, name, timed)


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    for name in ("ftp", "solve", "progress", "iterate", "pd_pair", "close", "set_range"):
        wrap(name)
    create = nat.Engine.create

    def timed_create(self, *a, **k):
        t0 = time.perf_counter()
        out = create(self, *a, **k)
        LOG.append(("create", t0, time.perf_counter(), 0.0, 0))
        return out
    nat.Engine.create = timed_create
    rng = ses.ses_range

    def timed_range(*a, **k):
        t0 = time.perf_counter()
        out = rng(*a, **k)
        LOG.append(("range", t0, time.perf_counter(), 0.0, 0))
        return out
    ses.ses_range = timed_range
    wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "ses_c2"
    w = bench.WORKLOADS[wl]
    inst = bench.make_instance(w, pinned=True)
    from paper_2405_09157_b200 import svm
    dev = None
    if "--resident" in sys.argv:
        dev = ses.ses_device(inst) if w["kind"] == "ses" else svm.svm_device(inst)
    for rep in range(reps):
        LOG.clear()
        t0 = time.perf_counter()
        r, _ = bench.solve(w, inst, dev)
        t1 = time.perf_counter()
        calls = sum(c[2] - c[1] for c in LOG)
        kern = sum(c[3] for c in LOG)
        gaps = [(LOG[i][1] - LOG[i - 1][2], LOG[i - 1][0], LOG[i][0]) for i in range(1, len(LOG))]
        gaps.sort(reverse=True)
        first = LOG[0][1] - t0 if LOG else 0.0
        pre = {c[0]: c[2] - c[1] for c in LOG if c[0] in ("range", "create")}
        print(f"rep {rep}: total {t1 - t0:.3f}s  native calls {len(LOG)} wall {calls:.3f}s "
              f"(ftp kernel {kern:.3f}s)  before first call {first:.3f}s  "
              f"host gaps {sum(g[0] for g in gaps):.3f}s  "
              + "  ".join(f"{k} {v:.3f}s" for k, v in pre.items()), flush=True)
        slow = sorted(LOG, key=lambda c: (c[2] - c[1]) - c[3], reverse=True)[:5]
        for c in slow:
            print(f"   {c[0]:9s} wall {c[2] - c[1]:.4f}s kernel {c[3]:.4f}s passes {c[4]}")
        for g in gaps[:3]:
            print(f"   gap {g[0]:.4f}s  {g[1]} -> {g[2]}")


if __name__ == "__main__":
    main()
