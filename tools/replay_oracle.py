"""Replay recorded device calls (tools/record_calls.py) on the oracle — the reference's
algorithm restated on the CPU, bit-exact with it — with identical arguments, and print
each call's outcome side by side.

    python tools/replay_oracle.py calls.json [first_call [last_call]]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
from paper_2405_09157_b200 import instances  # noqa: E402


def gf(x):
    return float(x) if isinstance(x, str) else x


def main():
    rec = json.load(open(sys.argv[1]))
    a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    b = int(sys.argv[3]) if len(sys.argv) > 3 else len(rec["calls"])
    n = rec["n"]
    if rec["kind"] == "ses":
        inst = instances.gen_ses(n, rec.get("d", 100), rec.get("seed", 0),
                                 rec.get("dist", "uniform-ball"))
        pr = O.SesProblem(inst.centers, inst.radii)
        D, _, _ = pr.range()
        spec = pr.spec(3.0 * D / math.sqrt(2.0))
        d = rec.get("d", 100)
    else:
        inst, _ = instances.gen_svm(n // 2, n - n // 2, 100, 0, 1.0)
        pr = O.SvmProblem(inst.P, inst.Q)
        spec = pr.spec()
        d = 100
    prog = (lambda y: pr.progress(y[:d]))
    for k in range(a, b):
        c = rec["calls"][k]
        t0 = time.time()
        if c["fn"] == "ftp":
            r = O.ftp(spec, c["alpha"], c["eps"], c["delta"], c["patience"], c["enabled"], prog,
                      c["cap"])
        else:
            lo, hi = (gf(x) for x in c["bounds"])
            r = O.refine(spec, c["alpha"], c["horizon"], c["delta"], c["patience"],
                         c["enabled"], prog, c["gain_rel"], (lo, hi), c["target"])
        dv = c["result"]
        print(f"call {k} {c['fn']} alpha {c['alpha']:.10f} h {c.get('horizon')}: device "
              f"{dv['type'][:4]} {dv['iterations']} {dv.get('reason', 'sep')} best "
              f"{dv['best_progress']} | oracle {type(r).__name__[:4]} {r.iterations} "
              f"{getattr(r, 'reason', 'sep')} best {r.best_progress} ({time.time() - t0:.0f}s)",
              flush=True)


if __name__ == "__main__":
    main()
