"""Headline-regime solves (eps=1e-3, d=100) on the GPU next to the reference's recorded
solves of the same instances (tests/golden/headline/*.json): per-step records side by side.

    python tools/headline_probe.py [ses:1000 svm:2000 ...]
"""
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09157_b200 import instances, ses, svm  # noqa: E402


def main():
    want = sys.argv[1:] or ["ses:1000", "svm:2000"]
    for w in want:
        kind, n = w.split(":")
        n = int(n)
        refs = [json.load(open(f)) for f in
                sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "headline",
                                              f"{kind}_n{n}_t*.json")))]
        t0 = time.time()
        if kind == "ses":
            inst = instances.gen_ses(n, 100, 0, "uniform-ball")
            rep, sol = ses.solve_ses(inst, 1e-3)
            val = sol.radius
        else:
            inst, _ = instances.gen_svm(n // 2, n - n // 2, 100, 0, 1.0)
            rep, sol = svm.solve_svm(inst, 1e-3)
            val = (sol.margin, sol.pd_distance)
        wall = time.time() - t0
        print(f"== {kind} n={n}: GPU {rep.total_iterations} its, {rep.search_steps} steps, "
              f"{rep.termination.value}, value {val}, {wall:.2f} s")
        for r in refs:
            s = r["solve"]
            v = s.get("radius", (s.get("margin"), s.get("pd_distance")))
            print(f"   ref threads={r['threads']}: {s['iterations']} its, {s['steps']} steps, "
                  f"{s['termination']}, value {v}")
        ref_steps = refs[0]["solve"]["search"] if refs else []
        for i, st in enumerate(rep.steps):
            rs = ref_steps[i] if i < len(ref_steps) else None
            print(f"   step {i}: alpha {st.alpha:.10f} its {st.iterations:7d} {st.reason:12s}"
                  + (f" | ref alpha {rs[0]:.10f} its {rs[3]:7d} {rs[5]}" if rs else ""))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
