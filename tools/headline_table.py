"""Device vs recorded reference solves for every family in tests/golden/headline/ (one
line per family: reference iterations per threads variant, device iterations, values).

    python tools/headline_table.py
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09157_b200 import instances, ses, svm  # noqa: E402


def main():
    groups = {}
    for f in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "headline", "*.json"))):
        rec = json.load(open(f))
        groups.setdefault((rec["kind"], tuple(rec["inst"]), rec["eps"]), []).append(rec)
    for (kind, args, eps), refs in sorted(groups.items(), key=lambda kv: (kv[0][0], str(kv[0][1]))):
        if kind == "ses":
            inst = instances.gen_ses(*args)
            rep, sol = ses.solve_ses(inst, eps)
            val, rv = sol.radius, [r["solve"]["radius"] for r in refs]
        else:
            inst, _ = instances.gen_svm(*args)
            rep, sol = svm.solve_svm(inst, eps)
            val, rv = sol.margin, [r["solve"]["margin"] for r in refs]
        its = [(r["threads"], r["solve"]["iterations"]) for r in refs]
        same = any([(s.iterations, s.reason) for s in rep.steps] ==
                   [(s[3], s[5]) for s in r["solve"]["search"]] for r in refs)
        print(f"| {kind} {args} eps={eps:g} | " + ", ".join(f"t{t}: {i:,}" for t, i in its)
              + f" | {rep.total_iterations:,} | {'identical steps' if same else 'differs'} | "
              f"{val:.10f} vs {', '.join(f'{v:.10f}' for v in rv)} |", flush=True)


if __name__ == "__main__":
    main()
