"""Quick end-to-end check of the CUDA engine against the golden fixtures (dev tool)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_09157_b200 import _native as nat, instances, ses, svm  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    eng = nat.cuda_engine()
    k = json.load(open(os.path.join(G, "kats.json")))
    th = np.linspace(0, 2 * np.pi, 32, endpoint=False)
    circ = ses.SesInstance(np.stack([np.cos(th), np.sin(th)], 1), np.zeros(32))
    t0 = time.time()
    r, s = ses.solve_ses(circ, 0.05, engine=eng)
    print("circle", s.radius, r.total_iterations, "ref", k["ses_circle32"]["radius"],
          k["ses_circle32"]["iterations"], f"{time.time()-t0:.2f}s", flush=True)
    inst = svm.SvmInstance(np.array([[1.0, 0.0]]), np.array([[-1.0, 0.0]]))
    r, s = svm.solve_svm(inst, 0.01, engine=eng)
    print("2pt", s.margin, s.pd_distance, r.total_iterations, flush=True)
    C = json.load(open(os.path.join(G, "calls.json")))
    for c in C:
        t0 = time.time()
        if c["kind"] == "ses":
            inst = instances.gen_ses(*c["inst"])
            r, s = ses.solve_ses(inst, c["eps"], engine=eng)
            print("ses", c["inst"][:2], s.radius, c["solve"]["radius"], r.total_iterations,
                  c["solve"]["iterations"], r.termination.value, f"{time.time()-t0:.2f}s",
                  f"kernel {r.kernel_ms:.1f}ms passes {r.passes}", flush=True)
        else:
            inst, _ = instances.gen_svm(*c["inst"])
            r, s = svm.solve_svm(inst, c["eps"], engine=eng)
            print("svm", c["inst"][:3], s.margin, c["solve"]["margin"], s.pd_distance,
                  c["solve"]["pd_distance"], r.total_iterations, c["solve"]["iterations"],
                  f"{time.time()-t0:.2f}s", f"kernel {r.kernel_ms:.1f}ms passes {r.passes}",
                  flush=True)


if __name__ == "__main__":
    main()
