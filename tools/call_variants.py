"""Re-run one recorded device call (tools/record_calls.py) on the GPU under different
reduction orders (grid sizes) to see how sensitive its outcome is.

    python tools/call_variants.py calls.json K [grid ...]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_09157_b200 import instances, meta, ses  # noqa: E402


def main():
    rec = json.load(open(sys.argv[1]))
    k = int(sys.argv[2])
    grids = [int(g) for g in sys.argv[3:]] or [0]
    d = rec.get("d", 100)
    inst = instances.gen_ses(rec["n"], d, rec.get("seed", 0), rec.get("dist", "uniform-ball"))
    D, _, _ = ses.ses_range(inst)
    c = rec["calls"][k]
    for g in grids:
        dev = ses.ses_device(inst, grid=g)
        spec = meta.OracleSpec(dev.cone, 3.0 * D / math.sqrt(2.0), d + 1, dev, math.sqrt(2.0),
                               meta.Orientation.MAX)
        st = meta.EarlyStopConfig(delta=c["delta"], patience=c["patience"],
                                  enabled=c["enabled"])
        b = tuple(float(x) for x in c["bounds"]) if c["fn"] != "ftp" else None
        for da in (0.0, 1e-12, -1e-12, 1e-9):
            t0 = time.time()
            a = c["alpha"] * (1.0 + da)
            if c["fn"] == "ftp":    # a bracketing test (solve_ftp)
                r = meta.solve_ftp(spec, a, c["eps"], st, dev.progress, c["cap"])
            else:
                r = meta.refine_run(spec, a, c["horizon"], st, dev.progress,
                                    gain_rel=c["gain_rel"], bounds=b, target=c["target"])
            print(f"grid {dev.handle.info()['grid']} alpha*(1{da:+g}): {type(r).__name__} "
                  f"{r.iterations} {getattr(r, 'reason', 'sep')} best {r.best_progress} "
                  f"({time.time() - t0:.2f}s)", flush=True)
        dev.close()


if __name__ == "__main__":
    main()
