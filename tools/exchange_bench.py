"""Cost of the per-pass rank exchange of the persistent kernel.

On one GPU the exchange protocol (peer stores of the pass vector into every rank's
mailbox, system-scope fence, release/acquire flags, rank-ordered fold) runs between
emulated ranks (SCMWU_VWORLD=W: CTA groups of one launch).  Pass vectors of 856 B (SES,
d = 100) and 8.3 KB (SVM, d = 512) on tiny instances, so a pass is almost only
synchronisation; the exchange cost is the difference to W = 1.  With >= 2 GPUs visible it
also times the NCCL all-gather of the same payloads (torchrun, one rank per GPU).

    python tools/exchange_bench.py            # emulated ranks on GPU 0
"""
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r"""
import math, os, sys
sys.path.insert(0, %(root)r)
from paper_2405_09157_b200 import instances, meta, ses, svm
kind, W = sys.argv[1], int(sys.argv[2])
if kind == "ses":
    inst = instances.gen_ses(148 * 32, 100, 0, "uniform-ball")
    dev = ses.ses_device(inst)
    D, L0, U0 = ses.ses_range(inst)
    spec = meta.OracleSpec(dev.cone, 3 * D / math.sqrt(2), 101, dev, math.sqrt(2),
                           meta.Orientation.MAX)
    alpha = U0
else:
    inst, _ = instances.gen_svm(148 * 16, 148 * 16, 512, 0, 1.0)
    dev = svm.svm_device(inst)
    D = inst.max_norm
    spec = meta.OracleSpec(dev.cone, 2 * D, 514, dev, 2.0, meta.Orientation.MIN,
                           counter_progress=True)
    alpha = 1e-3 * D
st = meta.EarlyStopConfig(enabled=False)
best = None
for _ in range(3):
    r = meta.refine_run(spec, alpha, 4096, st, dev.progress)
    us = r.kernel_ms * 1e3 / r.passes
    best = us if best is None else min(best, us)
print(f"RESULT {kind} W={W} grid={dev.handle.info()['grid']} {best:.2f}")
"""


def main():
    rows = []
    for kind in ("ses", "svm"):
        base = None
        for W in (1, 2, 4, 8):
            env = dict(os.environ)
            if W > 1:
                env["SCMWU_VWORLD"] = str(W)
            r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT}, kind, str(W)],
                               capture_output=True, text=True, env=env, timeout=600)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")]
            if not line:
                print(r.stderr[-2000:])
                continue
            us = float(line[0].split()[-1])
            base = us if W == 1 else base
            rows.append((kind, W, us, us - base))
            payload = (100 + 7) * 8 if kind == "ses" else (2 * 512 + 12) * 8
            print(f"{kind} payload {payload} B, {W} emulated rank(s): {us:.2f} us/pass "
                  f"(exchange +{us - base:.2f} us)", flush=True)


if __name__ == "__main__":
    main()
