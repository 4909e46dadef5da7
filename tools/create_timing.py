"""Handle creation cost against a plain pinned H2D copy of the same bytes (dev tool):

    python tools/create_timing.py [ses_c2|svm_c3]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_2405_09157_b200 import ses, svm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ses_c2"
w = bench.WORKLOADS[name]
inst = bench.make_instance(w, pinned=True)
if w["kind"] == "ses":
    D, _, _ = ses.ses_range(inst)
    x, nbytes = torch.from_numpy(inst.centers), inst.centers.nbytes
else:
    x, nbytes = torch.from_numpy(inst.P), inst.P.nbytes + inst.Q.nbytes
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = x.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del g
    dev = ses.ses_device(inst, D) if w["kind"] == "ses" else svm.svm_device(inst)
    t2 = time.perf_counter()
    dev.close()
    t3 = time.perf_counter()
    print(f"{name}: torch H2D of {x.numel() * 8 / 1e6:.0f} MB {t1 - t0:.4f}s  "
          f"create ({nbytes / 1e6:.0f} MB) {t2 - t1:.4f}s  close {t3 - t2:.4f}s", flush=True)
