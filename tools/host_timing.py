import sys, time
sys.path.insert(0, ".")
import bench
from paper_2405_09157_b200 import ses, _native as nat
import torch
w = bench.WORKLOADS["ses_c2"]
inst = bench.make_instance(w, pinned=True)
D, _, _ = ses.ses_range(inst)
eng = nat.cuda_engine()
for rep in range(3):
    t0 = time.perf_counter()
    X = torch.empty((10**6, 100), dtype=torch.float64, device="cuda")  # warm the allocator path
    del X
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dev = ses.ses_device(inst, D)
    t2 = time.perf_counter()
    f = dev.progress(inst.centers[0])
    t3 = time.perf_counter()
    spec = ses.OracleSpec(dev.cone, 3 * D / 2 ** 0.5, 101, dev, 2 ** 0.5, ses.Orientation.MAX)
    from paper_2405_09157_b200 import meta
    r = meta.solve_ftp(spec, 0.99 * D, 1e-3, meta.EarlyStopConfig(), dev.progress, cap=64)
    t4 = time.perf_counter()
    r = meta.solve_ftp(spec, 0.99 * D, 1e-3, meta.EarlyStopConfig(), dev.progress, cap=64)
    t5 = time.perf_counter()
    dev.close()
    t6 = time.perf_counter()
    print(f"rep {rep}: create {t2-t1:.3f}  progress {t3-t2:.4f}  first ftp(64) {t4-t3:.3f} (kernel {r.kernel_ms/1e3:.4f})  second ftp {t5-t4:.3f}  close {t6-t5:.3f}", flush=True)
