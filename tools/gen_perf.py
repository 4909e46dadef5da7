"""Per-pass throughput on device-generated instances, with clocks and power (dev tool).

    python tools/gen_perf.py ses N D [--horizon H] [--reps R] [--grid G]
    python tools/gen_perf.py svm N1 D [--horizon H] ...      (n2 = n1)
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["ses", "svm"])
    ap.add_argument("n", type=int)
    ap.add_argument("d", type=int)
    ap.add_argument("--horizon", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--dist", default="uniform-ball")
    a = ap.parse_args()
    if a.kind == "ses":
        w = dict(kind="ses", n=a.n, d=a.d, dist=a.dist, seed=0, eps=1e-3, horizon=a.horizon)
    else:
        w = dict(kind="svm", n1=a.n, n2=a.n, d=a.d, seed=0, gap=1.0, eps=1e-3,
                 horizon=a.horizon)
    t0 = time.time()
    inst = bench.gen_device(w, None, 0)
    if a.grid:
        inst.dev.handle.set_grid(a.grid)
    print(f"generate {time.time() - t0:.2f}s info {inst.dev.handle.info()}", flush=True)
    bpp = bench.alg_bytes_per_pass(w)
    bench.fixed_run(w, inst)
    for _ in range(a.reps):
        clk = bench.ClockSampler(0)
        clk.start()
        r = bench.fixed_run(w, inst)
        c = clk.stop()
        us = r.kernel_ms * 1e3 / max(r.passes, 1)
        print(f"{a.kind} n={a.n} d={a.d}: passes {r.passes} {us:.1f} us/pass "
              f"{bpp / us / 1e3:.0f} GB/s  sm {c['sm_mhz']} MHz power {c['power_w']} W "
              f"{c['reasons']}", flush=True)
    inst.close()


if __name__ == "__main__":
    main()
