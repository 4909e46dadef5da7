"""Benchmark: time-to-eps of the SCMWU solvers on the B200 engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ses_c4|svm_c4|ses_c2|...]
    python bench.py --impl reference ...      # CPU reference arm (the reference itself)

A *step* is one full solve (adaptive search to the reference's stopping rule) of the
largest single-GPU configuration of BASELINE.json: by default configs[3], SES
n=10^7, d=100 uniform-ball points (the reference's own generator), eps=1e-3.  With
--gpus N (N > 1) the rows are sharded over N ranks (one process per GPU; spawned
through torch.distributed.run when WORLD_SIZE is not set).

value    time-to-eps with the instance resident in HBM: the solve part of every step,
         device-timed with CUDA events on the engine's stream (host gaps between the
         kernel launches included), mean over the K steps, max over ranks.
e2e      the same steps end to end through the public API from pinned host memory:
         upload of X, the solve, results read back, device memory released.
roofline HBM roofline of the persistent kernel: algorithmic bytes 8 n (d+1) (SES) or
         8 n d (SVM) per streaming pass x passes / kernel event time, against
         MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference's own CPU path (baseline/_ref, else the oracle port) timed
         on this host on a row sample of the workload, scaled linearly in rows, times
         the reference's own iteration count for the workload's family
         (tests/golden/headline/).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "ses_c2": dict(kind="ses", n=10 ** 6, d=100, dist="uniform-ball", seed=0, eps=1e-3,
                   desc="SES n=10^6 d=100 uniform-in-ball points, eps=1e-3 (BASELINE configs[1])"),
    "svm_c3": dict(kind="svm", n1=500_000, n2=500_000, d=100, seed=0, gap=1.0, eps=1e-3,
                   desc="hard-margin SVM n=10^6 (5e5+5e5) d=100 gap 1, eps=1e-3 (configs[2])"),
    "ses_d100_small": dict(kind="ses", n=4_000, d=100, dist="uniform-ball", seed=0, eps=1e-3,
                           desc="SES n=4000 d=100 (shared-memory resident; diagnostics)"),
    "ses_c1": dict(kind="ses", n=10_000, d=10, dist="gaussian", seed=0, eps=1e-2,
                   desc="SES n=10^4 d=10 Gaussian, eps=1e-2 (configs[0])"),
    "ses_c4": dict(kind="ses", n=10 ** 7, d=100, dist="uniform-ball", seed=0, eps=1e-3,
                   desc="SES n=10^7 d=100 uniform-in-ball points, eps=1e-3 (BASELINE "
                        "configs[3], the largest single-GPU config; north_star n=10^7 d=100)"),
    "svm_c4": dict(kind="svm", n1=5 * 10 ** 6, n2=5 * 10 ** 6, d=100, seed=0, gap=1.0,
                   eps=1e-3,
                   desc="hard-margin SVM n=10^7 (5e6+5e6) d=100 gap 1, eps=1e-3 (north_star "
                        "n=10^7 d=100)"),
    # drawn on the device (devgen, sc_create_generated): no host copy of X exists
    "ses_c4_gen": dict(kind="ses", n=10 ** 7, d=100, dist="uniform-ball", seed=0, eps=1e-3,
                       generated=True,
                       desc="SES n=10^7 d=100 uniform-in-ball, eps=1e-3 (configs[3]), "
                            "generated on the device"),
    "svm_c5_gen": dict(kind="svm", n1=10 ** 7, n2=10 ** 7, d=512, seed=0, gap=1.0, eps=1e-3,
                       generated=True, horizon=64,
                       desc="SVM n=2x10^7 d=512 gap 1 (configs[4], 81.9 GB fp64), generated "
                            "on the device; per-iteration HBM GB/s over a 64-iteration "
                            "refine run"),
}
# Read-only streaming ceiling of the kernel's own access pattern on B200 (per-warp bulk-copy
# rings, no math; tools/stream_bench.cu, profiles/r01_overhead.md).  MEASURED_PEAKS.json's
# hbm_gbs is a copy (read + write) figure; a read-only kernel can exceed it.
READ_CEILING_GBS = 7400.0


def make_instance(w, pinned=False):
    """The workload's instance; ``pinned`` places the point arrays in page-locked host
    memory (the e2e contract: inputs are copied to the device from pinned memory)."""
    from paper_2405_09157_b200 import instances, ses, svm
    if w["kind"] == "ses":
        inst = instances.gen_ses(w["n"], w["d"], w["seed"], w["dist"])
    else:
        inst, _ = instances.gen_svm(w["n1"], w["n2"], w["d"], w["seed"], w["gap"])
    if not pinned:
        return inst

    def pin(a):
        import torch
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        out = t.numpy()          # shares the pinned buffer; `t` is kept alive below
        out[...] = a
        return out, t

    if w["kind"] == "ses":
        (c, tc), (r, tr) = pin(inst.centers), pin(inst.radii)
        inst = ses.SesInstance(centers=c, radii=r)
        make_instance._keep = (tc, tr)
    else:
        (P, tp), (Q, tq) = pin(inst.P), pin(inst.Q)
        inst = svm.SvmInstance(P=P, Q=Q)
        make_instance._keep = (tp, tq)
    return inst


def alg_bytes_per_pass(w):
    if w["kind"] == "ses":
        return 8 * w["n"] * (w["d"] + 1)
    return 8 * (w["n1"] + w["n2"]) * w["d"]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                pw.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU (oracle port) sample
def cpu_sample(w, inst, max_seconds=20.0, max_iters=100_000):
    """Time the oracle port for a bounded number of MWU iterations of the workload:
    one polish run (refine_run, stopping disabled) at the feasible end of the range,
    which never separates, so exactly `horizon` iterations (>= ceil(ln r)) run."""
    import oracle as O
    t_setup = time.perf_counter()
    if w["kind"] == "ses":
        prob = O.SesProblem(inst.centers, inst.radii)
        D, L0, U0 = prob.range()
        spec = prob.spec(3.0 * D / math.sqrt(2.0))
        alpha = U0
    else:
        prob = O.SvmProblem(inst.P, inst.Q)
        spec = prob.spec()
        alpha = 1e-3 * prob.D
    progress = (lambda y: prob.progress(y[:w["d"]]))
    setup = time.perf_counter() - t_setup
    # the shortest run refine_run allows is ceil(ln r) iterations; when that is cheap,
    # run again with as many iterations as fit in max_seconds
    t0 = time.perf_counter()
    res = O.refine(spec, alpha, 1, 1e-4, 10, False, progress)
    dt = time.perf_counter() - t0
    per = dt / res.iterations
    if dt < 0.1 * max_seconds:
        k = int(min(max_iters, max_seconds / max(per, 1e-9)))
        if k > res.iterations:
            t0 = time.perf_counter()
            res = O.refine(spec, alpha, k, 1e-4, 10, False, progress)
            dt = time.perf_counter() - t0
    return {"s_per_iter": dt / res.iterations, "iters": res.iterations, "seconds": dt,
            "setup_s": setup}


REF_ROOT = os.path.join(ROOT, "baseline", "_ref")


def _ref_cores(w):
    """Host threads the reference's CPU path uses: SES is numpy element-wise work plus numba
    loops (one thread); SVM's GEMVs run on OpenBLAS's default thread count."""
    if w["kind"] == "ses":
        return 1
    threads_env = os.environ.get("OPENBLAS_NUM_THREADS") or os.environ.get("OMP_NUM_THREADS")
    return int(threads_env) if threads_env else (os.cpu_count() or 1)


def reference_counts(w):
    """The reference's own iteration count for the workload's family (same kind, d, eps,
    distribution), from the largest recorded solve in tests/golden/headline/ (recorded by
    tests/golden/make_golden.py headline from the reference itself).  Returns
    (iterations, n of that record, threads variants)."""
    import glob
    best = None
    recs = []
    for f in glob.glob(os.path.join(ROOT, "tests", "golden", "headline", "*.json")):
        try:
            recs.append(json.load(open(f)))
        except (OSError, ValueError):
            continue
    try:   # the eps = 1e-2 solves (configs[0] family), threads 1/2/4/8
        recs += json.load(open(os.path.join(ROOT, "tests", "golden", "long.json")))
    except (OSError, ValueError):
        pass
    for rec in recs:
        if rec["kind"] != w["kind"] or rec["eps"] != w["eps"]:
            continue
        if w["kind"] == "ses":
            n = rec["inst"][0]
            if rec["inst"][1] != w["d"] or rec["inst"][3] != w.get("dist", "uniform-ball"):
                continue
        else:
            n = rec["inst"][0] + rec["inst"][1]
            if rec["inst"][2] != w["d"]:
                continue
        its = rec["solve"]["iterations"]
        th = rec.get("threads", 1)
        if best is None or n > best[1]:
            best = [its, n, [th]]
        elif n == best[1]:
            best[2].append(th)
            if th == 1:            # the reference's default (RunConfig.threads = 1)
                best[0] = its
    return best


def _import_reference():
    """The unmodified reference package installed into baseline/_ref (pip --target, see
    DESIGN.md §8); None when it is not installed (the oracle port is timed instead)."""
    if not os.path.isdir(os.path.join(REF_ROOT, "symcone")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench_ref")
    if REF_ROOT not in sys.path:
        sys.path.insert(0, REF_ROOT)
    try:
        import symcone  # noqa: F401
        from symcone import meta as rmeta, ses as rses, svm as rsvm
        return rmeta, rses, rsvm
    except Exception as exc:   # noqa: BLE001 - report and fall back to the port
        print(f"bench: reference import failed ({exc}); timing the oracle port",
              file=sys.stderr)
        return None


def ref_sample(w, inst, iters):
    """`iters` MWU iterations of the REFERENCE (its own refine_run, oracle and learner,
    R/meta.py:457-573) on `inst`: one polish run at the feasible end of the range with
    stopping disabled, so exactly `iters` iterations run (no separation).  Returns
    seconds per iteration."""
    ref = _import_reference()
    rmeta, rses, rsvm = ref
    d = w["d"]
    if w["kind"] == "ses":
        rinst = rses.SesInstance(centers=inst.centers, radii=inst.radii)
        D, L0, U0 = rses.ses_range(rinst)
        cone = rses.ses_cone(rinst.n, d)
        buf = __import__("numpy").empty(cone.ambient_dim)
        spec = rmeta.OracleSpec(cone=cone, width_rho=3.0 * D / math.sqrt(2.0), dual_dim=d + 1,
                                query=lambda p, a: rses.ses_oracle(rinst, p, a, out=buf),
                                trace_bound=math.sqrt(2.0),
                                orientation=rmeta.Orientation.MAX)
        progress = (lambda y: rses.ses_progress(rinst, y[:d]))
        alpha = U0
    else:
        rinst = rsvm.SvmInstance(P=inst.P, Q=inst.Q)
        D = rinst.max_norm
        n = rinst.n1 + rinst.n2
        spec = rmeta.OracleSpec(cone=rsvm.svm_cone(n), width_rho=2.0 * D, dual_dim=d + 2,
                                query=lambda p, a: rsvm.svm_oracle(rinst, p, a),
                                trace_bound=2.0, orientation=rmeta.Orientation.MIN)
        progress = (lambda y: rsvm.svm_progress(rinst, y[:d]))
        alpha = 1e-3 * D
    stop = rmeta.EarlyStopConfig(enabled=False)
    t0 = time.perf_counter()
    r = rmeta.refine_run(spec, alpha, iters, stop, progress)
    dt = time.perf_counter() - t0
    return dt / r.iterations, r.iterations, dt


def _sample_rows(w):
    """Row sample of a workload for the CPU arms: at most 10^5 rows (SES) / 10^5 (SVM) of
    the same distribution, drawn by the reference's generator; per-iteration time scales
    linearly in the rows (each iteration is a fixed number of passes over them)."""
    ws = dict(w)
    if w["kind"] == "ses":
        ws["n"] = min(w["n"], 100_000)
        factor = w["n"] / ws["n"]
    else:
        ws["n1"], ws["n2"] = min(w["n1"], 50_000), min(w["n2"], 50_000)
        factor = (w["n1"] + w["n2"]) / (ws["n1"] + ws["n2"])
    return ws, factor


def reference_arm(args, w, rank):
    """--impl reference: the reference's own CPU implementation of the path on this host.

    Each step times a bounded sample: `refine_run` of the unmodified reference
    (baseline/_ref; the oracle port when it is not installed) on a row sample of the
    workload, scaled linearly to the full row count, times the reference's own iteration
    count for the workload's family (the largest recorded reference solve of the same
    kind, d, distribution and eps; tests/golden/headline/).  A full CPU solve at these
    sizes takes days."""
    if rank != 0:
        return
    t0 = time.perf_counter()
    ws, factor = _sample_rows(w)
    inst = make_instance(ws)
    use_ref = _import_reference() is not None
    if use_ref:
        try:                     # the reference runs here (numba JIT included), or the port
            ref_sample(ws, inst, 1)
        except Exception as exc:  # noqa: BLE001
            print(f"bench: the reference failed on this host ({exc}); timing the oracle port",
                  file=sys.stderr)
            use_ref = False
    kind = "reference" if use_ref else "port"
    fixed = w.get("horizon") is not None   # per-iteration GB/s workloads (C5 shape)
    counts = reference_counts(w)
    if counts is None and not fixed:
        raise SystemExit("no reference iteration count recorded for this workload family "
                         "(tests/golden/headline/)")
    iters, n_rec, threads = counts if counts else (0, 0, [])

    def sample(k):
        if use_ref:
            return ref_sample(ws, inst, k)
        s = cpu_sample(ws, inst, max_seconds=args.cpu_seconds, max_iters=k)
        return s["s_per_iter"], s["iters"], s["seconds"]

    for _ in range(max(1, args.warmup)):   # includes the numba JIT of the reference
        sample(1)
    # size the per-step sample to ~cpu_seconds of work (>= ceil(ln r) iterations)
    spi0, _, _ = sample(1)
    k = max(1, int(args.cpu_seconds / max(spi0, 1e-9)))
    spis = []
    for _ in range(args.steps):
        spi, got, _ = sample(k)
        spis.append(spi)
    spi = statistics.median(spis) * factor
    value = spi * iters
    metric, unit, hib = "time-to-eps (s)", "s", False
    if fixed:
        value = alg_bytes_per_pass(w) / spi / 1e9
        metric, unit, hib = "per-iteration HBM GB/s", "GB/s", True
    rows = ws["n"] if w["kind"] == "ses" else ws["n1"] + ws["n2"]
    cores = _ref_cores(w)
    desc = (f"{got} MWU iterations per step (one refine_run of the "
            f"{'unmodified reference, baseline/_ref' if use_ref else 'oracle port'}) on a "
            f"{rows}-row sample of the workload's distribution, {spi / factor:.4f} s/iter "
            f"scaled x{factor:g} to the full rows = {spi:.3f} s/iter; " +
            ("GB/s = algorithmic bytes per iteration / s" if fixed else
             f"x {iters} iterations = the reference's own count for this family (its "
             f"recorded solve at n={n_rec}, threads {sorted(threads)}; "
             f"tests/golden/headline/)"))
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": spi * 1000.0, "higher_is_better": hib, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"],
                   "reference_iterations": iters, "reference_iterations_n": n_rec,
                   "s_per_iter": spi},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def solve(w, inst, device=None):
    from paper_2405_09157_b200 import ses, svm
    if w["kind"] == "ses":
        return ses.solve_ses(inst, w["eps"], device=device)
    return svm.solve_svm(inst, w["eps"], device=device)


def _shared_instance(w, rank, comm):
    """Multi-rank runs: rank 0 draws the instance with the reference's generator and
    writes it to /dev/shm; every rank memory-maps it (each uploads only its own rows)."""
    from paper_2405_09157_b200 import instances
    import torch.distributed as tdist
    tag = (f"scmwu_bench_{w['kind']}_{w.get('n', 0)}_{w.get('n1', 0)}_{w.get('n2', 0)}_"
           f"{w['d']}_{w['seed']}.npyd")
    path = os.path.join("/dev/shm", tag)
    if rank == 0 and not os.path.isdir(path):
        instances.save(path, make_instance(w))
    tdist.barrier()
    return instances.load(path)


def exchange_latency_us(w, world, reps=200):
    """Latency of the per-pass exchange payload (the reduced pass vector: d+7 doubles SES,
    2d+12 SVM; 864 B / 8.3 KB at d = 100 / 512) as an NCCL all-gather over this node's
    NVLink, CUDA-event timed on the current stream, max over ranks.  It feeds the
    HBM+NVLink roofline of a sharded run."""
    import torch
    import torch.distributed as tdist
    rw = w["d"] + 7 if w["kind"] == "ses" else 2 * w["d"] + 12
    x = torch.zeros(rw, dtype=torch.float64, device="cuda")
    out = torch.empty(world * rw, dtype=torch.float64, device="cuda")
    for _ in range(20):
        tdist.all_gather_into_tensor(out, x)
    torch.cuda.synchronize()
    tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tdist.all_gather_into_tensor(out, x)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], device="cuda")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item()), rw * 8


def our_arm(args, w, rank, world):
    import torch
    from paper_2405_09157_b200 import ses, svm
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    t_gen = time.perf_counter()
    comm = None
    if dist:
        from paper_2405_09157_b200 import shard
        comm = shard.Comm()
        inst = _shared_instance(w, rank, comm)
    else:
        inst = make_instance(w, pinned=torch.cuda.is_available())
    gen_s = time.perf_counter() - t_gen

    def make_device():
        if comm is not None:   # row-sharded: this rank's rows, in-kernel NVLink exchange
            return (shard.ses_device_sharded(inst, comm, device=local) if w["kind"] == "ses"
                    else shard.svm_device_sharded(inst, comm, device=local))
        return (ses.ses_device(inst, device=local) if w["kind"] == "ses"
                else svm.svm_device(inst, device=local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    def step():
        """One step through the public API from host arrays: upload the instance (pinned
        host memory -> HBM), solve to the reference's stopping rule, read the results
        back, release the device memory.  The solve part is also timed on the device
        (CUDA events on the engine's stream, from the moment X is resident)."""
        t0 = time.perf_counter()
        dev = make_device()
        dev.handle.mark(0)
        rep, sol = solve(w, inst, dev)
        dev.handle.mark(1)
        dev_s = dev.handle.elapsed_ms() / 1000.0
        info = dev.handle.info()
        launches = dev.handle.launches()
        dev.close()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, dev_s, rep, sol, info, launches

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    times, e2e_times, reports, launches = [], [], [], 0
    info = None
    for _ in range(args.steps):
        e2e_s, dev_s, rep, sol, info, nl = step()
        times.append(dev_s)
        e2e_times.append(e2e_s)
        reports.append((rep, sol))
        launches += nl
    barrier()
    clk = clocks.stop()
    t_step = sum(times) / len(times)   # the K timed steps / K (then max over ranks)
    e2e = sum(e2e_times) / len(e2e_times)
    if dist:
        t = torch.tensor([t_step, e2e], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t_step, e2e = float(t[0].item()), float(t[1].item())
    print(f"bench: e2e per step {['%.3f' % t for t in e2e_times]} s; solve (device) "
          f"{['%.3f' % t for t in times]} s", file=sys.stderr)
    kernel_s = sum(r.kernel_ms for r, _ in reports) / 1000.0
    passes = sum(r.passes for r, _ in reports)
    width_passes = sum(r.width_passes for r, _ in reports)
    rep_e, _ = reports[-1]
    if w["kind"] == "ses":
        h2d = (inst.centers.nbytes + inst.radii.nbytes) // world
        d2h = (w["d"] + 1) * 8 * 2 * rep_e.search_steps + 8 * 4
    else:
        h2d = (inst.P.nbytes + inst.Q.nbytes) // world
        d2h = (w["d"] + 2) * 8 * 2 * rep_e.search_steps + inst.n1 * 8 + inst.n2 * 8

    peak, peak_kind = measured_peak()
    bpp = alg_bytes_per_pass(w) // world
    achieved = passes * bpp / kernel_s / 1e9 if kernel_s > 0 else 0.0
    rep0, sol0 = reports[-1]
    nvl = None
    if dist:
        # HBM+NVLink roofline: every pass streams this rank's rows at the HBM peak and
        # pays one exchange of the pass vector
        t_x, xbytes = exchange_latency_us(w, world)
        per_step = passes / len(reports)
        ideal = per_step * (bpp / (peak * 1e9) + t_x * 1e-6)
        nvl = {"exchange_bytes": xbytes, "t_exchange_us": t_x,
               "measured": "NCCL all-gather of the pass vector, CUDA events, max over ranks",
               "ideal_s_per_step": ideal, "frac": ideal / t_step if t_step > 0 else None}
    iters = [r.total_iterations for r, _ in reports]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_pass")
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": "time-to-eps (s)", "value": t_step, "unit": "s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1000.0,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (the reference's generator, instances.gen_ses / gen_svm)",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"],
                   "parallelism": (f"row-sharded x{world} (in-kernel NVLink exchange)"
                                   if world > 1 else "1 GPU"),
                   "iterations": rep0.total_iterations,
                   "iterations_all_steps": sorted(set(iters)),
                   "search_steps": rep0.search_steps,
                   "termination": rep0.termination.value,
                   "l2": "inputs larger than L2 (X = %.0f MB)" % (alg_bytes_per_pass(w) / 1e6)
                   if alg_bytes_per_pass(w) > 126e6 else "inputs fit in L2",
                   "kernel": info, "generate_s": gen_s,
                   "timing": "each step: upload from pinned host memory + solve + results "
                             "read back + release (e2e, wall clock); value = the solve part "
                             "on the device (CUDA events on the engine stream, X resident)"},
        "result": ({"radius": sol0.radius, "lower": rep0.primal_value,
                    "enclosure_slack": sol0.enclosure_slack} if w["kind"] == "ses" else
                   {"margin": sol0.margin, "pd_distance": sol0.pd_distance}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "read_ceiling": READ_CEILING_GBS,
                     "frac_of_read_ceiling": achieved / READ_CEILING_GBS,
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_pass": bpp,
                     "us_per_pass": kernel_s / passes * 1e6 if passes else None,
                     "kernel_s": kernel_s, "passes": passes,
                     "exact_width_passes": width_passes},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if nvl is not None:
        line["roofline"]["hbm_nvlink"] = nvl
    if rank == 0 and not args.no_cpu_baseline:
        spi, desc, kind = cpu_scaled(w, args.cpu_seconds)
        counts = reference_counts(w)
        its, note = ((counts[0], f"the reference's own count for this family (recorded solve "
                                 f"at n={counts[1]})") if counts else
                     (rep0.total_iterations, "the GPU solve's count"))
        line["cpu_baseline"] = {
            "value": spi * its, "unit": "s", "cores": _ref_cores(w), "kind": kind,
            "sample": f"{desc}; x {its} iterations = {note}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


# ------------------------------------------------------------------ device-generated workloads
def gen_device(w, comm, local):
    from paper_2405_09157_b200 import devgen
    if w["kind"] == "ses":
        return devgen.gen_ses_device(w["n"], w["d"], w["seed"], w["dist"], device=local,
                                     comm=comm)
    return devgen.gen_svm_device(w["n1"], w["n2"], w["d"], w["seed"], w["gap"], device=local,
                                 comm=comm)


def fixed_run(w, inst):
    """One refine_run of exactly w['horizon'] iterations (stopping disabled) at the
    feasible end of the range, so it never separates: a fixed amount of streaming work."""
    from paper_2405_09157_b200 import meta
    dev = inst.dev
    if w["kind"] == "ses":
        spec = meta.OracleSpec(dev.cone, 3.0 * inst.D / math.sqrt(2.0), w["d"] + 1, dev,
                               math.sqrt(2.0), meta.Orientation.MAX)
        alpha = inst.D
    else:
        spec = meta.OracleSpec(dev.cone, 2.0 * inst.D, w["d"] + 2, dev, 2.0,
                               meta.Orientation.MIN, counter_progress=True)
        alpha = 1e-3 * inst.D
    return meta.refine_run(spec, alpha, w["horizon"], meta.EarlyStopConfig(enabled=False),
                           dev.progress)


def gen_arm(args, w, rank, world):
    import torch
    dist = world > 1
    comm = None
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        from paper_2405_09157_b200 import shard
        comm = shard.Comm()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    fixed = w.get("horizon") is not None

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    def vmax(x):
        if not dist:
            return x
        t = torch.tensor([x], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    def step(inst):
        return fixed_run(w, inst) if fixed else solve(w, inst)

    t0 = time.perf_counter()
    inst = gen_device(w, comm, local)
    gen_s = time.perf_counter() - t0
    h = inst.dev.handle
    info = h.info()
    for _ in range(args.warmup):
        step(inst)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    l0 = h.launches()
    times, outs = [], []
    for _ in range(args.steps):
        h.mark(0)
        outs.append(step(inst))
        h.mark(1)
        times.append(h.elapsed_ms() / 1000.0)
    barrier()
    launches = h.launches() - l0
    clk = clocks.stop()
    t_step = vmax(sum(times) / len(times))   # the K timed steps / K, max over ranks
    if fixed:
        kernel_s = sum(r.kernel_ms for r in outs) / 1000.0
        passes = sum(r.passes for r in outs)
        iters = outs[-1].iterations
    else:
        kernel_s = sum(r.kernel_ms for r, _ in outs) / 1000.0
        passes = sum(r.passes for r, _ in outs)
        iters = outs[-1][0].total_iterations
    inst.close()
    # e2e through the public API: generate on the device + the step, host results read back
    barrier()
    t0 = time.perf_counter()
    inst_e = gen_device(w, comm, local)
    out_e = step(inst_e)
    inst_e.close()
    torch.cuda.synchronize()
    e2e_s = vmax(time.perf_counter() - t0)
    bpp = alg_bytes_per_pass(w)
    peak, peak_kind = measured_peak()
    achieved = passes * bpp / kernel_s / 1e9 if kernel_s > 0 else 0.0
    if fixed:
        # per-iteration HBM throughput of the whole job (all ranks' rows)
        value = passes / args.steps * bpp / t_step / 1e9
        metric, unit, hib = "per-iteration HBM GB/s", "GB/s", True
        e2e_v = passes / args.steps * bpp / e2e_s / 1e9
        sd = w["d"] + (1 if w["kind"] == "ses" else 2)
        d2h = 2 * sd * 8
    else:
        value, metric, unit, hib, e2e_v = t_step, "time-to-eps (s)", "s", False, e2e_s
        rep_e = out_e[0]
        d2h = (w["d"] + 2) * 8 * 2 * rep_e.search_steps + 8 * 4
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_pass")
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1000.0, "higher_is_better": hib,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, drawn on the device (Philox; same distribution as gen_ses/gen_svm)",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"],
                   "parallelism": (f"row-sharded x{world} (in-kernel NVLink exchange)"
                                   if world > 1 else "1 GPU"),
                   "iterations": iters, "generate_s": gen_s,
                   "l2": "inputs larger than L2 (X = %.0f MB)" % (bpp / 1e6), "kernel": info},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "read_ceiling": READ_CEILING_GBS,
                     "frac_of_read_ceiling": achieved / READ_CEILING_GBS,
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_pass": bpp,
                     "us_per_pass": kernel_s / passes * 1e6 if passes else None,
                     "kernel_s": kernel_s, "passes": passes},
        "e2e": {"value": e2e_v, "unit": unit, "h2d_bytes_per_step":
                8 * w["d"] if w["kind"] == "svm" else 0, "d2h_bytes_per_step": int(d2h),
                "note": "generation on the device + the step; X never exists on the host"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and not args.no_cpu_baseline:
        spi, desc, kind = cpu_scaled(w, args.cpu_seconds)
        counts = None if fixed else reference_counts(w)
        its = counts[0] if counts else iters
        cv = bpp / spi / 1e9 if fixed else spi * its
        line["cpu_baseline"] = {
            "value": cv, "unit": unit, "cores": _ref_cores(w), "kind": kind,
            "sample": desc + ("; GB/s = algorithmic bytes / s" if fixed else
                              f"; x {its} iterations = " +
                              (f"the reference's own count for this family (recorded solve "
                               f"at n={counts[1]})" if counts else "the GPU solve's count"))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


def cpu_scaled(w, seconds):
    """Seconds per MWU iteration of the reference's CPU path (baseline/_ref; the oracle
    port when the reference is not installed) at the workload's FULL size, measured on a
    row sample of the same distribution and scaled linearly in the number of rows (each
    iteration is a fixed number of passes over them).  Returns (s/iter, text, kind)."""
    ws, factor = _sample_rows(w)
    inst = make_instance(ws)
    rows = ws["n"] if w["kind"] == "ses" else ws["n1"] + ws["n2"]
    use_ref = _import_reference() is not None
    if use_ref:
        try:
            ref_sample(ws, inst, 1)              # numba JIT of the reference
        except Exception as exc:  # noqa: BLE001
            print(f"bench: the reference failed on this host ({exc}); timing the oracle port",
                  file=sys.stderr)
            use_ref = False
    if use_ref:
        spi0, _, _ = ref_sample(ws, inst, 1)
        k = max(1, int(seconds / max(spi0, 1e-9)))
        spi, its, _ = ref_sample(ws, inst, k)
        return spi * factor, (
            f"{its} MWU iterations (one refine_run of the unmodified reference, "
            f"baseline/_ref) on a {rows}-row sample of the same distribution, {spi:.4f} "
            f"s/iter scaled x{factor:g} to the full row count"), "reference"
    s = cpu_sample(ws, inst, max_seconds=seconds)
    return s["s_per_iter"] * factor, (
        f"{s['iters']} MWU iterations (one refine_run) of the oracle port on a {rows}-row "
        f"sample of the same distribution, {s['s_per_iter']:.4f} s/iter scaled x{factor:g} to "
        f"the full row count"), "port"


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: launch N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and return its exit code."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if args.impl != "reference" and have < args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ses_c4", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, w, rank)
    elif w.get("generated"):
        gen_arm(args, w, rank, world)
    else:
        our_arm(args, w, rank, world)


if __name__ == "__main__":
    main()
