"""Benchmark: time-to-eps of the SCMWU solvers on the B200 engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload ses_c2|svm_c3|ses_c1|ses_c4]
    python bench.py --impl reference ...      # CPU reference arm (the oracle port)

A *step* is one full solve (adaptive search to the reference's stopping rule)
of the workload BASELINE.json's metric is quoted on: by default configs[1],
SES n=10^6, d=100 uniform-ball points, eps=1e-3 on one B200.

value    time-to-eps with the instance already resident in HBM, device-timed
         with CUDA events on the engine's stream (host gaps between kernel
         launches included), max over ranks.
e2e      the same solve through the public API (solve_ses / solve_svm) from
         host numpy arrays: H2D of the instance and D2H of the result inside.
roofline HBM roofline of the persistent kernel: algorithmic bytes
         8 n (d+1) (SES) or 8 n d (SVM) per streaming pass x passes / kernel
         event time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the oracle port (oracle/, numpy + C restatement of the reference)
         timed on this host for a bounded sample of iterations of the same
         workload; time-to-eps extrapolated as s/iter x GPU iterations.
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
                   desc="SES n=10^7 d=100 uniform-in-ball, eps=1e-3 (configs[3])"),
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
# GPU iteration counts of full solves measured by this bench (profiles/); used only by the
# reference arm to extrapolate the CPU port's s/iter to a time-to-eps.
ITERS_EST = {"ses_c2": 15_515, "svm_c3": 320_146, "ses_c1": 103_672, "ses_c4": 360_000}


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


def reference_arm(args, w, rank):
    if rank != 0:
        return
    if w.get("generated"):
        return reference_arm_scaled(args, w)
    inst = make_instance(w)
    t0 = time.perf_counter()
    samples = []
    for _ in range(args.warmup):
        cpu_sample(w, inst, max_seconds=3.0, max_iters=1)
    for _ in range(args.steps):
        samples.append(cpu_sample(w, inst, max_seconds=args.cpu_seconds))
    spi = statistics.median(s["s_per_iter"] for s in samples)
    iters = ITERS_EST[args.workload]
    value = spi * iters
    line = {
        "impl": "reference", "metric": "time-to-eps (s)", "value": value, "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": value * 1000.0, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"],
                   "extrapolated_from_iters": iters},
        "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": "port",
                         "sample": f"{samples[-1]['iters']} MWU iterations (one refine_run) of "
                                   f"the workload per step; {spi:.4f} s/iter x {iters} "
                                   f"iterations (the GPU solve's count; extrapolated)"},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


def reference_arm_scaled(args, w):
    """Reference arm of the device-generated workloads: the host cannot hold these
    instances (C5 is 82 GB), so each step times the oracle port on a row sample and scales
    per-iteration time linearly to the full row count."""
    t0 = time.perf_counter()
    ws = _sample_cfg(w)
    warm = make_instance(ws)
    for _ in range(args.warmup):
        cpu_sample(ws, warm, max_seconds=1.0, max_iters=1)
    spis = []
    for _ in range(args.steps):
        spi, desc = cpu_scaled(w, args.cpu_seconds)
        spis.append(spi)
    spi = statistics.median(spis)
    bpp = alg_bytes_per_pass(w)
    if w.get("horizon") is not None:
        value, metric, unit, hib = bpp / spi / 1e9, "per-iteration HBM GB/s", "GB/s", True
    else:
        iters = ITERS_EST.get(args.workload.replace("_gen", ""), 0)
        value, metric, unit, hib = spi * iters, "time-to-eps (s)", "s", False
        desc += f"; x {iters} iterations (the GPU solve's count; extrapolated)"
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": spi * 1000.0, "higher_is_better": hib, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"]},
        "cpu_baseline": {"value": value, "unit": unit, "cores": 1, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


def _sample_cfg(w):
    ws = dict(w)
    if w["kind"] == "ses":
        ws["n"] = min(w["n"], 2_000)
    else:
        ws["n1"], ws["n2"] = min(w["n1"], 1_000), min(w["n2"], 1_000)
    return ws


# ------------------------------------------------------------------ our arm
def solve(w, inst, device=None):
    from paper_2405_09157_b200 import ses, svm
    if w["kind"] == "ses":
        return ses.solve_ses(inst, w["eps"], device=device)
    return svm.solve_svm(inst, w["eps"], device=device)


def our_arm(args, w, rank, world):
    import torch
    from paper_2405_09157_b200 import ses, svm
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        tdist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    inst = make_instance(w, pinned=torch.cuda.is_available())
    t_up = time.perf_counter()
    comm = None
    if dist:
        from paper_2405_09157_b200 import shard
        comm = shard.Comm()

    def make_device():
        if comm is not None:   # row-sharded: this rank's rows, in-kernel NVLink exchange
            return (shard.ses_device_sharded(inst, comm, device=local) if w["kind"] == "ses"
                    else shard.svm_device_sharded(inst, comm, device=local))
        return (ses.ses_device(inst, device=local) if w["kind"] == "ses"
                else svm.svm_device(inst, device=local))

    dev = make_device()
    upload_s = time.perf_counter() - t_up
    info = dev.handle.info()
    for _ in range(args.warmup):
        solve(w, inst, dev)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            tdist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    l0 = dev.handle.launches()
    reports = []
    times = []
    for _ in range(args.steps):
        dev.handle.mark(0)
        rep, sol = solve(w, inst, dev)
        dev.handle.mark(1)
        times.append(dev.handle.elapsed_ms() / 1000.0)
        reports.append((rep, sol))
    barrier()
    launches = dev.handle.launches() - l0
    clk = clocks.stop()
    t_step = sum(times) / len(times)   # the K timed steps / K (then max over ranks)
    if dist:
        t = torch.tensor([t_step], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        t_step = float(t.item())
    kernel_s = sum(r.kernel_ms for r, _ in reports) / 1000.0
    passes = sum(r.passes for r, _ in reports)
    width_passes = sum(r.width_passes for r, _ in reports)
    dev.close()

    # e2e: public API from host arrays (upload + download inside the timed region)
    e2e_times = []
    for _ in range(max(1, args.steps)):
        barrier()
        t0 = time.perf_counter()
        if comm is None:
            rep_e, sol_e = solve(w, inst, None)
        else:                  # upload of this rank's shard + solve + download
            dev_e = make_device()
            rep_e, sol_e = solve(w, inst, dev_e)
            dev_e.close()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    if dist:
        t = torch.tensor([sum(e2e_times) / len(e2e_times)], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_times = [float(t.item())]
    e2e = sum(e2e_times) / len(e2e_times)
    print(f"bench: e2e per step {['%.3f' % t for t in e2e_times]} s", file=sys.stderr)
    if w["kind"] == "ses":
        h2d = inst.centers.nbytes + inst.radii.nbytes
        d2h = (w["d"] + 1) * 8 * 2 * rep_e.search_steps + 8 * 4
    else:
        h2d = inst.P.nbytes + inst.Q.nbytes
        d2h = (w["d"] + 2) * 8 * 2 * rep_e.search_steps + inst.n1 * 8 + inst.n2 * 8

    peak, peak_kind = measured_peak()
    achieved = passes * alg_bytes_per_pass(w) / kernel_s / 1e9 if kernel_s > 0 else 0.0
    rep0, sol0 = reports[-1]
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
        "data": "synthetic",
        "config": {"workload": w["desc"], "eps": w["eps"], "seed": w["seed"],
                   "parallelism": (f"row-sharded x{world} (in-kernel NVLink exchange)"
                                   if world > 1 else "1 GPU"),
                   "iterations": rep0.total_iterations, "search_steps": rep0.search_steps,
                   "termination": rep0.termination.value,
                   "l2": "inputs larger than L2 (X = %.0f MB)" % (alg_bytes_per_pass(w) / 1e6)
                   if alg_bytes_per_pass(w) > 126e6 else "inputs fit in L2",
                   "kernel": info, "upload_s": upload_s},
        "result": ({"radius": sol0.radius, "lower": rep0.primal_value,
                    "enclosure_slack": sol0.enclosure_slack} if w["kind"] == "ses" else
                   {"margin": sol0.margin, "pd_distance": sol0.pd_distance}),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "read_ceiling": READ_CEILING_GBS,
                     "frac_of_read_ceiling": achieved / READ_CEILING_GBS,
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "alg_bytes_per_pass": alg_bytes_per_pass(w),
                     "us_per_pass": kernel_s / passes * 1e6 if passes else None,
                     "kernel_s": kernel_s, "passes": passes,
                     "exact_width_passes": width_passes},
        "e2e": {"value": e2e, "unit": "s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and not args.no_cpu_baseline:
        s = cpu_sample(w, inst, max_seconds=args.cpu_seconds)
        its = rep0.total_iterations
        line["cpu_baseline"] = {
            "value": s["s_per_iter"] * its, "unit": "s", "cores": 1, "kind": "port",
            "sample": f"{s['iters']} MWU iterations (one refine_run) of the workload on the "
                      f"oracle port ({s['s_per_iter']:.4f} s/iter); time-to-eps "
                      f"extrapolated x {its} GPU iterations"}
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
        spi, desc = cpu_scaled(w, args.cpu_seconds)
        cv = bpp / spi / 1e9 if fixed else spi * iters
        line["cpu_baseline"] = {"value": cv, "unit": unit, "cores": 1, "kind": "port",
                                "sample": desc + (f"; x {iters} GPU iterations" if not fixed
                                                  else "; GB/s = algorithmic bytes / s")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


def cpu_scaled(w, seconds):
    """Seconds per MWU iteration of the oracle port at the workload's FULL size, measured
    on a row sample (numpy generation of the same distribution) and scaled linearly in the
    number of rows (each iteration is one pass over them)."""
    ws = dict(w)
    if w["kind"] == "ses":
        ws["n"] = min(w["n"], 100_000)
        factor = w["n"] / ws["n"]
    else:
        ws["n1"] = min(w["n1"], 50_000)
        ws["n2"] = min(w["n2"], 50_000)
        factor = (w["n1"] + w["n2"]) / (ws["n1"] + ws["n2"])
    s = cpu_sample(ws, make_instance(ws), max_seconds=seconds)
    rows = ws["n"] if w["kind"] == "ses" else ws["n1"] + ws["n2"]
    return s["s_per_iter"] * factor, (
        f"{s['iters']} MWU iterations (one refine_run) of the oracle port on a {rows}-row "
        f"sample of the same distribution, {s['s_per_iter']:.4f} s/iter scaled x{factor:g} to "
        f"the full row count")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ses_c2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        reference_arm(args, w, rank)
    elif w.get("generated"):
        gen_arm(args, w, rank, world)
    else:
        our_arm(args, w, rank, world)


if __name__ == "__main__":
    main()
