"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports the read-only reference from
/root/reference/pkg/src, which does not exist on the GPU box).  The JSON files
it writes under tests/golden/ are committed and are what the tests read.

    python tests/golden/make_golden.py quick      # KATs, generators, traces, small solves
    python tests/golden/make_golden.py calls      # per-call solve_ftp/refine_run records
    python tests/golden/make_golden.py long       # C1 and n=2000 solves, threads 1/2/4/8
    python tests/golden/make_golden.py baselines  # meb_baseline / gilbert_baseline records
    python tests/golden/make_golden.py headline KIND N THREADS
        # one headline-regime solve (eps=1e-3, d=100: SES uniform-ball / SVM gap 1)
        # with its per-call records -> tests/golden/headline/KIND_nN_tTHREADS.json
    python tests/golden/make_golden.py family KIND EPS THREADS ARGS...
        # the same for another instance family (ses: n d seed dist; svm: n1 n2 d seed gap)

Instances are NOT stored: tests regenerate them from (n, d, seed, dist) with
paper_2405_09157_b200.instances, whose bit-exactness against the reference
generator is itself pinned here by SHA-256 digests (``generators.json``).
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF_SRC)

import symcone  # noqa: E402  (the reference)
from symcone import cones, instances, meta, mwu, ses, svm  # noqa: E402
from symcone.config import RunConfig  # noqa: E402


def _f(x):
    if x is None:
        return None
    x = float(x)
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return x


def _v(a):
    return None if a is None else [float(v) for v in np.asarray(a).ravel()]


def _digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, indent=1)
    print("wrote", path, file=sys.stderr)


# ---------------------------------------------------------------- generators
GEN_SES = [(10, 3, 0, "gaussian"), (64, 3, 3, "gaussian"), (300, 4, 5, "gaussian"),
           (10_000, 10, 0, "gaussian"), (2000, 10, 0, "gaussian"),
           (1000, 100, 0, "uniform-ball"), (33, 5, 7, "uniform-ball"),
           (32, 2, 0, "sphere-surface"), (256, 3, 0, "sphere-surface"),
           (2048, 3, 0, "sphere-surface"), (31, 4, 2, "sphere-surface")]
GEN_SVM = [(1, 1, 2, 0, 1.0), (50, 50, 4, 1, 1.0), (150, 150, 5, 2, 1.0),
           (1000, 1000, 10, 0, 1.0), (37, 21, 6, 4, 0.5), (500, 500, 100, 0, 1.0)]


def gen_generators():
    out = {"ses": [], "svm": []}
    for n, d, seed, dist in GEN_SES:
        inst = instances.gen_ses(n, d, seed, dist)
        out["ses"].append({"n": n, "d": d, "seed": seed, "dist": dist,
                           "centers": _digest(inst.centers),
                           "radii": _digest(inst.radii)})
    for n1, n2, d, seed, gap in GEN_SVM:
        inst, direction = instances.gen_svm(n1, n2, d, seed, gap)
        out["svm"].append({"n1": n1, "n2": n2, "d": d, "seed": seed, "gap": gap,
                           "P": _digest(inst.P), "Q": _digest(inst.Q),
                           "direction": _digest(direction)})
    dump("generators.json", out)


# ---------------------------------------------------------------- KATs (SPEC)
def gen_kats():
    k = {}
    # Scmwu Orthant(2), eta=1, loss (1,-1) -> p
    c2 = cones.cone(cones.Orthant(2))
    L = mwu.Scmwu(c2, 1.0)
    L.observe(cones.Element(c2, np.array([1.0, -1.0])))
    k["scmwu_orthant2_eta1"] = _v(L.current().coords)
    L = mwu.Scmwu(c2, 0.5)
    for _ in range(200):
        L.observe(cones.Element(c2, np.array([1.0, 0.0])))
    k["scmwu_orthant2_200steps"] = _v(L.current().coords)
    k["init_soc3"] = _v(mwu.Scmwu(cones.cone(cones.SecondOrder(3)), 0.3).current().coords)
    k["init_orth2_soc1"] = _v(mwu.Scmwu(cones.cone(cones.Orthant(2), cones.SecondOrder(1)),
                                        0.3).current().coords)
    # normalized_exp on a mixed cone, including a large-scale argument
    cm = cones.cone(cones.Orthant(2), cones.SecondOrder(3), cones.SecondOrder(3),
                    cones.SecondOrder(2))
    rng = np.random.default_rng(11)
    x = rng.standard_normal(cm.ambient_dim)
    k["normexp_mixed_x"] = _v(x)
    k["normexp_mixed"] = _v(cones.normalized_exp(cones.Element(cm, x)).coords)
    k["normexp_mixed_x1000"] = _v(cones.normalized_exp(cones.Element(cm, 1000 * x)).coords)
    k["inf_norm_mixed"] = _f(cones.inf_norm(cones.Element(cm, x)))
    # ses_oracle n=2, p=e/2, alpha=1.5 (SPEC :335-336)
    inst = ses.SesInstance(centers=np.array([[0.0, 0.0], [1.0, 0.0]]), radii=np.zeros(2))
    cs = ses.ses_cone(2, 2)
    e = cones.identity(cs)
    p = cones.Element(cs, e.coords / cones.trace(e))
    o = ses.ses_oracle(inst, p, 1.5)
    k["ses_oracle_n2"] = {"p": _v(p.coords), "value": _f(o.oracle_value), "y": _v(o.y),
                          "res_inf": _f(cones.inf_norm(o.residual))}
    # svm_oracle P={(1,0)}, Q={(-1,0)}, p=(1/2,1/2), alpha=1 (SPEC :414)
    sinst = svm.SvmInstance(P=np.array([[1.0, 0.0]]), Q=np.array([[-1.0, 0.0]]))
    o = svm.svm_oracle(sinst, cones.Element(svm.svm_cone(2), np.array([0.5, 0.5])), 1.0)
    k["svm_oracle_2pt"] = {"value": _f(o.oracle_value), "y": _v(o.y),
                           "res": _v(o.residual.coords), "cand": _f(o.candidate_value)}
    # end-to-end KATs from SPEC
    th = np.linspace(0, 2 * np.pi, 32, endpoint=False)
    circ = ses.SesInstance(centers=np.stack([np.cos(th), np.sin(th)], 1), radii=np.zeros(32))
    r, s = ses.solve_ses(circ, 0.05)
    k["ses_circle32"] = _solve_ses_rec(r, s)
    col = ses.SesInstance(centers=np.array([[0.0], [1.0], [2.0]]), radii=np.zeros(3))
    r, s = ses.solve_ses(col, 0.05)
    k["ses_collinear3"] = _solve_ses_rec(r, s)
    r, s = svm.solve_svm(sinst, 0.01)
    k["svm_two_point"] = _solve_svm_rec(r, s)
    dump("kats.json", k)


def _solve_ses_rec(r, s):
    return {"radius": _f(s.radius), "center": _v(s.center), "slack": _f(s.enclosure_slack),
            "primal": _f(r.primal_value), "dual": _f(r.dual_value),
            "iterations": r.total_iterations, "steps": r.search_steps,
            "termination": r.termination.value,
            "search": [[_f(st.alpha), _f(st.eps), st.iteration_bound, st.iterations,
                        st.separated, st.reason] for st in r.steps]}


def _solve_svm_rec(r, s):
    return {"margin": _f(s.margin), "w": _v(s.w), "pd_distance": _f(s.pd_distance),
            "mu": _v(s.pd_point[0]) if len(s.pd_point[0]) <= 64 else _digest(s.pd_point[0]),
            "gam": _v(s.pd_point[1]) if len(s.pd_point[1]) <= 64 else _digest(s.pd_point[1]),
            "mu_sum": _f(np.sum(s.pd_point[0])), "mu_max": _f(np.max(s.pd_point[0])),
            "excentricity": _f(s.excentricity),
            "primal": _f(r.primal_value), "dual": _f(r.dual_value),
            "iterations": r.total_iterations, "steps": r.search_steps,
            "termination": r.termination.value,
            "search": [[_f(st.alpha), _f(st.eps), st.iteration_bound, st.iterations,
                        st.separated, st.reason] for st in r.steps]}


# ---------------------------------------------------------------- per-iteration traces
def ses_trace(inst, alpha, eta, K):
    """Reference learner + oracle at a fixed level: per-iteration records."""
    D, _, _ = ses.ses_range(inst)
    rho = 3.0 * D / cones.SQRT2
    cone_k = ses.ses_cone(inst.n, inst.d)
    L = mwu.Scmwu(cone_k, eta)
    y_sum = np.zeros(inst.d + 1)
    rec = []
    for t in range(1, K + 1):
        p = L.current()
        P = p.coords.reshape(inst.n - 1, inst.d + 1)
        o = ses.ses_oracle(inst, p, alpha)
        if isinstance(o, meta.Separated):
            rec.append({"t": t, "separated": True, "value": _f(o.oracle_value)})
            break
        y_sum += o.y
        width = cones.inf_norm(o.residual) / rho
        f = ses.ses_progress(inst, (y_sum / t)[:inst.d])
        rec.append({"t": t, "value": _f(o.oracle_value), "u": _v(o.y[:-1]),
                    "s": _v(P[:, :inst.d].sum(axis=0)),
                    "width": _f(width), "f": _f(f), "p_sig_sum": _f(P[:, inst.d].sum())})
        L.observe(o.residual, prescale=1.0 / rho)
    return {"alpha": alpha, "eta": eta, "rho": rho, "records": rec}


def svm_trace(inst, alpha, eta, K):
    D = inst.max_norm
    rho = 2.0 * D
    cone_k = svm.svm_cone(inst.n1 + inst.n2)
    L = mwu.Scmwu(cone_k, eta)
    y_sum = np.zeros(inst.d + 2)
    rec = []
    for t in range(1, K + 1):
        p = L.current()
        o = svm.svm_oracle(inst, p, alpha)
        if isinstance(o, meta.Separated):
            rec.append({"t": t, "separated": True, "value": _f(o.oracle_value)})
            break
        y_sum += o.y
        width = cones.inf_norm(o.residual) / rho
        f = svm.svm_progress(inst, (y_sum / t)[:inst.d])
        mu, gam = svm.extract_pd(p, inst.n1)
        z = inst.P.T @ mu - inst.Q.T @ gam
        rec.append({"t": t, "value": _f(o.oracle_value), "w": _v(o.y[:inst.d]),
                    "s1": _f(o.y[inst.d]), "s2": _f(o.y[inst.d + 1]),
                    "cand": _f(o.candidate_value), "width": _f(width), "f": _f(f),
                    "dist": _f(np.linalg.norm(z)), "tr_mu": _f(p.coords[:inst.n1].sum())})
        L.observe(o.residual, prescale=1.0 / rho)
    return {"alpha": alpha, "eta": eta, "rho": rho, "records": rec}


def gen_traces():
    out = {}
    inst = instances.gen_ses(64, 3, 3, "gaussian")
    D, _, _ = ses.ses_range(inst)
    r = 2 * (inst.n - 1)
    for name, frac, T in [("ses64_hi", 0.9, 2048), ("ses64_mid", 0.7, 512)]:
        tr = ses_trace(inst, frac * D, math.sqrt(math.log(r) / T), 300)
        tr.update({"inst": ["ses", 64, 3, 3, "gaussian"], "T": T})
        out[name] = tr
    inst = instances.gen_ses(33, 5, 7, "uniform-ball")
    D, _, _ = ses.ses_range(inst)
    tr = ses_trace(inst, 0.55 * D, math.sqrt(math.log(2 * 32) / 64), 120)
    tr.update({"inst": ["ses", 33, 5, 7, "uniform-ball"], "T": 64})
    out["ses33_lo"] = tr
    sinst, _ = instances.gen_svm(50, 50, 4, 1, 1.0)
    for name, alpha, T in [("svm50_a", 1.0, 2048), ("svm50_b", 1.5, 512), ("svm50_c", 0.3, 64)]:
        tr = svm_trace(sinst, alpha, math.sqrt(math.log(100) / T), 400)
        tr.update({"inst": ["svm", 50, 50, 4, 1, 1.0], "T": T})
        out[name] = tr
    dump("traces.json", out)


# ---------------------------------------------------------------- per-call records
def _result_rec(res):
    if isinstance(res, meta.PrimalCertificate):
        return {"type": "primal", "iterations": res.iterations,
                "oracle_value": _f(res.oracle_value), "alpha": _f(res.alpha),
                "best_progress": _f(res.best_progress), "best_y": _v(res.best_y),
                "best_counter": _f(res.best_counter)}
    return {"type": "dual", "iterations": res.iterations, "reason": res.reason,
            "eps_eff": _f(res.eps_eff), "value": _f(res.value), "y_tilde": _v(res.y_tilde),
            "best_progress": _f(res.best_progress), "best_y": _v(res.best_y),
            "best_counter": _f(res.best_counter)}


def record_calls(fn):
    """Run fn() with meta.solve_ftp / meta.refine_run wrapped by recorders."""
    calls = []
    orig_ftp, orig_ref = meta.solve_ftp, meta.refine_run

    def ftp(oracle, alpha, eps, stopping=None, progress=None, cap=None):
        res = orig_ftp(oracle, alpha, eps, stopping, progress, cap)
        calls.append({"fn": "ftp", "alpha": _f(alpha), "eps": _f(eps), "cap": cap,
                      "delta": stopping.delta, "patience": stopping.patience,
                      "enabled": stopping.enabled, "result": _result_rec(res)})
        return res

    def ref(oracle, alpha, horizon, stopping, progress, gain_rel=None, bounds=None,
            target=None):
        res = orig_ref(oracle, alpha, horizon, stopping, progress, gain_rel, bounds, target)
        calls.append({"fn": "refine", "alpha": _f(alpha), "horizon": horizon,
                      "gain_rel": _f(gain_rel), "bounds": [_f(b) for b in bounds],
                      "target": _f(target), "delta": stopping.delta,
                      "patience": stopping.patience, "enabled": stopping.enabled,
                      "result": _result_rec(res)})
        return res

    meta.solve_ftp, meta.refine_run = ftp, ref
    try:
        out = fn()
    finally:
        meta.solve_ftp, meta.refine_run = orig_ftp, orig_ref
    return out, calls


CALL_CASES = [
    ("ses", (300, 4, 5, "gaussian"), 1e-2),
    ("ses", (64, 3, 3, "gaussian"), 1e-2),
    ("svm", (150, 150, 5, 2, 1.0), 1e-2),
    ("svm", (50, 50, 4, 1, 1.0), 1e-2),
    ("svm", (37, 21, 6, 4, 0.5), 1e-2),
]


def gen_calls():
    out = []
    for kind, args, eps in CALL_CASES:
        t0 = time.time()
        if kind == "ses":
            inst = instances.gen_ses(*args)
            (r, s), calls = record_calls(lambda: ses.solve_ses(inst, eps))
            rec = _solve_ses_rec(r, s)
            D, _, _ = ses.ses_range(inst)
            extra = {"D": _f(D)}
        else:
            inst, _ = instances.gen_svm(*args)
            (r, s), calls = record_calls(lambda: svm.solve_svm(inst, eps))
            rec = _solve_svm_rec(r, s)
            extra = {"D": _f(inst.max_norm)}
        out.append({"kind": kind, "inst": list(args), "eps": eps, "solve": rec,
                    "calls": calls, "wall_s": time.time() - t0, **extra})
        print(kind, args, "iters", rec["iterations"], "calls", len(calls),
              f"{time.time() - t0:.1f}s", file=sys.stderr)
    dump("calls.json", out)


# ---------------------------------------------------------------- long end-to-end solves
LONG_CASES = [
    ("ses", (2000, 10, 0, "gaussian"), 1e-2, (1, 2, 4, 8)),
    ("svm", (1000, 1000, 10, 0, 1.0), 1e-2, (1, 2)),
    ("ses", (10_000, 10, 0, "gaussian"), 1e-2, (1, 2, 4, 8)),
    ("ses", (32, 2, 0, "sphere-surface"), 1e-2, (1,)),
    ("ses", (256, 3, 0, "sphere-surface"), 1e-2, (1,)),
    ("ses", (2048, 3, 0, "sphere-surface"), 1e-2, (1,)),
]


def gen_long(which=None):
    path = os.path.join(HERE, "long.json")
    out = json.load(open(path)) if os.path.exists(path) else []
    done = {(o["kind"], tuple(o["inst"]), o["eps"], o["threads"]) for o in out}
    for kind, args, eps, threads in LONG_CASES:
        for th in threads:
            key = (kind, tuple(args), eps, th)
            if key in done:
                continue
            t0 = time.time()
            cfg = RunConfig(eps=eps, threads=th)
            if kind == "ses":
                inst = instances.gen_ses(*args)
                r, s = ses.solve_ses(inst, eps, cfg)
                rec = _solve_ses_rec(r, s)
            else:
                inst, _ = instances.gen_svm(*args)
                r, s = svm.solve_svm(inst, eps, cfg)
                rec = _solve_svm_rec(r, s)
            wall = time.time() - t0
            out.append({"kind": kind, "inst": list(args), "eps": eps, "threads": th,
                        "wall_s": wall, "solve": rec})
            print(kind, args, th, rec["iterations"], f"{wall:.1f}s", file=sys.stderr)
            dump("long.json", out)


# ---------------------------------------------------------------- verification baselines
# (kind, instance args, radii seed or None, solver args); the radii, when present, are
# drawn as rng(seed).uniform(0, 0.1, n)
BASE_CASES = [
    ("meb", (300, 4, 1, "gaussian"), None, {"eps_base": 0.05}),
    ("meb", (200, 7, 2, "uniform-ball"), 11, {"eps_base": 0.1}),
    ("meb", (64, 3, 0, "sphere-surface"), None, {"eps_base": 0.1}),
    ("gilbert", (150, 120, 5, 3, 0.5), None, {"gap_tol": 1e-6, "max_iters": 100_000}),
    ("gilbert", (80, 90, 3, 4, 0.1), None, {"gap_tol": 1e-8, "max_iters": 2000}),
    ("gilbert", (40, 30, 12, 5, 2.0), None, {"gap_tol": 1e-10, "max_iters": 50_000}),
]


def gen_baselines():
    from symcone import baselines
    out = []
    for kind, args, rseed, kw in BASE_CASES:
        if kind == "meb":
            inst = instances.gen_ses(*args)
            rad = (np.random.default_rng(rseed).uniform(0.0, 0.1, args[0])
                   if rseed is not None else None)
            r = baselines.meb_baseline(inst.centers, rad, **kw)
            out.append({"kind": kind, "inst": list(args), "radii_seed": rseed, "kw": kw,
                        "value": _f(r.value), "center": _v(r.certificate),
                        "iterations": int(r.iterations)})
        else:
            inst, _ = instances.gen_svm(*args)
            r = baselines.gilbert_baseline(inst.P, inst.Q, **kw)
            mu, gam = r.certificate
            out.append({"kind": kind, "inst": list(args), "kw": kw, "value": _f(r.value),
                        "gap": _f(r.gap), "iterations": int(r.iterations),
                        "mu": _v(mu), "gam": _v(gam)})
        print(kind, args, out[-1]["value"], out[-1]["iterations"], file=sys.stderr)
    dump("baselines.json", out)


# ---------------------------------------------------------------- headline regime
# BASELINE configs[1..4] run at eps=1e-3, d=100 (SES uniform-ball, SVM gap 1); these
# record the reference's own solves of the same families at sizes it finishes in
# minutes to hours, so the device's refine/stop behaviour can be compared with it.
def gen_headline(kind: str, n: int, threads: int, args=None, eps: float = 1e-3,
                 name: str | None = None):
    t0 = time.time()
    cfg = RunConfig(eps=eps, threads=threads)
    if kind == "ses":
        args = tuple(args) if args is not None else (n, 100, 0, "uniform-ball")
        inst = instances.gen_ses(*args)
        (r, s), calls = record_calls(lambda: ses.solve_ses(inst, eps, cfg))
        rec = _solve_ses_rec(r, s)
        D, _, _ = ses.ses_range(inst)
    else:
        args = tuple(args) if args is not None else (n // 2, n - n // 2, 100, 0, 1.0)
        inst, _ = instances.gen_svm(*args)
        (r, s), calls = record_calls(lambda: svm.solve_svm(inst, eps, cfg))
        rec = _solve_svm_rec(r, s)
        D = inst.max_norm
    wall = time.time() - t0
    for c in calls:  # the per-call y vectors are not needed here; keep the files small
        c["result"].pop("y_tilde", None)
        c["result"].pop("best_y", None)
    out = {"kind": kind, "inst": list(args), "eps": eps, "threads": threads,
           "wall_s": wall, "D": _f(D), "s_per_iter": wall / max(1, rec["iterations"]),
           "solve": rec, "calls": calls}
    os.makedirs(os.path.join(HERE, "headline"), exist_ok=True)
    dump(os.path.join("headline", name or f"{kind}_n{n}_t{threads}.json"), out)
    print(kind, args, threads, rec["iterations"], rec["termination"], f"{wall:.1f}s",
          file=sys.stderr)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "quick"
    if what == "quick":
        gen_generators()
        gen_kats()
        gen_traces()
    elif what == "baselines":
        gen_baselines()
    elif what == "calls":
        gen_calls()
    elif what == "long":
        gen_long()
    elif what == "headline":
        gen_headline(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    elif what == "family":
        # family KIND EPS THREADS ARGS...  (ses: n d seed dist; svm: n1 n2 d seed gap)
        kind, eps, th = sys.argv[2], float(sys.argv[3]), int(sys.argv[4])
        raw = sys.argv[5:]
        if kind == "ses":
            fargs = (int(raw[0]), int(raw[1]), int(raw[2]), raw[3])
            n = fargs[0]
        else:
            fargs = (int(raw[0]), int(raw[1]), int(raw[2]), int(raw[3]), float(raw[4]))
            n = fargs[0] + fargs[1]
        tag = "_".join(str(a) for a in fargs)
        gen_headline(kind, n, th, fargs, eps, f"{kind}_{tag}_e{eps:g}_t{th}.json")
    else:
        raise SystemExit(f"unknown group {what}")
