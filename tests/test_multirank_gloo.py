"""Row-sharded solves with world_size 2 on the CPU (gloo).

Each process holds half of the rows in a sharded handle of the CPU emulator;
the per-pass rank vectors are exchanged through a gloo all-gather and folded
in rank order — the same protocol the CUDA kernel runs over NVLink mailboxes.
A sharded solve must take the same decisions as the single-process solve
(SVM: identical iteration counts; values to rounding of the fold order)."""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, args, eps, out_path):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import build
    from paper_2405_09157_b200 import _native as nat
    from paper_2405_09157_b200 import instances, ses, shard, svm
    eng = nat.Engine(build.EMU_LIB)
    comm = shard.Comm()
    if kind == "svm_calls":
        # replay the reference's first recorded feasibility tests on the sharded device
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import parity as P
        from paper_2405_09157_b200 import meta
        inst, _ = instances.gen_svm(*args)
        dev = shard.svm_device_sharded(inst, comm, engine=eng)
        spec = meta.OracleSpec(dev.cone, 2.0 * inst.max_norm, inst.d + 2, dev, 2.0,
                               meta.Orientation.MIN, counter_progress=True)
        golden = json.load(open(os.path.join(ROOT, "tests", "golden", "calls.json")))
        calls = [c for c in golden if c["inst"] == list(args)][0]["calls"][:eps]
        bad = [P.compare_call(P.replay(c, spec, dev), c["result"], 1e-9, dev.progress)
               for c in calls]
        res = {"bad": bad, "n": len(calls)}
    elif kind == "ses":
        inst = instances.gen_ses(*args)
        dev = shard.ses_device_sharded(inst, comm, engine=eng)
        rep, sol = ses.solve_ses(inst, eps, device=dev)
        res = {"radius": sol.radius, "center": list(sol.center), "iters": rep.total_iterations,
               "steps": rep.search_steps, "term": rep.termination.value,
               "slack": sol.enclosure_slack, "n_local": dev.handle.prob.n_local,
               "D": dev.handle.prob.D, "D_host": ses.ses_range(inst)[0]}
    else:
        inst, _ = instances.gen_svm(*args)
        dev = shard.svm_device_sharded(inst, comm, engine=eng)
        rep, sol = svm.solve_svm(inst, eps, device=dev)
        res = {"margin": sol.margin, "pd": sol.pd_distance, "iters": rep.total_iterations,
               "steps": rep.search_steps, "term": rep.termination.value,
               "mu_sum": float(sol.pd_point[0].sum()), "n_mu": len(sol.pd_point[0]),
               "n_local": dev.handle.prob.n_local,
               "D": dev.handle.prob.D, "D_host": inst.max_norm}
    with open(f"{out_path}.{rank}", "w") as fh:
        json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, kind, args, eps, world=2):
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(world, _free_port(), kind, args, eps, out), nprocs=world,
                       join=True, start_method="spawn")
    return [json.load(open(f"{out}.{r}")) for r in range(world)]


def test_row_ranges_partition():
    from paper_2405_09157_b200 import shard
    assert shard.row_ranges(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert shard.row_ranges(5, 5) == [(i, i + 1) for i in range(5)]
    with pytest.raises(ValueError):
        shard.row_ranges(2, 3)


def test_fold_ranks_order_and_ops():
    import numpy as np
    from paper_2405_09157_b200 import shard
    ops = shard.red_ops(0, 2)          # SES: T Lin Rad sum, M F Wd Fw max, Sd sum
    rows = np.array([[1.0, 2, 3, 4, 5, 6, 7, 8, 9], [10.0, 20, 30, -4, 50, -6, 70, 80, 90]])
    got = shard.fold_ranks(rows, ops)
    assert list(got) == [11.0, 22, 33, 4, 50, 6, 70, 88, 99]


def test_svm_sharded_replays_reference_calls(tmp_path):
    """The reference's first three recorded tests (bracketing phase), replayed on a
    2-rank sharded device, match the reference's results to 1e-9."""
    res = _run(tmp_path, "svm_calls", (37, 21, 6, 4, 0.5), 3)
    for r in res:
        assert r["n"] == 3 and all(not b for b in r["bad"]), r["bad"]


def test_svm_sharded_solve_matches_single(tmp_path, emu_engine):
    from paper_2405_09157_b200 import instances, svm
    args = (30, 25, 4, 8, 1.0)
    inst, _ = instances.gen_svm(*args)
    rep, sol = svm.solve_svm(inst, 0.1, engine=emu_engine)
    res = _run(tmp_path, "svm", args, 0.1)
    for r in res:   # both ranks report the same solve
        assert r["iters"] == rep.total_iterations and r["steps"] == rep.search_steps
        assert r["term"] == rep.termination.value
        assert r["margin"] == pytest.approx(sol.margin, rel=1e-12)
        assert r["pd"] == pytest.approx(sol.pd_distance, rel=1e-12)
        assert r["n_mu"] == inst.n1 and r["mu_sum"] == pytest.approx(1.0, rel=1e-12)
    assert res[0]["n_local"] + res[1]["n_local"] == inst.n1 + inst.n2
    # the range from the shards' rows, max-reduced: bit-identical to the host expression
    assert all(r["D"] == r["D_host"] == inst.max_norm for r in res)


def test_ses_sharded_matches_single(tmp_path, emu_engine):
    from paper_2405_09157_b200 import instances, ses
    args = (40, 3, 5, "gaussian")
    inst = instances.gen_ses(*args)
    rep, sol = ses.solve_ses(inst, 0.1, engine=emu_engine)
    res = _run(tmp_path, "ses", args, 0.1)
    assert res[0] == {**res[1], "n_local": res[0]["n_local"]}   # ranks agree exactly
    r = res[0]
    assert r["term"] == rep.termination.value
    assert abs(r["slack"]) <= 1e-9 * r["radius"]
    assert r["radius"] == pytest.approx(sol.radius, rel=2e-3)   # SES: within the spread
    # the range from the shards' rows (rank 1 has no anchor row: v1, g1 from set_globals)
    assert r["D"] == r["D_host"] == ses.ses_range(inst)[0]
