"""The multi-GPU exchange on one GPU: SCMWU_VWORLD=W splits the grid of the
persistent kernel into W CTA groups, each acting as one rank with its own rows (the
np.array_split rule of shard.row_ranges), its own grid barrier and its own mailbox; the
groups run the real in-kernel exchange (flags with st.release / ld.acquire, parity
double-buffered mailboxes, rank-ordered fold) with each other.  All groups are CTAs of ONE
cooperative launch, so they are co-resident by construction (the profiling guide forbids
emulating ranks as separate launches that wait on one another).

A sharded solve must equal the single-GPU solve up to the summation order of the fold:
identical iteration counts / search steps (SVM) and values to 1e-9."""
import math

import numpy as np
import pytest

from paper_2405_09157_b200 import instances, meta, ses, svm

pytestmark = pytest.mark.gpu


def _svm_solve(inst, monkeypatch, world):
    if world > 1:
        monkeypatch.setenv("SCMWU_VWORLD", str(world))
    else:
        monkeypatch.delenv("SCMWU_VWORLD", raising=False)
    dev = svm.svm_device(inst)
    try:
        return svm.solve_svm(inst, 1e-2, device=dev)
    finally:
        dev.close()
        monkeypatch.delenv("SCMWU_VWORLD", raising=False)


@pytest.mark.parametrize("world", [2, 4])
def test_svm_solve_with_emulated_ranks(monkeypatch, world):
    inst, _ = instances.gen_svm(3000, 2500, 20, 7, 1.0)
    r1, s1 = _svm_solve(inst, monkeypatch, 1)
    rw, sw = _svm_solve(inst, monkeypatch, world)
    assert rw.total_iterations == r1.total_iterations
    assert rw.search_steps == r1.search_steps
    assert math.isclose(sw.margin, s1.margin, rel_tol=1e-9)
    assert math.isclose(sw.pd_distance, s1.pd_distance, rel_tol=1e-9)
    assert np.allclose(sw.w, s1.w, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("world", [2, 4])
def test_ses_refine_with_emulated_ranks(monkeypatch, world):
    inst = instances.gen_ses(20_000, 30, 3, "uniform-ball")
    D, _, _ = ses.ses_range(inst)
    out = []
    for w in (1, world):
        if w > 1:
            monkeypatch.setenv("SCMWU_VWORLD", str(w))
        else:
            monkeypatch.delenv("SCMWU_VWORLD", raising=False)
        dev = ses.ses_device(inst, D)
        spec = meta.OracleSpec(dev.cone, 3 * D / math.sqrt(2), inst.d + 1, dev, math.sqrt(2),
                               meta.Orientation.MAX)
        r = meta.refine_run(spec, 0.9 * D, 256, meta.EarlyStopConfig(enabled=False),
                            dev.progress)
        out.append(r)
        dev.close()
    monkeypatch.delenv("SCMWU_VWORLD", raising=False)
    a, b = out
    assert type(a) is type(b) and a.iterations == b.iterations
    assert math.isclose(a.best_progress, b.best_progress, rel_tol=1e-9)
    assert np.allclose(a.y_tilde, b.y_tilde, rtol=1e-9, atol=1e-12)
