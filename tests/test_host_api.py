"""Host-side API mirror of the reference (config, result plumbing, instances,
argument validation) — everything that does not need a GPU."""
import math

import numpy as np
import pytest

from paper_2405_09157_b200 import RunConfig, instances, meta, ses, svm


def test_run_config_validation():
    RunConfig()
    for kw in ({"eps": 0.0}, {"eps": 1.0}, {"delta": 0.0}, {"patience": 0}, {"threads": 0}):
        with pytest.raises(ValueError):
            RunConfig(**kw)


def test_iteration_bound_and_early_stop():
    # same operation order as the reference (R/meta.py:212)
    assert meta.iteration_bound(math.sqrt(2), 3.0, 10, 0.1, 1.0) == math.ceil(
        4.0 * math.sqrt(2) ** 2 * 3.0 ** 2 * math.log(10) / (0.1 ** 2 * 1.0 ** 2))
    assert meta.early_stop_check([1.0] * 12, 1e-4, 10)
    assert not meta.early_stop_check([1.0, 2.0, 1.0, 2.0], 1e-4, 2)
    assert meta.early_stop_check([0.0, 0.0, 1.0, 1.0, 1.0], 1e-4, 2)   # zero prev skipped
    with pytest.raises(ValueError):
        meta.early_stop_check([1.0], 0.0, 1)


def test_instance_text_round_trip(tmp_path):
    inst = instances.gen_ses(7, 3, 1, "uniform-ball")
    text = instances.serialize_ses(inst, comments=["hello"])
    back = instances.parse(text)
    assert np.array_equal(back.centers, inst.centers) and np.array_equal(back.radii, inst.radii)
    s, _ = instances.gen_svm(4, 5, 2, 3)
    back = instances.parse(instances.serialize_svm(s))
    assert np.array_equal(back.P, s.P) and np.array_equal(back.Q, s.Q)
    p = str(tmp_path / "x.npz")
    instances.save(p, s)
    b2 = instances.load(p)
    assert np.array_equal(b2.P, s.P)


def test_binary_instance_dir_round_trip(tmp_path):
    """.npyd directories: exact round trip, memory-mapped on load."""
    inst = instances.gen_ses(50, 4, 2, "gaussian")
    inst = ses.SesInstance(centers=inst.centers, radii=np.linspace(0.0, 0.1, 50))
    p = str(tmp_path / "a.npyd")
    instances.save(p, inst)
    back = instances.load(p)
    assert not back.centers.flags.owndata     # a view of the file mapping, no copy
    assert np.array_equal(back.centers, inst.centers) and np.array_equal(back.radii, inst.radii)
    s, _ = instances.gen_svm(6, 9, 3, 1)
    q = str(tmp_path / "b.npyd")
    instances.save(q, s)
    b2 = instances.load(q, mmap=False)
    assert np.array_equal(b2.P, s.P) and np.array_equal(b2.Q, s.Q)


@pytest.mark.parametrize("text", ["", "ses 2", "ses 2 1\n1 2\n", "foo 1 2\n", "svm 1 1 1\n1\n",
                                  "ses 2 1\n1 0\nnan 0\n"])
def test_instance_parse_errors(text):
    with pytest.raises(instances.InstanceFormatError):
        instances.parse(text)


def test_instance_validation():
    with pytest.raises(ValueError):
        ses.SesInstance(np.zeros((1, 2)), np.zeros(1))
    with pytest.raises(ValueError):
        ses.SesInstance(np.zeros((3, 2)), -np.ones(3))
    with pytest.raises(ValueError):
        svm.SvmInstance(np.zeros((2, 2)), np.zeros((2, 3)))
    with pytest.raises(ValueError):
        instances.gen_ses(1, 2, 0)
    with pytest.raises(ValueError):
        instances.gen_svm(1, 1, 1, 0, gap=0.0)


def test_degenerate_ses_needs_no_device():
    # all points identical: D == 0 short-circuits (R/ses.py:150-158)
    inst = ses.SesInstance(np.ones((4, 3)), np.zeros(4))
    rep, sol = ses.solve_ses(inst, 0.1)
    assert sol.radius == 0.0 and rep.termination is meta.Termination.RANGE_CONVERGED


def test_eps_validation():
    inst = ses.SesInstance(np.eye(3), np.zeros(3))
    with pytest.raises(ValueError):
        ses.solve_ses(inst, 1.5)
    with pytest.raises(ValueError):
        meta.adaptive_search(lambda a: None, 2.0, 1.0, 0.1)


def test_foreign_progress_callback_rejected(emu_engine):
    inst = instances.gen_ses(10, 2, 0)
    dev = ses.ses_device(inst, engine=emu_engine)
    D, _, _ = ses.ses_range(inst)
    spec = meta.OracleSpec(dev.cone, 3 * D / math.sqrt(2), 3, dev, math.sqrt(2),
                           meta.Orientation.MAX)
    with pytest.raises(TypeError):
        meta.solve_ftp(spec, 1.0, 0.1, progress=lambda y: 0.0)
    r = meta.solve_ftp(spec, 0.9 * D, 0.5, progress=None, cap=64)
    assert r.best_progress is None       # no progress callback: no offers
    dev.close()


def test_width_violation_raises(emu_engine):
    """A wrong (too small) width makes the observe check fire (R/mwu.py:62-64)."""
    inst = instances.gen_ses(20, 3, 0)
    D, _, _ = ses.ses_range(inst)
    h = emu_engine.create(0, inst.centers, None, inst.radii, D=D, rho=0.1 * D, R=math.sqrt(2),
                          rank=2 * 19)
    dev = meta.DeviceProblem(h, ses.ses_cone(20, 3), 0)
    spec = meta.OracleSpec(dev.cone, 0.1 * D, 4, dev, math.sqrt(2), meta.Orientation.MAX)
    with pytest.raises(meta.WidthViolationError) as ei:
        meta.solve_ftp(spec, 0.9 * D, 0.1, progress=dev.progress, cap=64)
    assert ei.value.iteration == 1 and ei.value.norm > 0.1 * D
    dev.close()
