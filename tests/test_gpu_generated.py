"""On-device instance generation (sc_create_generated).

Generated instances have no numpy counterpart (Philox, not PCG64), so parity is
anchored two ways: (1) properties of the rows themselves, read back with
sc_read_rows: the distribution's invariants, independence from the row sharding, the
device range D against numpy's; (2) a solve over the generated rows equals, bit for
bit, the solve over the same rows uploaded from the host through sc_create.
"""
import numpy as np
import pytest

from paper_2405_09157_b200 import _native as nat
from paper_2405_09157_b200.devgen import gen_ses_device, gen_svm_device
from paper_2405_09157_b200.ses import SesInstance
from paper_2405_09157_b200.svm import SvmInstance
from paper_2405_09157_b200.ses import solve_ses
from paper_2405_09157_b200.shard import row_ranges
from paper_2405_09157_b200.svm import solve_svm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dist", ["gaussian", "uniform-ball", "sphere-surface"])
def test_ses_rows_invariants_and_sharding(dist):
    eng = nat.cuda_engine()
    n, d, seed = 1001, 37, 11         # odd n (sphere: unpaired last row), odd d (padding)
    h, D, v1 = eng.create_generated(nat.SC_SES, n, d, seed, nat.GEN_DISTS[dist])
    X = h.read_rows()
    assert np.array_equal(X[0], v1)
    D_np = float(np.linalg.norm(X[1:] - X[0], axis=1).max())
    assert abs(D - D_np) <= 1e-13 * D_np
    norms = np.linalg.norm(X, axis=1)
    if dist == "gaussian":
        assert abs(X.mean()) < 0.03 and abs(X.var() - 1.0) < 0.03
    elif dist == "uniform-ball":
        assert norms.max() <= 1.0 + 1e-12
        # E|x| = d/(d+1) for the uniform ball
        assert abs(norms.mean() - d / (d + 1)) < 0.01
    else:
        assert np.allclose(norms, 1.0, atol=1e-12)
        k = n // 2
        assert np.array_equal(X[k:2 * k], -X[:k])
    # the same rows whatever the sharding
    parts, Ds = [], []
    for world in (2, 3):
        parts = []
        for r, (r0, r1) in enumerate(row_ranges(n, world)):
            hs, Ds_r, v1s = eng.create_generated(nat.SC_SES, n, d, seed, nat.GEN_DISTS[dist],
                                                 shard=(world, r, r0, r1 - r0))
            assert np.array_equal(v1s, v1)
            parts.append(hs.read_rows())
            Ds.append(Ds_r)
            hs.close()
        assert np.array_equal(np.concatenate(parts), X)
        assert max(Ds[-world:]) == D
    # a different seed gives different rows
    h2, _, _ = eng.create_generated(nat.SC_SES, n, d, seed + 1, nat.GEN_DISTS[dist])
    assert not np.array_equal(h2.read_rows(), X)
    h.close()
    h2.close()


def test_svm_rows_invariants_and_sharding():
    eng = nat.cuda_engine()
    n1, n2, d, seed, gap = 700, 500, 24, 5, 0.5
    inst = gen_svm_device(n1, n2, d, seed, gap)
    X = inst.dev.handle.read_rows()
    P, Q = X[:n1], X[n1:]
    shift = (1.0 + gap / 2.0) * inst.axis
    assert np.linalg.norm(P - shift, axis=1).max() <= 1.0 + 1e-12
    assert np.linalg.norm(Q + shift, axis=1).max() <= 1.0 + 1e-12
    assert (P @ inst.axis).min() - (Q @ inst.axis).max() >= gap - 1e-12
    D_np = float(np.linalg.norm(X, axis=1).max())
    assert abs(inst.D - D_np) <= 1e-13 * D_np
    w0 = P.mean(axis=0) - Q.mean(axis=0)
    assert np.allclose(inst.w0, w0, rtol=1e-12, atol=1e-12)
    parts = []
    for r, (r0, r1) in enumerate(row_ranges(n1 + n2, 3)):
        hs, _, _ = eng.create_generated(nat.SC_SVM, n1 + n2, d, seed, nat.SC_GEN_SVM_CLUSTERS,
                                        n1=n1, gap=gap, direction=inst.axis,
                                        shard=(3, r, r0, r1 - r0))
        parts.append(hs.read_rows())
        hs.close()
    assert np.array_equal(np.concatenate(parts), X)
    inst.close()


def test_generated_arguments_rejected():
    eng = nat.cuda_engine()
    with pytest.raises(nat.NativeError):
        eng.create_generated(nat.SC_SES, 100, 8, 0, nat.SC_GEN_SVM_CLUSTERS)
    with pytest.raises(nat.NativeError):      # SVM without a direction
        eng.create_generated(nat.SC_SVM, 100, 8, 0, nat.SC_GEN_SVM_CLUSTERS, n1=50)
    with pytest.raises(ValueError):
        gen_ses_device(100, 8, 0, dist="cube")


def test_ses_solve_generated_equals_uploaded():
    inst = gen_ses_device(3000, 20, seed=3, dist="uniform-ball")
    X = inst.dev.handle.read_rows()
    host = SesInstance(centers=X, radii=np.zeros(X.shape[0]))
    # pin the range to numpy's value so both paths see identical constants
    D_np = float(np.linalg.norm(X[1:] - X[0], axis=1).max())
    inst.dev.handle.set_range(D_np)
    inst.D = D_np
    rep_g, sol_g = solve_ses(inst, 1e-2)
    rep_h, sol_h = solve_ses(host, 1e-2)
    assert rep_g.total_iterations == rep_h.total_iterations
    assert sol_g.radius == sol_h.radius
    assert np.array_equal(sol_g.center, sol_h.center)
    assert sol_g.enclosure_slack == sol_h.enclosure_slack
    inst.close()


def test_svm_solve_generated_equals_uploaded():
    n1, n2 = 1500, 1200
    inst = gen_svm_device(n1, n2, 16, seed=9, gap=0.4)
    X = inst.dev.handle.read_rows()
    host = SvmInstance(P=X[:n1], Q=X[n1:])
    inst.dev.handle.set_range(host.max_norm)
    inst.D = host.max_norm
    inst.w0 = host.P.mean(axis=0) - host.Q.mean(axis=0)
    rep_g, sol_g = solve_svm(inst, 1e-2)
    rep_h, sol_h = solve_svm(host, 1e-2)
    assert rep_g.total_iterations == rep_h.total_iterations
    assert sol_g.margin == sol_h.margin
    assert np.array_equal(sol_g.w, sol_h.w)
    assert sol_g.pd_distance == sol_h.pd_distance
    # the clusters are gap apart along the axis, so the margin is at least gap/2
    assert sol_g.margin >= 0.4 / 2 * (1 - 1e-2) - 1e-9
    inst.close()
