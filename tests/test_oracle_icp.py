"""Oracle restatement of the global-pose ICP (estimate_global_pose,
solver.cpp:536-614) and of the Eigen LDLT it solves with, pinned by
properties: LDLT against a dense solve (incl. pivoting and the pseudo-inverse
of a zero pivot), ICP recovering a rigid translation of the observed sphere,
refusing non-improving steps, and the degraded path (too few
correspondences: pose unchanged)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import (CorrespondParams, Frame, FusionParams, IcpParams, Intrinsics, Pose,
                                       Volume)

K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)


def test_ldlt_matches_dense_solve():
    rng = np.random.default_rng(5)
    for n in (1, 3, 6, 8):
        m = rng.normal(size=(n, n))
        a = m @ m.T + 0.05 * np.eye(n)
        b = rng.normal(size=n)
        np.testing.assert_allclose(O.ldlt_solve(a, b), np.linalg.solve(a, b), rtol=1e-10, atol=1e-12)
    # pivoting: a tiny leading diagonal entry moves behind the larger ones
    a = np.diag([1e-6, 5.0, 2.0, 7.0, 0.5, 3.0])
    a[0, 5] = a[5, 0] = 1e-4
    b = np.arange(1.0, 7.0)
    np.testing.assert_allclose(a @ O.ldlt_solve(a, b), b, rtol=1e-12, atol=1e-12)
    # zero pivot: pseudo-inverse of D (the component is set to zero)
    a = np.zeros((3, 3))
    a[0, 0] = 2.0
    np.testing.assert_array_equal(O.ldlt_solve(a, np.array([4.0, 1.0, 1.0])), [2.0, 0.0, 0.0])


def sphere_setup(n=48, shift=(0.0, 0.0, 0.0)):
    """Bootstrap-fuse the sphere at the origin pose, then observe it shifted;
    returns the model geometry buffer (identity pose), the observed maps and
    the volume."""
    voxel = 0.7 / (n - 1)
    vol = Volume((n, n, n), voxel, (-0.35, -0.35, 0.85))
    d0, c0 = O.synth_render(K)
    f0 = Frame(K, d0, c0)
    boot = FusionParams.make()
    boot.bootstrap = 1
    O.integrate_frame(vol, f0, Pose.make(), boot)
    O.compute_active_set(vol)
    d1, c1 = O.synth_render(K, center=tuple(np.array([0.0, 0.0, 1.2]) + np.array(shift)))
    maps = O.backproject_depth(Frame(K, d1, c1))
    mesh = O.extract_mesh(vol)
    mesh.compute_normals()
    buf = mesh.rasterize(K)
    return buf, maps, vol


def test_icp_identity_converges_without_moving():
    buf, maps, vol = sphere_setup()
    r = O.estimate_global_pose(buf, maps, K, vol, Pose.make(), IcpParams.make())
    assert not r.degraded and r.converged
    assert r.iterations >= 1
    # the fused surface sits ~0.2 mm off the analytic sphere: the pose stays within that
    assert np.linalg.norm(r.pose.vector()) < 5e-4
    assert np.abs(r.pose.matrix() - np.eye(3)).max() < 1e-4
    assert r.rms < 1e-3


def test_icp_recovers_translation():
    shift = np.array([0.008, -0.006, 0.01])
    buf, maps, vol = sphere_setup(shift=tuple(shift))
    r = O.estimate_global_pose(buf, maps, K, vol, Pose.make(), IcpParams.make())
    assert not r.degraded and r.iterations >= 2
    # for a sphere a lateral shift and a rotation about the camera are the same
    # motion, so the pose is not unique -- where it puts the sphere's centre is
    c0 = np.array([0.0, 0.0, 1.2])
    moved = r.pose.matrix() @ c0 + r.pose.vector() - c0
    assert np.linalg.norm(moved - shift) < 5e-4, moved
    rt = r.pose.matrix()
    np.testing.assert_allclose(rt @ rt.T, np.eye(3), atol=1e-12)
    assert np.linalg.det(rt) == pytest.approx(1.0, abs=1e-12)


def test_icp_steps_only_lower_the_error():
    shift = np.array([0.004, 0.0, -0.004])
    buf, maps, vol = sphere_setup(shift=tuple(shift))
    prev = np.inf
    for iters in range(1, 6):
        r = O.estimate_global_pose(buf, maps, K, vol, Pose.make(), IcpParams.make(max_iters=iters))
        assert r.rms <= prev * (1 + 1e-12)
        prev = r.rms


def test_icp_degraded_keeps_pose():
    buf, maps, vol = sphere_setup()
    empty = O.backproject_depth(Frame(K, np.zeros((240, 320), np.float32)))
    init = Pose.make(translation=[0.01, 0.02, -0.03])
    r = O.estimate_global_pose(buf, empty, K, vol, init, IcpParams.make())
    assert r.degraded and r.iterations == 0
    np.testing.assert_array_equal(r.pose.vector(), init.vector())
    np.testing.assert_array_equal(r.pose.matrix(), init.matrix())
