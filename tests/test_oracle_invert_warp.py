"""Oracle restatement of DeformableVolume::invert_warp (volume.cpp:68-126,
damped Gauss-Newton with the analytic trilinear Jacobian and Eigen's
PartialPivLU), pinned by the reference's own property (test_volume.cpp:94-107:
the warp of the inverted point reproduces y within 1e-5) and the identity /
rigid fields."""
import numpy as np

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Pose, Volume


def field(n=12, rot=(0.0, 0.0, 0.0), t=(0.0, 0.0, 0.0), jitter=0.0, seed=1):
    v = Volume((n, n, n), 0.05, (-0.3, -0.3, 0.9))
    can = v.canonical_positions()
    r = O.euler_to_matrix(rot)
    v.deformed[:] = can @ r.T + np.asarray(t)
    if jitter:
        v.deformed += np.random.default_rng(seed).uniform(-jitter, jitter, v.deformed.shape)
    return v


def inner_points(v, k=200, seed=3):
    lo = np.asarray(v.origin) + v.voxel_size
    hi = np.asarray(v.origin) + v.voxel_size * (np.asarray(v.dims) - 2)
    return np.random.default_rng(seed).uniform(lo, hi, (k, 3))


def test_identity_field_inverts_to_target():
    v = field()
    x = inner_points(v)
    y = x.copy()
    got, ok = O.invert_warp(v, Pose.make(), y, x + 0.01)
    assert ok.all()
    np.testing.assert_allclose(got, x, atol=1e-6)


def test_rigid_and_jittered_fields_reproduce_y():  # test_volume.cpp:94-107
    for rot, t, jit in [((0.05, -0.03, 0.02), (0.01, -0.02, 0.005), 0.0), ((0.0, 0.02, 0.0), (0, 0, 0), 0.004)]:
        v = field(rot=rot, t=t, jitter=jit)
        x = inner_points(v)
        pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.002, 0.0, -0.001))
        y = np.array([O.warp_point(v, pose, p) for p in x])
        got, ok = O.invert_warp(v, pose, y, x + 0.005)
        assert ok.mean() > 0.98
        back = np.array([O.warp_point(v, pose, p) for p in got[ok]])
        assert np.max(np.linalg.norm(back - y[ok], axis=1)) <= 1e-5


def test_seed_outside_grid_fails():
    v = field()
    got, ok = O.invert_warp(v, Pose.make(), np.array([[0.0, 0.0, 1.1]]), np.array([[5.0, 5.0, 5.0]]))
    assert not ok[0]
