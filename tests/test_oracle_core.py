"""Pins the oracle's core/volume restatement against the reference's own unit
tests (proj/tests/test_core.cpp, test_volume.cpp).  CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Pose, Volume


def rot_axis(axis, ang):
    a = np.asarray(axis, float)
    a = a / np.linalg.norm(a)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(ang) * k + (1 - np.cos(ang)) * k @ k


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def test_euler_convention_is_rz_ry_rx():  # test_core.cpp:19-25
    abc = (0.3, -0.7, 1.1)
    r = rot_axis((0, 0, 1), abc[2]) @ rot_axis((0, 1, 0), abc[1]) @ rot_axis((1, 0, 0), abc[0])
    assert np.linalg.norm(O.euler_to_matrix(abc) - r) < 1e-12


def test_euler_round_trip():  # test_core.cpp:27-35
    rng = np.random.default_rng(11)
    for _ in range(200):
        r = random_rotation(rng)
        assert np.linalg.norm(O.euler_to_matrix(O.matrix_to_euler(r)) - r) < 1e-12


@pytest.mark.parametrize("eps", [0.0, 1e-9, 1e-5])
def test_euler_gimbal(eps):  # test_core.cpp:37-43
    r = O.euler_to_matrix((0.4, np.pi / 2 - eps, -0.9))
    back = O.euler_to_matrix(O.matrix_to_euler(r))
    c = (np.trace(r.T @ back) - 1) * 0.5
    assert np.arccos(np.clip(c, -1, 1)) < 1e-6


def test_svd3_matches_numpy():
    rng = np.random.default_rng(5)
    for _ in range(300):
        a = rng.normal(size=(3, 3))
        if rng.random() < 0.2:  # rank-deficient cases
            a[:, 2] = a[:, 0] * rng.normal()
        u, s, v = O.svd3(a)
        assert np.allclose(u @ np.diag(s) @ v.T, a, atol=1e-12)
        assert np.allclose(u.T @ u, np.eye(3), atol=1e-12)
        assert np.allclose(v.T @ v, np.eye(3), atol=1e-12)
        assert np.all(np.diff(s) <= 0)
        assert np.allclose(s, np.linalg.svd(a, compute_uv=False), atol=1e-12)


def make_grid():  # test_volume.cpp:11-13
    return Volume((8, 8, 8), 0.1, (-0.4, -0.4, 1.0))


def test_anchors_sum_to_one_and_exact_at_nodes():  # test_volume.cpp:26-51
    v = make_grid()
    rng = O.Rng(3)
    for _ in range(100):
        x = v.origin + np.array([rng.uniform(0, 0.7) for _ in range(3)])
        idx, w = O.trilinear_anchors(v, x)
        assert abs(w.sum() - 1) < 1e-12
        assert np.linalg.norm(w @ v.canonical_positions()[idx] - x) < 1e-12
    i = v.linear_index(2, 3, 4)
    idx, w = O.trilinear_anchors(v, v.canonical_position(i))
    best = int(np.argmax(w))
    assert abs(w[best] - 1) < 1e-12 and idx[best] == i


def test_contains_slack():  # test_volume.cpp:53-67
    v = make_grid()
    hi = v.origin + v.voxel_size * (np.array(v.dims) - 1)
    assert O.contains(v, hi) and O.contains(v, hi + 1e-12)
    assert not O.contains(v, hi + 1e-3)
    assert O.contains(v, v.origin) and not O.contains(v, v.origin - 1e-3)
    idx, _ = O.trilinear_anchors(v, hi)
    assert idx.min() >= 0 and idx.max() < v.num_points
    with pytest.raises(O.OracleError):
        O.trilinear_anchors(v, hi + 1e-3)


def test_interpolate_identity():  # test_volume.cpp:69-73
    v = make_grid()
    x = np.array([-0.07, 0.21, 1.33])
    assert np.linalg.norm(O.warp_point(v, Pose.make(), x) - x) < 1e-12
