"""Pins the oracle's fusion restatement against proj/tests/test_fusion.cpp and
acceptance.cpp criterion 9.  CPU only."""
import numpy as np

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import EXEC_PARALLEL, EXEC_SERIAL, FusionParams, Pose, Volume
from tests.fixtures import plane_frame


def small_volume():  # test_fusion.cpp:18-20
    return Volume((10, 10, 10), 0.03, (-0.135, -0.135, 1.2))


def test_running_average():  # test_fusion.cpp:24-44
    v = small_volume()
    p = FusionParams.make(bootstrap=1)
    O.integrate_frame(v, plane_frame(1.32, 100.0), Pose.make(), p)
    i = v.linear_index(4, 4, 2)
    sdf1 = min(1.32 - v.canonical_position(i)[2], v.truncation)
    assert abs(v.tsdf[i] - sdf1) <= 1e-6 * abs(sdf1)
    assert v.weight[i] == 1.0 and abs(v.color[i, 0] - 100) < 1e-4
    O.integrate_frame(v, plane_frame(1.30, 40.0), Pose.make(), p)
    sdf2 = min(1.30 - v.canonical_position(i)[2], v.truncation)
    assert abs(v.tsdf[i] - 0.5 * (sdf1 + sdf2)) <= 1e-6 * abs(0.5 * (sdf1 + sdf2))
    assert v.weight[i] == 2.0 and abs(v.color[i, 0] - 70) < 1e-4


def test_weight_saturates():  # test_fusion.cpp:46-54
    v = small_volume()
    p = FusionParams.make(bootstrap=1, w_max=3.0)
    for _ in range(6):
        O.integrate_frame(v, plane_frame(1.32), Pose.make(), p)
    assert v.weight[v.linear_index(4, 4, 2)] == 3.0


def test_age_gate():  # test_fusion.cpp:56-79
    v = small_volume()
    v.active[:] = 1
    p = FusionParams.make()
    s0 = O.integrate_frame(v, plane_frame(1.32), Pose.make(), p)
    assert s0.fused == 0 and s0.skipped_gate == v.num_points
    allidx = np.arange(v.num_points, dtype=np.int32)
    O.advance_ages(v, allidx)
    O.advance_ages(v, allidx)
    assert O.integrate_frame(v, plane_frame(1.32), Pose.make(), p).fused == 0
    O.advance_ages(v, allidx)
    s3 = O.integrate_frame(v, plane_frame(1.32), Pose.make(), p)
    assert s3.fused > 0 and s3.skipped_gate == 0
    v.active[v.linear_index(4, 4, 2)] = 0
    assert O.integrate_frame(v, plane_frame(1.32), Pose.make(), p).skipped_gate == 1


def test_occlusion():  # test_fusion.cpp:81-94
    v = small_volume()
    s = O.integrate_frame(v, plane_frame(1.25), Pose.make(), FusionParams.make(bootstrap=1))
    assert s.skipped_occluded > 0
    assert v.weight[v.linear_index(4, 4, 9)] == 0.0
    front = v.linear_index(4, 4, 0)
    expect = min(1.25 - 1.2, v.truncation)
    assert abs(v.tsdf[front] - expect) <= 1e-6 * expect


def test_exec_independent():  # test_fusion.cpp:96-106
    a, b = small_volume(), small_volume()
    p = FusionParams.make(bootstrap=1)
    O.integrate_frame(a, plane_frame(1.3), Pose.make(), p, EXEC_PARALLEL)
    O.integrate_frame(b, plane_frame(1.3), Pose.make(), p, EXEC_SERIAL)
    assert np.array_equal(a.tsdf, b.tsdf) and np.array_equal(a.weight, b.weight)


def test_expansion_rigid_extrapolation():  # test_fusion.cpp:108-137
    v = small_volume()
    O.integrate_frame(v, plane_frame(1.32), Pose.make(), FusionParams.make(bootstrap=1))
    O.compute_active_set(v)
    r = O.euler_to_matrix((0.1, -0.05, 0.2))
    t = np.array([0.04, 0.01, -0.02])
    e = O.matrix_to_euler(r)
    act = v.active.astype(bool)
    v.deformed[act] = v.canonical_positions()[act] @ r.T + t
    v.euler[act] = e
    v.age[act] = 7
    v.tsdf[:] = (1.365 - v.canonical_positions()[:, 2]).astype(np.float32)
    s = O.expand_grid(v)
    assert s.activated > 0 and s.orphans == 0
    for i in np.nonzero(v.active)[0]:
        assert np.linalg.norm(v.deformed[i] - (r @ v.canonical_position(i) + t)) < 1e-9
        if v.age[i] == 0:
            assert np.linalg.norm(O.euler_to_matrix(v.euler[i]) - r) < 1e-9


def test_acceptance_c9_exact_average_and_permutation():  # acceptance.cpp:685-743
    v = small_volume()
    boot = FusionParams.make(bootstrap=1)
    depths = (1.32, 1.30)
    for z in depths:
        O.integrate_frame(v, plane_frame(z), Pose.make(), boot)
    for (x, y, z) in ((4, 4, 2), (2, 7, 4), (8, 1, 3)):
        k = v.linear_index(x, y, z)
        zz = O.warp_point(v, Pose.make(), v.canonical_position(k))[2]
        d0 = min(float(np.float32(depths[0])) - zz, v.truncation)
        d1 = min(float(np.float32(depths[1])) - zz, v.truncation)
        expected = np.float32((1.0 * float(np.float32(d0)) + 1.0 * d1) / 2.0)
        assert v.tsdf[k] == expected and v.weight[k] == 2.0
    zs = [1.32, 1.30, 1.33, 1.29, 1.31, 1.305]
    fwd, rev = small_volume(), small_volume()
    for z in zs:
        O.integrate_frame(fwd, plane_frame(z), Pose.make(), boot)
    for z in reversed(zs):
        O.integrate_frame(rev, plane_frame(z), Pose.make(), boot)
    m = (fwd.weight > 0) & (rev.weight > 0)
    assert np.max(np.abs(fwd.tsdf[m].astype(float) - rev.tsdf[m].astype(float))) < 1e-6
