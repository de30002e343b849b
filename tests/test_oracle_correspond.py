"""Pins the oracle's association / isosurface / raster restatement against
proj/tests/test_correspond.cpp, test_isosurface.cpp and acceptance.cpp
criteria 8 and 10.  CPU only."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import (DENSE_PLANE, EXEC_PARALLEL, EXEC_SERIAL, SPARSE_POINT,
                                       CorrespondParams, Intrinsics, Pose, Volume)
from tests.fixtures import K320, plane_frame, sphere_volume


def test_confidence_kat_exact():  # acceptance.cpp:663-679, test_correspond.cpp:26-37
    p = CorrespondParams.make()
    assert O.dense_confidence(0, 1, 1, p) == 1.0
    assert O.dense_confidence(p.eps_d, 1, 1, p) == 4.0 / 9.0
    assert O.dense_confidence(0, 1 - p.eps_n, 1, p) == 4.0 / 9.0
    assert O.dense_confidence(0, 1, 1 - p.eps_v, p) == 4.0 / 9.0
    assert O.dense_confidence(p.eps_d + 1e-9, 1, 1, p) == 0.0
    assert O.dense_confidence(0, 1 - p.eps_n - 1e-9, 1, p) == 0.0
    assert O.dense_confidence(0, 1, 1 - p.eps_v - 1e-9, p) == 0.0


def backproject(k, x, y, d):
    return np.array([(x - k.cx) / k.fx * d, (y - k.cy) / k.fy * d, d])


def test_backprojection_plane():  # test_correspond.cpp:39-61
    f = plane_frame(1.4)
    m = O.backproject_depth(f)
    ms = O.backproject_depth(f, EXEC_SERIAL)
    for y in range(1, m.height - 1, 17):
        for x in range(1, m.width - 1, 13):
            i = y * m.width + x
            assert m.point_valid[i] and m.normal_valid[i]
            assert abs(m.point[i, 2] - 1.4) < 1e-6
            assert np.linalg.norm(m.point[i] - backproject(f.intrinsics, x, y, 1.4)) < 1e-6
            assert np.linalg.norm(m.normal[i] - (0, 0, -1)) < 1e-9
    assert np.array_equal(m.point, ms.point) and np.array_equal(m.normal, ms.normal)
    assert not m.normal_valid[5 * m.width + 0]
    h = plane_frame(1.4)
    h.depth[60, 50] = 0
    mh = O.backproject_depth(h)
    assert not mh.point_valid[60 * 320 + 50] and not mh.normal_valid[60 * 320 + 51]


def test_sample_point_normal():  # test_correspond.cpp:63-76
    f = plane_frame(1.3)
    m = O.backproject_depth(f)
    ok, p, n = O.sample_point_normal(m, (100.5, 80.5))
    assert ok and abs(p[2] - 1.3) < 1e-6
    a = backproject(f.intrinsics, 100, 80, 1.3)
    b = backproject(f.intrinsics, 101, 81, 1.3)
    assert np.linalg.norm(p - 0.5 * (a + b)) < 1e-6
    assert np.linalg.norm(n - (0, 0, -1)) < 1e-9
    assert not O.sample_point_normal(m, (-5, 10))[0]


def plane_volume(plane_z):
    v = Volume((16, 16, 16), 0.02, (-0.15, -0.15, 1.25))
    v.tsdf[:] = (plane_z - v.canonical_positions()[:, 2]).astype(np.float32)
    v.weight[:] = 1.0
    return v


def test_dense_association_plane():  # test_correspond.cpp:78-107
    f = plane_frame(1.4)
    v = plane_volume(1.4)
    mesh = O.extract_mesh(v)
    mesh.compute_normals()
    buf = mesh.rasterize(f.intrinsics)
    corrs = O.find_dense_correspondences(buf, O.backproject_depth(f), f.intrinsics,
                                         CorrespondParams.make(), v)
    assert len(corrs) > 1000
    assert np.all(corrs["kind"] == DENSE_PLANE)
    assert np.all(corrs["confidence"] > 0.95) and np.all(corrs["confidence"] <= 1 + 1e-12)
    assert np.max(np.linalg.norm(corrs["target"] - corrs["canonical"], axis=1)) < 1e-6
    assert np.max(np.linalg.norm(corrs["target_normal"] - (0, 0, -1), axis=1)) < 1e-9
    assert np.max(np.abs(corrs["anchor_weight"].sum(axis=1) - 1)) < 1e-12


def test_dense_association_prunes_by_distance():  # test_correspond.cpp:109-123
    f = plane_frame(1.4)
    v = plane_volume(1.32)
    mesh = O.extract_mesh(v)
    mesh.compute_normals()
    buf = mesh.rasterize(f.intrinsics)
    assert len(O.find_dense_correspondences(buf, O.backproject_depth(f), f.intrinsics,
                                            CorrespondParams.make(), v)) == 0


def test_sparse_constraints_inside_only():  # test_correspond.cpp:125-135
    v = Volume((8, 8, 8), 0.1, (0, 0, 0))
    out = O.sparse_to_constraints([[0.35, 0.35, 0.35], [5, 5, 5]], [[0.36, 0.35, 0.35], [5, 5, 5]], v)
    assert len(out) == 1 and out[0]["kind"] == SPARSE_POINT and out[0]["confidence"] == 1.0
    assert np.array_equal(out[0]["target"], [0.36, 0.35, 0.35])


def euler_characteristic(tris, nv):
    e = set()
    for t in tris:
        for k in range(3):
            a, b = int(t[k]), int(t[(k + 1) % 3])
            e.add((min(a, b), max(a, b)))
    return nv - len(e) + len(tris)


def test_mc_sphere_topology():  # test_isosurface.cpp:33-50
    center = np.array([0.05, -0.03, 1.2])
    v = sphere_volume(40, 0.025, center, 0.31)
    m = O.extract_mesh(v)
    assert len(m.vertices_canonical) > 500
    assert np.max(np.abs(np.linalg.norm(m.vertices_canonical - center, axis=1) - 0.31)) < 0.0125
    assert euler_characteristic(m.triangles, len(m.vertices_canonical)) == 2
    from collections import Counter
    cnt = Counter()
    for t in m.triangles:
        for k in range(3):
            a, b = int(t[k]), int(t[(k + 1) % 3])
            cnt[(min(a, b), max(a, b))] += 1
    assert set(cnt.values()) == {2}


def test_mc_plane_exact():  # test_isosurface.cpp:52-63
    v = Volume((12, 12, 12), 0.05, (0, 0, 1.0))
    v.tsdf[:] = (v.canonical_positions()[:, 2] - 1.2625).astype(np.float32)
    v.weight[:] = 1
    m = O.extract_mesh(v)
    assert len(m.triangles) > 0
    assert np.max(np.abs(m.vertices_canonical[:, 2] - 1.2625)) < 1e-9


def test_mc_unobserved_cells():  # test_isosurface.cpp:65-72
    v = sphere_volume(24, 0.04, (0, 0, 1.2), 0.3)
    v.weight[v.canonical_positions()[:, 0] > 0] = 0
    m = O.extract_mesh(v)
    assert len(m.triangles) > 0 and np.all(m.vertices_canonical[:, 0] <= 0.04 + 1e-9)


def test_winding_normals_outward():  # test_isosurface.cpp:74-82
    m = O.extract_mesh(sphere_volume(32, 0.025, (0, 0, 1.2), 0.3))
    m.compute_normals()
    radial = m.vertices_deformed - (0, 0, 1.2)
    radial /= np.linalg.norm(radial, axis=1)[:, None]
    assert np.all(np.sum(m.normals_deformed * radial, axis=1) > 0.8)


def test_warped_vertices():  # test_isosurface.cpp:84-94
    v = sphere_volume(24, 0.04, (0, 0, 1.2), 0.3)
    shift = np.array([0.07, -0.02, 0.05])
    v.deformed += shift
    pose = Pose.make(O.euler_to_matrix((0, 0.1, 0)), (0.01, 0, 0))
    m = O.extract_mesh(v, pose)
    exp = (m.vertices_canonical + shift) @ pose.matrix().T + pose.vector()
    assert np.max(np.linalg.norm(m.vertices_deformed - exp, axis=1)) < 1e-12


def test_rasterizer():  # test_isosurface.cpp:96-127
    center = np.array([0, 0, 1.2])
    m = O.extract_mesh(sphere_volume(40, 0.02, center, 0.3))
    m.compute_normals()
    K = K320
    buf = m.rasterize(K, EXEC_PARALLEL)
    ser = m.rasterize(K, EXEC_SERIAL)
    assert np.array_equal(buf.depth, ser.depth) and np.array_equal(buf.point, ser.point)
    val = buf.valid()
    assert val.sum() > 3000
    p = buf.point[val]
    assert np.max(np.abs(np.linalg.norm(p - center, axis=1) - 0.3)) < 0.02
    assert np.max(np.linalg.norm(buf.canonical[val] - p, axis=1)) < 1e-9
    ys, xs = np.nonzero(val.reshape(K.height, K.width))
    u = K.fx * p[:, 0] / p[:, 2] + K.cx
    vv = K.fy * p[:, 1] / p[:, 2] + K.cy
    assert np.max(np.abs(u - xs)) < 0.51 and np.max(np.abs(vv - ys)) < 0.51
    assert abs(buf.depth[120 * 320 + 160] - 0.9) < 0.02 * 0.9
