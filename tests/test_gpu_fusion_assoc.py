"""Parity of the B200 fusion and association kernels (libwfk.so) against the
oracle.  Everything here is decided by fp64 geometry evaluated in the
reference's operation order, so the outputs are compared bit for bit:
fusion values and FusionStats, active sets, back-projection maps, the marching
cubes mesh (vertex numbering, triangle order, positions, colors), normals,
the rasterised geometry buffer and the selected correspondences."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import (CORR_DTYPE, CorrespondParams, Frame, FusionParams, Intrinsics, Pose,
                                       Volume)
from tests.fixtures import K320, plane_frame, sphere_tsdf, sphere_volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def sphere_frame(k=K320, center=(0.02, -0.01, 1.2), radius=0.3, holes=True):
    """Analytic depth + color of a sphere (ray/sphere intersection)."""
    ys, xs = np.mgrid[0:k.height, 0:k.width]
    d = np.stack([(xs - k.cx) / k.fx, (ys - k.cy) / k.fy, np.ones_like(xs, float)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    c = np.asarray(center)
    b = d @ c
    disc = b * b - c @ c + radius * radius
    t = b - np.sqrt(np.maximum(disc, 0))
    depth = np.where(disc > 0, t * d[..., 2], 0).astype(np.float32)
    if holes:
        depth[::17, ::13] = 0
    color = (np.stack([xs % 255, ys % 255, (xs + ys) % 255], -1)).astype(np.float32)
    return Frame(k, depth, color)


def assert_volume_equal(a: Volume, b: Volume, fields=("tsdf", "weight", "color", "age", "active")):
    for f in fields:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


@pytest.mark.parametrize("bootstrap", [1, 0])
def test_integrate_bit_exact(ctx, bootstrap):
    v = Volume((40, 40, 40), 0.018, (-0.35, -0.35, 0.85))
    v.deformed += np.random.default_rng(0).uniform(-0.004, 0.004, v.deformed.shape)
    if not bootstrap:
        v.active[::2] = 1
        v.age[:] = np.random.default_rng(1).integers(0, 6, v.num_points)
    ref = v.copy()
    pose = Pose.make(O.euler_to_matrix((0.01, -0.02, 0.015)), (0.003, -0.002, 0.01))
    fr = sphere_frame()
    p = FusionParams.make(bootstrap=bootstrap)
    s_ref = O.integrate_frame(ref, fr, pose, p)
    ctx.upload_volume(v)
    ctx.upload_frame(fr)
    s = ctx.integrate_frame(pose, p)
    ctx.download_volume(v)
    assert s.as_tuple() == s_ref.as_tuple()
    assert s.fused > 1000
    assert_volume_equal(v, ref)


def test_integrate_plane_kats(ctx):  # test_fusion.cpp:24-54, acceptance C9
    v = Volume((10, 10, 10), 0.03, (-0.135, -0.135, 1.2))
    ref = v.copy()
    p = FusionParams.make(bootstrap=1, w_max=3.0)
    ctx.upload_volume(v)
    for z, g in ((1.32, 100.0), (1.30, 40.0), (1.33, 7.0), (1.31, 250.0)):
        fr = plane_frame(z, g)
        s_ref = O.integrate_frame(ref, fr, Pose.make(), p)
        ctx.upload_frame(fr)
        s = ctx.integrate_frame(Pose.make(), p)
        assert s.as_tuple() == s_ref.as_tuple()
    ctx.download_volume(v)
    assert_volume_equal(v, ref)


def test_age_gate_and_ages(ctx):  # test_fusion.cpp:56-79
    v = Volume((10, 10, 10), 0.03, (-0.135, -0.135, 1.2))
    v.active[:] = 1
    ctx.upload_volume(v)
    ctx.upload_frame(plane_frame(1.32))
    p = FusionParams.make()
    assert ctx.integrate_frame(Pose.make(), p).fused == 0
    ctx.advance_ages(np.arange(v.num_points))
    ctx.advance_active_ages()
    assert ctx.integrate_frame(Pose.make(), p).fused == 0
    ctx.advance_ages(np.arange(v.num_points))
    s3 = ctx.integrate_frame(Pose.make(), p)
    assert s3.fused > 0 and s3.skipped_gate == 0


def test_expand_grid_bit_exact(ctx):
    v = Volume((24, 24, 24), 0.02, (-0.23, -0.23, 0.95))
    fr = sphere_frame(holes=False)
    O.integrate_frame(v, fr, Pose.make(), FusionParams.make(bootstrap=1))
    O.compute_active_set(v)
    act = v.active.astype(bool)
    rng = np.random.default_rng(3)
    v.deformed[act] += rng.uniform(-0.003, 0.003, (act.sum(), 3))
    v.euler[act] = rng.uniform(-0.1, 0.1, (act.sum(), 3))
    v.age[act] = 4
    # move the surface so the active set must grow
    sphere_tsdf(v, (0.02, -0.01, 1.2), 0.27)
    v.tsdf[:] = np.clip(v.tsdf, -v.truncation, v.truncation)
    ref = v.copy()
    s_ref = O.expand_grid(ref)
    ctx.upload_volume(v)
    s = ctx.expand_grid()
    ctx.download_volume(v)
    assert (s.activated, s.orphans) == (s_ref.activated, s_ref.orphans)
    assert s.activated > 0
    assert_volume_equal(v, ref, ("active", "age"))
    new = ref.active.astype(bool) & ~act
    # rigid extrapolation uses R_j = euler_to_matrix (device sin/cos): 1e-15 m
    assert np.max(np.abs(v.deformed - ref.deformed)) < 1e-14
    assert np.array_equal(v.euler, ref.euler)
    assert new.sum() == s.activated


def test_backproject_bit_exact(ctx):
    fr = sphere_frame()
    m_ref = O.backproject_depth(fr)
    ctx.upload_frame(fr)
    m = ctx.backproject_depth()
    assert np.array_equal(m.point_valid, m_ref.point_valid)
    assert np.array_equal(m.normal_valid, m_ref.normal_valid)
    assert np.array_equal(m.point, m_ref.point)
    assert np.array_equal(m.normal, m_ref.normal)


def fused_sphere_volume(n=48):
    voxel = 0.7 / (n - 1)
    v = Volume((n, n, n), voxel, (-0.35, -0.35, 0.85))
    O.integrate_frame(v, sphere_frame(holes=False), Pose.make(), FusionParams.make(bootstrap=1))
    O.compute_active_set(v)
    return v


def test_extract_mesh_bit_exact(ctx):
    v = fused_sphere_volume()
    v.color[:] = np.random.default_rng(4).uniform(0, 255, v.color.shape).astype(np.float32)
    act = v.active.astype(bool)
    v.deformed[act] += np.random.default_rng(5).uniform(-0.002, 0.002, (act.sum(), 3))
    pose = Pose.make(O.euler_to_matrix((0.0, 0.02, 0.01)), (0.004, 0.0, -0.003))
    mr = O.extract_mesh(v, pose)
    ctx.upload_volume(v)
    nv, nt = ctx.extract_mesh(pose)
    assert (nv, nt) == (len(mr.vertices_canonical), len(mr.triangles))
    assert nt > 1000
    m = ctx.download_mesh()
    assert np.array_equal(m.triangles, mr.triangles)
    assert np.array_equal(m.vertices_canonical, mr.vertices_canonical)
    assert np.array_equal(m.vertices_deformed, mr.vertices_deformed)
    assert np.array_equal(m.colors, mr.colors)
    mr.compute_normals()
    ctx.compute_normals()
    m = ctx.download_mesh()
    assert np.array_equal(m.normals_deformed, mr.normals_deformed)


def test_mc_kats_on_device(ctx):  # test_isosurface.cpp:33-72
    center = np.array([0.05, -0.03, 1.2])
    v = sphere_volume(40, 0.025, center, 0.31)
    ctx.upload_volume(v)
    ctx.extract_mesh(Pose.make())
    m = ctx.download_mesh()
    assert len(m.vertices_canonical) > 500
    assert np.max(np.abs(np.linalg.norm(m.vertices_canonical - center, axis=1) - 0.31)) < 0.0125
    mr = O.extract_mesh(v)
    assert np.array_equal(m.triangles, mr.triangles)
    v = Volume((12, 12, 12), 0.05, (0, 0, 1.0))
    v.tsdf[:] = (v.canonical_positions()[:, 2] - 1.2625).astype(np.float32)
    v.weight[:] = 1
    ctx.upload_volume(v)
    ctx.extract_mesh(Pose.make())
    m = ctx.download_mesh()
    assert np.max(np.abs(m.vertices_canonical[:, 2] - 1.2625)) < 1e-9


def test_rasterize_bit_exact(ctx):
    v = fused_sphere_volume()
    mr = O.extract_mesh(v)
    mr.compute_normals()
    K = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)
    br = mr.rasterize(K)
    ctx.upload_volume(v)
    ctx.extract_mesh(Pose.make())
    ctx.compute_normals()
    b = ctx.rasterize(K)
    assert np.array_equal(b.depth, br.depth)
    assert np.array_equal(b.point, br.point)
    assert np.array_equal(b.normal, br.normal)
    assert np.array_equal(b.canonical, br.canonical)
    assert np.isfinite(b.depth).sum() > 10000


def test_rasterize_ties_lower_index_wins(ctx):
    # two coincident triangles with different canonical pre-images
    from types import SimpleNamespace
    K = Intrinsics.make(100, 100, 15.5, 15.5, 32, 32)
    verts = np.array([[-0.1, -0.1, 1.0], [0.1, -0.1, 1.0], [0.0, 0.1, 1.0]])
    m = SimpleNamespace(vertices_canonical=np.concatenate([verts, verts + 5.0]),
                        vertices_deformed=np.concatenate([verts, verts]),
                        normals_deformed=np.tile([0.0, 0.0, -1.0], (6, 1)),
                        colors=np.zeros((6, 3), np.float32),
                        triangles=np.array([[3, 4, 5], [0, 1, 2]], np.int32))
    ctx.upload_mesh(m)
    b = ctx.rasterize(K)
    val = np.isfinite(b.depth)
    assert val.sum() > 20
    assert np.all(b.canonical[val][:, 0] > 4)  # triangle 0 (canonical +5) wins every tie
    from oracle.pyoracle import Mesh, lib, _check
    import ctypes as C
    from paper_1603_08161_b200.abi import MeshView, ptr
    can, de, nr = m.vertices_canonical.copy(), m.vertices_deformed.copy(), m.normals_deformed.copy()
    col, tri = m.colors.copy(), m.triangles.copy()
    mv = MeshView(6, 2, ptr(can, C.c_double), ptr(de, C.c_double), ptr(nr, C.c_double), ptr(col, C.c_float),
                  ptr(tri, C.c_int32))
    h = C.c_void_p()
    _check(lib().wfo_mesh_import(C.byref(mv), C.byref(h)))
    br = Mesh(h).rasterize(K)
    assert np.array_equal(b.depth, br.depth) and np.array_equal(b.canonical, br.canonical)


def test_dense_correspondences_bit_exact(ctx):
    v = fused_sphere_volume()
    act = v.active.astype(bool)
    v.deformed[act] += np.random.default_rng(6).uniform(-0.003, 0.003, (act.sum(), 3))
    K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
    fr = sphere_frame(K, center=(0.025, -0.012, 1.205))
    mr = O.extract_mesh(v)
    mr.compute_normals()
    br = mr.rasterize(K)
    maps = O.backproject_depth(fr)
    cp = CorrespondParams.make()
    cr = O.find_dense_correspondences(br, maps, K, cp, v)
    ctx.upload_volume(v)
    ctx.upload_frame(fr)
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(Pose.make())
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    n = ctx.find_dense_correspondences(K, cp, drop_inactive=False)
    assert n == len(cr) and n > 1000
    got = ctx.download_constraints()
    for f in ("kind", "canonical", "anchor_index", "anchor_weight", "target", "target_normal", "confidence"):
        assert np.array_equal(got[f], cr[f]), f
    # pipeline.cpp:220-229 anchor filter
    n2 = ctx.find_dense_correspondences(K, cp, drop_inactive=True)
    keep = np.all(v.active[cr["anchor_index"]] != 0, axis=1)
    assert n2 == keep.sum()


def test_dense_association_plane_kat(ctx):  # test_correspond.cpp:78-107
    fr = plane_frame(1.4)
    v = Volume((16, 16, 16), 0.02, (-0.15, -0.15, 1.25))
    v.tsdf[:] = (1.4 - v.canonical_positions()[:, 2]).astype(np.float32)
    v.weight[:] = 1
    ctx.upload_volume(v)
    ctx.upload_frame(fr)
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(Pose.make())
    ctx.compute_normals()
    ctx.rasterize(fr.intrinsics, download=False)
    n = ctx.find_dense_correspondences(fr.intrinsics, CorrespondParams.make())
    c = ctx.download_constraints()
    assert n > 1000
    assert np.all(c["confidence"] > 0.95)
    assert np.max(np.linalg.norm(c["target"] - c["canonical"], axis=1)) < 1e-6


def test_mesh_warp_bit_exact(ctx):
    """redeform (pipeline.cpp:167-172): mesh vertices re-warped through a new field and pose"""
    v = fused_sphere_volume()
    pose0 = Pose.make()
    mr = O.extract_mesh(v, pose0)
    ctx.upload_volume(v)
    ctx.extract_mesh(pose0)
    act = v.active.astype(bool)
    v.deformed[act] += np.random.default_rng(8).uniform(-0.003, 0.003, (act.sum(), 3))
    pose = Pose.make(O.euler_to_matrix((0.01, -0.02, 0.03)), (0.002, 0.001, -0.004))
    ctx.upload_volume(v)
    ctx.mesh_warp(pose)
    mr.warp(v, pose)
    m = ctx.download_mesh()
    assert np.array_equal(m.vertices_deformed, mr.vertices_deformed)


def test_constraints_append_drops_inactive(ctx):
    """wfk_constraints_append: caller records after the dense ones, keeping only
    those whose eight anchors are active (pipeline.cpp:229-236)"""
    from tests.fixtures import active_sphere_volume, random_dense_constraints, rigid_motion_constraints
    v = active_sphere_volume(12, 0.05)
    dense = random_dense_constraints(v, 50, seed=2)
    sparse = rigid_motion_constraints(v, np.eye(3), (0.01, 0.0, 0.0))
    sparse["kind"] = 1  # WFK_SPARSE_POINT
    # deactivate one anchor of every third record
    for i in range(0, len(sparse), 3):
        v.active[sparse["anchor_index"][i][0]] = 0
    ctx.upload_volume(v)
    ctx.upload_constraints(dense)
    kept = ctx.append_constraints(sparse, drop_inactive=True)
    keep = np.array([all(v.active[a] for a in s["anchor_index"]) for s in sparse])
    assert kept == keep.sum() and 0 < kept < len(sparse)
    got = ctx.download_constraints()
    assert len(got) == len(dense) + kept
    assert got[: len(dense)].tobytes() == np.ascontiguousarray(dense, CORR_DTYPE).tobytes()
    assert got[len(dense):].tobytes() == np.ascontiguousarray(sparse[keep], CORR_DTYPE).tobytes()
