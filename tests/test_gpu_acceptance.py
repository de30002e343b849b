"""Acceptance criteria of the reference run on the B200 path.

Criterion 3 (acceptance.cpp:399-457): ten identical frames of a large spherical
cap leave the deformation at the identity, the TSDF equal to the analytic
projective TSDF and the canonical mesh on the sphere.

Criterion 4 (acceptance.cpp:460-502): the global-pose ICP tracks a camera
moving rigidly in a five-wall room corner to < 0.1 degree and < 1 mm.

Criterion 7 (acceptance.cpp:616-656): feature
ablation on a tangentially sliding textured plane.  Point-to-plane terms
cannot see motion along the plane; the sparse feature term can, so with the
feature front-end on, the drift of tracked material points must stay below
half of the dense-only drift.  Run on the B200 path (wfk_process_frame) with
the drift tracker of acceptance.cpp:188-214 (wfk_invert_warp).

The scene is rendered here in numpy (test infrastructure): plane z = 1.3 m
facing the camera inside the bounds |x|, |y| <= 0.25 m, the Dots texture of
synthcam.cpp:98-119 (scale 0.03 m, seed 7, dot radius 0.3) on the material
point, rigid translation 2 mm per frame along x, 30 frames at 320x240.
"""
import numpy as np
import pytest

from paper_1603_08161_b200.abi import Frame, Intrinsics, Pose, SolverParams, Volume

pytestmark = pytest.mark.gpu

K = Intrinsics.make(280.0, 280.0, 159.5, 119.5, 320, 240)
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & M64
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return x ^ (x >> np.uint64(31))


def hash_cell(ix, iy, iz, seed):
    h = np.full(ix.shape, np.uint64(seed))
    for v in (ix, iy, iz):
        h = splitmix64(h ^ v.astype(np.int64).view(np.uint64))
    return h


def rand01(h):
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def dots_color(p, scale=0.03, seed=7, dot_radius=0.3):
    """texture_color (synthcam.cpp:98-119), Dots, at material points p (n x 3)"""
    cell = p / scale
    f = np.floor(cell)
    h = hash_cell(f[:, 0], f[:, 1], f[:, 2], seed)
    margin = dot_radius + 0.05
    h1 = splitmix64(h)
    h2 = splitmix64(h1)
    center = f + margin + np.stack([rand01(h), rand01(h1), rand01(h2)], 1) * (1 - 2 * margin)
    inside = np.linalg.norm(cell - center, axis=1) < dot_radius
    hc = splitmix64(h ^ np.uint64(0xD0D5))
    hc1 = splitmix64(hc)
    hc2 = splitmix64(hc1)
    rgb = np.stack([20 + 160 * rand01(hc), 20 + 160 * rand01(hc1), 20 + 160 * rand01(hc2)], 1)
    out = np.full(p.shape, 210.0)
    out[inside] = rgb[inside]
    return out.astype(np.float32)


def shift(f):
    return np.array([0.002 * f, 0.0, 0.0])  # WarpType::Rigid, trans_per_frame


def render(f, z=1.3, half=0.25):
    v, u = np.mgrid[0:K.height, 0:K.width].astype(np.float64)
    p = np.stack([(u - K.cx) / K.fx * z, (v - K.cy) / K.fy * z, np.full(u.shape, z)], -1).reshape(-1, 3)
    inside = (np.abs(p[:, 0]) <= half) & (np.abs(p[:, 1]) <= half)
    depth = np.where(inside, z, 0.0).astype(np.float32).reshape(K.height, K.width)
    color = dots_color(p - shift(f)).reshape(K.height, K.width, 3)
    color[~inside.reshape(K.height, K.width)] = 0
    return Frame(K, depth, color)


def truth_samples(z=1.3, half=0.25, n=17, cap=200):
    """truth_surface_samples (acceptance.cpp:153-186) for the plane: grid points projected onto it"""
    g = np.linspace(-half, half, n)
    pts = [(x, y, z) for y in g for x in g]
    return np.array(pts[:cap])


def tangential_drift(ctx, use_features, frames=30):
    from paper_1603_08161_b200.wfk import pipeline_config
    n, voxel, origin = 64, 0.01, (-0.315, -0.315, 1.0)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make(), use_features=use_features)
    pose = Pose.make()
    pts = truth_samples()
    last = pts.copy()
    ref = np.zeros_like(pts)
    has = np.zeros(len(pts), bool)
    total, count = 0.0, 0
    for f in range(frames):
        rec = ctx.process_frame(render(f), pose, cfg, f)
        pose = rec.pose
        y = pts + shift(f)  # the material points' current world positions
        c, ok = ctx.invert_warp(pose, y, last)
        ok = ok.astype(bool)
        last[ok] = c[ok]
        first = ok & ~has
        ref[first] = c[first]
        again = ok & has
        total += np.linalg.norm(c[again] - ref[again], axis=1).sum()
        count += int(again.sum())
        has |= ok
    return total / count if count else -1.0


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def test_feature_ablation_tangential_drift(ctx):  # acceptance criterion 7
    both = tangential_drift(ctx, True)
    dense_only = tangential_drift(ctx, False)
    print(f"drift sparse+dense {both:.5f} m, dense-only {dense_only:.5f} m, ratio {both / dense_only:.3f}")
    assert both >= 0 and dense_only > 0
    assert both < 0.5 * dense_only


def test_static_sequence_identity(ctx):  # acceptance criterion 3 (acceptance.cpp:399-457)
    """ten identical frames of a large face-on spherical cap: the deformation
    stays the identity, the TSDF matches the analytic projective TSDF and the
    canonical mesh lies on the sphere"""
    from paper_1603_08161_b200.wfk import pipeline_config
    from tools import synthscene as S
    center, radius = np.array([0.0, 0.0, 2.2]), 1.0
    s = S.Scene.make(K, frames=1).add_shape(S.SPHERE, center=tuple(center), radius=radius)  # acceptance.cpp:406-412
    depth, color = S.render(s, 0)
    fr = Frame(K, depth, color)
    n, voxel, origin = 64, 0.01, (-0.315, -0.315, 1.05)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make())
    pose = Pose.make()
    for f in range(10):
        pose = ctx.process_frame(fr, pose, cfg, f).pose
    ctx.download_volume(vol)
    act = vol.active.astype(bool)
    can = vol.canonical_positions()
    max_deform = np.max(np.linalg.norm(vol.deformed[act] - can[act], axis=1))
    # analytic projective TSDF along each voxel's camera ray
    w = vol.weight > 0
    p = can[w]
    d = p / np.linalg.norm(p, axis=1, keepdims=True)
    b = d @ center
    disc = b * b - center @ center + radius * radius
    ok = disc >= 0
    sdf = (b - np.sqrt(np.where(ok, disc, 0))) * d[:, 2] - p[:, 2]
    trunc = 4 * voxel
    ok &= sdf >= -trunc
    sdf = np.minimum(sdf, trunc)
    tsdf_err = np.max(np.abs(vol.tsdf[w][ok] - sdf[ok]))
    nv, nt = ctx.extract_mesh(Pose.make())
    m = ctx.download_mesh()
    mesh_err = np.max(np.abs(np.linalg.norm(m.vertices_canonical - center, axis=1) - radius))
    print(f"max deform {max_deform:.2e} m, tsdf err {tsdf_err:.2e}, mesh err {mesh_err:.2e}")
    assert nt > 0
    assert max_deform < 1e-4
    assert tsdf_err < voxel / 4
    assert mesh_err < voxel / 2


def axis_angle(axis, angle):
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    kx = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(angle) * kx + (1 - np.cos(angle)) * kx @ kx


def room_frame(R, t):
    """the five-wall room of acceptance.cpp:463-478 seen from camera pose (R, t)
    (world -> camera), walls n . p = offset, free space n . p > offset"""
    walls = [((0, 0, -1), -1.45), ((1, 0, 0), -0.26), ((-1, 0, 0), -0.26), ((0, 1, 0), -0.26), ((0, -1, 0), -0.26)]
    v, u = np.mgrid[0:K.height, 0:K.width].astype(np.float64)
    d_cam = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones_like(u)], -1).reshape(-1, 3)
    o_w = -R.T @ t
    d_w = d_cam @ R  # R^T d for each row
    best = np.full(len(d_w), np.inf)
    for n, off in walls:
        n = np.array(n, np.float64)
        nd = d_w @ n
        with np.errstate(divide="ignore", invalid="ignore"):
            th = (off - n @ o_w) / nd
        ok = (nd < 0) & (th > 0)
        best = np.where(ok & (th < best), th, best)
    hit = np.isfinite(best)
    depth = np.where(hit, best, 0.0).astype(np.float32).reshape(K.height, K.width)
    p_w = o_w + best[:, None] * d_w
    color = np.zeros((len(d_w), 3), np.float32)
    color[hit] = dots_color(p_w[hit], scale=0.06)
    return Frame(K, depth, color.reshape(K.height, K.width, 3))


def test_rigid_tracking_room_corner(ctx):  # acceptance criterion 4 (acceptance.cpp:460-502)
    from paper_1603_08161_b200.wfk import pipeline_config
    n, voxel, origin = 64, 0.01, (-0.315, -0.315, 0.95)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make())
    pose = Pose.make()
    worst_rot = worst_trans = 0.0
    for f in range(30):
        R = axis_angle((0.2, 1.0, 0.1), np.deg2rad(0.25) * f)
        t = np.array([0.0015, 0.001, 0.001]) * f
        rec = ctx.process_frame(room_frame(R, t), pose, cfg, f)
        pose = rec.pose
        Rg, tg = rec.pose.matrix(), rec.pose.vector()
        cosang = np.clip((np.trace(Rg.T @ R) - 1) / 2, -1, 1)
        worst_rot = max(worst_rot, np.rad2deg(np.arccos(cosang)))
        worst_trans = max(worst_trans, np.linalg.norm(tg - t))
    print(f"worst pose error {worst_rot:.4f} deg, {worst_trans * 1e3:.3f} mm")
    assert worst_rot < 0.1 and worst_trans < 0.001
