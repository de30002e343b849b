"""Global-pose ICP (estimate_global_pose, solver.cpp:536-614) on the B200
against the oracle restatement, on identical inputs (the volume, the
observed frame and -- bit-exact on both sides -- the mesh, geometry buffer and
maps).  The 6x6 normal equations are summed in a different (fixed) order on
the device, so poses agree to rounding, not bitwise; the decisions (iteration
count, convergence, degraded) must agree exactly."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Frame, FusionParams, IcpParams, Intrinsics, Pose, Volume

pytestmark = pytest.mark.gpu

K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def fused_volume(n=48, jitter=0.0):
    vol = Volume((n, n, n), 0.7 / (n - 1), (-0.35, -0.35, 0.85))
    d0, c0 = O.synth_render(K)
    boot = FusionParams.make()
    boot.bootstrap = 1
    O.integrate_frame(vol, Frame(K, d0, c0), Pose.make(), boot)
    O.compute_active_set(vol)
    if jitter:
        act = vol.active.astype(bool)
        vol.deformed[act] += np.random.default_rng(3).uniform(-jitter, jitter, (act.sum(), 3))
    return vol


def run_both(ctx, vol, frame, initial, params):
    mesh = O.extract_mesh(vol, initial)
    mesh.compute_normals()
    buf = mesh.rasterize(K)
    maps = O.backproject_depth(frame)
    ref = O.estimate_global_pose(buf, maps, K, vol, initial, params)
    ctx.upload_volume(vol)
    ctx.upload_frame(frame)
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(initial)
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    got = ctx.estimate_global_pose(K, initial, params)
    return ref, got


@pytest.mark.parametrize("shift,jitter", [((0.0, 0.0, 0.0), 0.0), ((0.008, -0.006, 0.01), 0.0),
                                          ((-0.004, 0.003, -0.006), 0.002)])
def test_icp_parity(ctx, shift, jitter):
    vol = fused_volume(jitter=jitter)
    d1, c1 = O.synth_render(K, center=tuple(np.array([0.0, 0.0, 1.2]) + np.array(shift)))
    ref, got = run_both(ctx, vol, Frame(K, d1, c1), Pose.make(), IcpParams.make())
    assert got.degraded == ref.degraded == 0
    assert got.iterations == ref.iterations and got.converged == ref.converged
    assert got.rms == pytest.approx(ref.rms, rel=1e-9)
    np.testing.assert_allclose(got.pose.matrix(), ref.pose.matrix(), atol=1e-10)
    np.testing.assert_allclose(got.pose.vector(), ref.pose.vector(), atol=1e-10)


def test_icp_parity_from_nonidentity_pose(ctx):
    vol = fused_volume()
    ang = 0.01
    r0 = np.array([[np.cos(ang), 0, np.sin(ang)], [0, 1, 0], [-np.sin(ang), 0, np.cos(ang)]])
    init = Pose.make(rotation=r0, translation=[0.003, 0.0, -0.002])
    d1, c1 = O.synth_render(K, center=(0.005, 0.0, 1.21))
    ref, got = run_both(ctx, vol, Frame(K, d1, c1), init, IcpParams.make(max_iters=7))
    assert got.iterations == ref.iterations and got.converged == ref.converged
    np.testing.assert_allclose(got.pose.matrix(), ref.pose.matrix(), atol=1e-10)
    np.testing.assert_allclose(got.pose.vector(), ref.pose.vector(), atol=1e-10)


def test_icp_degraded_keeps_pose(ctx):
    vol = fused_volume()
    init = Pose.make(translation=[0.01, 0.02, -0.03])
    ref, got = run_both(ctx, vol, Frame(K, np.zeros((240, 320), np.float32)), init, IcpParams.make())
    assert got.degraded == ref.degraded == 1 and got.iterations == 0
    np.testing.assert_array_equal(got.pose.vector(), init.vector())


def test_icp_from_host_buffers(ctx):
    """The drop-in path: the caller's GeometryBuffer and
    PointNormalMap uploaded as they are, the volume's field re-used."""
    vol = fused_volume(jitter=0.001)
    d1, c1 = O.synth_render(K, center=(0.006, -0.004, 1.207))
    fr = Frame(K, d1, c1)
    mesh = O.extract_mesh(vol)
    mesh.compute_normals()
    buf = mesh.rasterize(K)
    maps = O.backproject_depth(fr)
    params = IcpParams.make()
    ref = O.estimate_global_pose(buf, maps, K, vol, Pose.make(), params)
    ctx.upload_volume(vol)
    ctx.upload_gbuffer(buf)
    ctx.upload_maps(maps)
    got = ctx.estimate_global_pose(K, Pose.make(), params)
    assert got.iterations == ref.iterations and got.converged == ref.converged and not got.degraded
    np.testing.assert_allclose(got.pose.vector(), ref.pose.vector(), atol=1e-10)
    np.testing.assert_allclose(got.pose.matrix(), ref.pose.matrix(), atol=1e-10)
