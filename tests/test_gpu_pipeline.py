"""End-to-end parity of the per-frame hot path (Reconstructor::process_frame,
pipeline.cpp:143-262, with the global-pose ICP and the feature front-end):
the B200 path (wfk_process_frame) against the oracle's restatement on the same
synthetic bend sequence."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import FEATURE_DTYPE, CorrespondParams, Frame, FusionParams, Intrinsics, Pose, SolverParams, Volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def bend_frames(ctx, K, n_frames, amplitude, frames_total=10, frequency=0.0, start=0):
    """frames of the bend-sphere sequence (linear ramp over frames_total when
    frequency is 0, synthcam.cpp:138-143), rendered by tools/synthscene --
    bit-identical to the reference's SyntheticScene -- and fed to both sides"""
    from tools import synthscene as S
    sc = S.bend_sphere(K, frames=frames_total, amplitude=amplitude, frequency=frequency)
    return [Frame(K, *S.render(sc, f)) for f in range(start, start + n_frames)]


@pytest.mark.parametrize("n,reassoc,levels,icp", [(32, 1, 1, True), (48, 2, 3, True), (48, 2, 3, False)])
def test_process_frame_parity(ctx, n, reassoc, levels, icp):
    from paper_1603_08161_b200.wfk import pipeline_config
    K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    solver = SolverParams.make(levels=levels)
    frames = bend_frames(ctx, K, 4, 1.0)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=solver, reassociations=reassoc, estimate_pose=icp)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=solver, reassociations=reassoc, estimate_pose=icp)
    pose = Pose.make()
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose  # the Reconstructor's pose_ carried to the next frame
        if i == 0:
            assert rg.fusion.fused == rr.fusion.fused
            continue
        if icp:
            if i == 1:
                assert rg.icp_iterations == rr.icp_iterations and rg.icp_degraded == rr.icp_degraded
            np.testing.assert_allclose(rg.pose.matrix(), rr.pose.matrix(), atol=1e-7)
            np.testing.assert_allclose(rg.pose.vector(), rr.pose.vector(), atol=1e-7)
        if i == 1 and reassoc == 1:  # identical inputs up to this frame's solve: integer work is exact
            assert rg.dense_count == rr.dense_count
            assert rg.trace_len == rr.trace_len
        else:
            assert abs(rg.dense_count - rr.dense_count) <= max(3, 0.002 * rr.dense_count)
        assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-3)
        assert abs(rg.fusion.fused - rr.fusion.fused) <= max(3, 0.002 * rr.fusion.fused)
        assert rg.expansion.activated == pytest.approx(rr.expansion.activated, abs=3)
    ctx.download_volume(vol)
    arr = ref.volume_arrays()
    act = arr["active"].astype(bool)
    assert (vol.active != arr["active"]).sum() <= 8
    both = act & vol.active.astype(bool)
    dev = np.max(np.linalg.norm(vol.deformed[both] - arr["deformed"][both], axis=1)) / voxel
    assert dev <= 1e-3, dev


def test_process_frame_features_parity(ctx):
    """The feature front-end inside process_frame (pipeline.cpp:95-141, 185-217):
    per-frame match / sparse / added counts and the FeatureStore against the oracle."""
    from paper_1603_08161_b200.wfk import pipeline_config
    n = 48
    K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    solver = SolverParams.make(levels=3)
    frames = bend_frames(ctx, K, 5, 1.0)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=solver, reassociations=2)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    ctx.set_feature_store(np.zeros(0, FEATURE_DTYPE))
    cfg = pipeline_config(solver=solver, reassociations=2)
    assert cfg.use_features == 1
    pose = Pose.make()
    total_sparse = 0
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose
        if i <= 1:  # identical inputs so far: integer work is exact
            assert rg.features_added == rr.features_added
            assert rg.match_count == rr.match_count and rg.sparse_count == rr.sparse_count
        else:
            assert abs(rg.features_added - rr.features_added) <= 2
            assert abs(rg.match_count - rr.match_count) <= 2
            assert abs(rg.sparse_count - rr.sparse_count) <= 2
        if i > 0:
            assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-3)
        total_sparse += rg.sparse_count
    assert total_sparse > 0, "the sequence should produce sparse feature constraints"
    sg, sr = ctx.feature_store(), ref.feature_store()
    assert abs(len(sg) - len(sr)) <= 4 and len(sr) > 20
    # the bootstrap frame's positions are exact (identity warp), later ones to the inversion tolerance
    b = int((sr["frame_id"] == 0).sum())
    assert b > 0 and int((sg["frame_id"] == 0).sum()) == b
    for f in ("pixel", "world_pos", "canonical_pos", "frame_id"):
        np.testing.assert_array_equal(sg[f][:b], sr[f][:b])
    np.testing.assert_allclose(sg["descriptor"][:b], sr["descriptor"][:b], rtol=0, atol=1e-5)
    m = min(len(sg), len(sr))
    same = (sg["frame_id"][:m] == sr["frame_id"][:m]) & np.all(sg["pixel"][:m] == sr["pixel"][:m], axis=1)
    assert same.mean() > 0.95
    dev = np.linalg.norm(sg["canonical_pos"][:m][same] - sr["canonical_pos"][:m][same], axis=1).max() / voxel
    assert dev <= 1e-3, dev


def test_process_frame_features_frame_without_color(ctx):
    """a frame without color skips the sparse term and add_features (pipeline.cpp:96, 188)"""
    from paper_1603_08161_b200.wfk import pipeline_config
    n = 32
    K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    solver = SolverParams.make(levels=2)
    frames = bend_frames(ctx, K, 4, 1.0)
    frames[2] = Frame(K, frames[2].depth, None)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=solver, reassociations=1)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=solver, reassociations=1)
    pose = Pose.make()
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose
        if i == 2:
            assert rg.match_count == rr.match_count == 0 and rg.features_added == rr.features_added == 0
        else:
            assert rr.features_added > 0 and abs(rg.features_added - rr.features_added) <= 2
    assert abs(len(ctx.feature_store()) - len(ref.feature_store())) <= 4


def test_config2_sequence_parity(ctx):
    """BASELINE configs[1]: 640x480 depth, 64^3 lattice, depth + ARAP + sparse
    feature terms, default solver / correspondence / fusion parameters, ICP on:
    four frames of the bend sequence against the oracle Reconstructor."""
    from paper_1603_08161_b200.wfk import pipeline_config
    n = 64
    K = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    frames = bend_frames(ctx, K, 4, 2.0, frames_total=60)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=SolverParams.make(), reassociations=3)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=3)
    pose = Pose.make()
    sparse = 0
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose
        if i == 0:
            assert rg.fusion.fused == rr.fusion.fused and rg.features_added == rr.features_added
            continue
        assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-6)  # measured 1e-10 .. 1e-14
        assert abs(rg.dense_count - rr.dense_count) <= max(3, 0.002 * rr.dense_count)
        assert abs(rg.sparse_count - rr.sparse_count) <= 2
        np.testing.assert_allclose(rg.pose.vector(), rr.pose.vector(), atol=1e-6)
        sparse += rg.sparse_count
    assert sparse > 0
    ctx.download_volume(vol)
    arr = ref.volume_arrays()
    both = arr["active"].astype(bool) & vol.active.astype(bool)
    assert (vol.active != arr["active"]).sum() <= 16
    dev = np.max(np.linalg.norm(vol.deformed[both] - arr["deformed"][both], axis=1)) / voxel
    assert dev <= 1e-3, dev


def test_config3_short_sequence_parity(ctx):
    """BASELINE configs[2] (the bench workload): 640x480, 128^3, defaults --
    the first three frames against the oracle Reconstructor."""
    from paper_1603_08161_b200.wfk import pipeline_config
    n = 128
    K = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    frames = bend_frames(ctx, K, 3, 2.0, frames_total=300)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=SolverParams.make(), reassociations=3)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=3)
    pose = Pose.make()
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose
        if i == 0:
            assert rg.fusion.fused == rr.fusion.fused and rg.features_added == rr.features_added
            continue
        assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-6)  # measured 1e-10 .. 1e-14
        assert abs(rg.dense_count - rr.dense_count) <= max(3, 0.002 * rr.dense_count)
        assert rg.pcg_iterations == rr.pcg_iterations
    ctx.download_volume(vol)
    arr = ref.volume_arrays()
    both = arr["active"].astype(bool) & vol.active.astype(bool)
    assert (vol.active != arr["active"]).sum() <= 16
    dev = np.max(np.linalg.norm(vol.deformed[both] - arr["deformed"][both], axis=1)) / voxel
    assert dev <= 1e-3, dev


def test_config1_fixed_work_parity(ctx):
    """BASELINE configs[0] as SURVEY.md 8(d) row 1 states it: 320x240, 32^3,
    depth + ARAP only (use_features 0), levels 1, one reassociation, 5 GN x 10
    PCG fixed work (flip_flop_rel_tol 0, pcg_tol 0), 10 frames of the bend."""
    from paper_1603_08161_b200.wfk import pipeline_config
    n = 32
    K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
    voxel = 0.7 / (n - 1)
    origin = (-0.35, -0.35, 0.85)
    solver = SolverParams.make(levels=1, flip_flop_iters=5, flip_flop_rel_tol=0.0, pcg_max_iters=10, pcg_tol=0.0)
    frames = bend_frames(ctx, K, 10, 1.0)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=solver, reassociations=1, use_features=False)
    vol = Volume((n, n, n), voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=solver, reassociations=1, use_features=False)
    pose = Pose.make()
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr)
        rg = ctx.process_frame(fr, pose, cfg, i)
        pose = rg.pose
        if i == 0:
            continue
        assert rg.trace_len == rr.trace_len == 5
        assert rg.pcg_iterations == rr.pcg_iterations == 50  # fixed work
        assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-6)  # measured 1e-10 .. 1e-14
    ctx.download_volume(vol)
    arr = ref.volume_arrays()
    both = arr["active"].astype(bool) & vol.active.astype(bool)
    dev = np.max(np.linalg.norm(vol.deformed[both] - arr["deformed"][both], axis=1)) / voxel
    assert dev <= 1e-3, dev
