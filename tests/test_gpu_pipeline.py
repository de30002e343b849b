"""End-to-end parity of the per-frame hot path (Reconstructor::process_frame,
pipeline.cpp:143-262, with the global-pose ICP and the feature front-end):
the B200 path (wfk_process_frame) against the checker -- the reference's own
code (oracle/_ref) when built, else the port -- on identical synthetic frames
(tools/synthscene).  Integer outcomes (constraint / match / feature counts,
fused and activated voxels, PCG iteration counts, trace lengths) must be
EQUAL frame by frame; energies agree to 1e-9 relative (measured <= 1e-12) and
the deformation field to 1e-6 voxel (measured ~1e-10), the device's PCG dot
order and libm being the only differences."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import FEATURE_DTYPE, CorrespondParams, Frame, FusionParams, Intrinsics, Pose, SolverParams, Volume

pytestmark = pytest.mark.gpu

INT_FIELDS = ("dense_count", "sparse_count", "match_count", "features_added", "pcg_iterations", "trace_len",
              "anomalies", "icp_degraded")


def assert_records_equal(rg, rr, frame):
    for k in INT_FIELDS:
        assert getattr(rg, k) == getattr(rr, k), (frame, k, getattr(rg, k), getattr(rr, k))
    if rr.icp_iterations >= 0:  # not part of the reference's FrameRecord (the ref build reports -1)
        assert rg.icp_iterations == rr.icp_iterations, frame
    assert (rg.fusion.fused, rg.fusion.skipped_gate, rg.fusion.skipped_frustum, rg.fusion.skipped_occluded) == \
        (rr.fusion.fused, rr.fusion.skipped_gate, rr.fusion.skipped_frustum, rr.fusion.skipped_occluded), frame
    assert (rg.expansion.activated, rg.expansion.orphans) == (rr.expansion.activated, rr.expansion.orphans), frame
    if rr.energy.total != 0:
        assert rg.energy.total == pytest.approx(rr.energy.total, rel=1e-9), frame
    np.testing.assert_allclose(rg.pose.matrix(), rr.pose.matrix(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(rg.pose.vector(), rr.pose.vector(), rtol=0, atol=1e-11)


def assert_volumes_match(vol, arr, voxel):
    assert np.array_equal(vol.active, arr["active"])
    assert np.array_equal(vol.age, arr["age"])
    both = arr["active"].astype(bool)
    if both.any():
        dev = np.max(np.linalg.norm(vol.deformed[both] - arr["deformed"][both], axis=1)) / voxel
        assert dev <= 1e-6, dev


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
        assert_records_equal(rg, rr, i)
    ctx.download_volume(vol)
    assert_volumes_match(vol, ref.volume_arrays(), voxel)


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
        assert_records_equal(rg, rr, i)
        total_sparse += rg.sparse_count
    assert total_sparse > 0, "the sequence should produce sparse feature constraints"
    sg, sr = ctx.feature_store(), ref.feature_store()
    assert len(sg) == len(sr) > 20
    for f in ("pixel", "frame_id"):
        np.testing.assert_array_equal(sg[f], sr[f])
    # the bootstrap frame's positions are exact (identity warp), later ones to the inversion tolerance
    b = int((sr["frame_id"] == 0).sum())
    for f in ("world_pos", "canonical_pos"):
        np.testing.assert_array_equal(sg[f][:b], sr[f][:b])
    np.testing.assert_allclose(sg["descriptor"], sr["descriptor"], rtol=0, atol=1e-5)
    dev = np.linalg.norm(sg["canonical_pos"] - sr["canonical_pos"], axis=1).max() / voxel
    assert dev <= 1e-6, dev
    ctx.download_volume(vol)
    assert_volumes_match(vol, ref.volume_arrays(), voxel)


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
        assert_records_equal(rg, rr, i)
        if i == 2:
            assert rg.match_count == 0 and rg.features_added == 0
        else:
            assert rr.features_added > 0
    assert len(ctx.feature_store()) == len(ref.feature_store())


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
        assert_records_equal(rg, rr, i)
        sparse += rg.sparse_count
    assert sparse > 0
    ctx.download_volume(vol)
    assert_volumes_match(vol, ref.volume_arrays(), voxel)


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
        assert_records_equal(rg, rr, i)
        if i > 0:
            assert rg.trace_len == 5 and rg.pcg_iterations == 50  # fixed work
    ctx.download_volume(vol)
    assert_volumes_match(vol, ref.volume_arrays(), voxel)
