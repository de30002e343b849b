"""Feature front-end on the B200 (features.cpp:12-433) against the oracle
restatement on the textured synthetic sphere: the pyramid and DoG images
bit-exact, the keypoint set exact, orientations and descriptors to the
rounding of the device transcendentals."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import FeatureParams, Frame, Intrinsics

pytestmark = pytest.mark.gpu

K320 = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
K640 = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def frame(K, center=(0.0, 0.0, 1.2), amplitude=0.0):
    d, c = O.synth_render(K, center=center, amplitude=amplitude)
    return Frame(K, d, c)


def test_pyramid_bit_exact(ctx):
    fr = frame(K320)
    ctx.upload_frame(fr)
    ctx.detect_features()
    for o, l in [(0, 0), (0, 1), (1, 3), (3, 2)]:
        assert np.array_equal(ctx.feature_pyramid_level(o, l), O.pyramid_level(fr, o, l)), (o, l)
    for o, l in [(0, 0), (0, 1), (2, 2)]:
        assert np.array_equal(ctx.feature_pyramid_level(o, l, dog=True), O.pyramid_level(fr, o, l, dog=True))


@pytest.mark.parametrize("K,center,amp", [(K320, (0.0, 0.0, 1.2), 0.0), (K640, (0.0, 0.0, 1.2), 0.0),
                                          (K640, (0.02, -0.01, 1.25), 1.5)])
def test_features_parity(ctx, K, center, amp):
    fr = frame(K, center, amp)
    ref, nk_ref = O.detect_features(fr)
    ctx.upload_frame(fr)
    got, nk = ctx.detect_features()
    assert nk == nk_ref and len(got) == len(ref) and len(got) > 10
    np.testing.assert_array_equal(got["pixel"], ref["pixel"])
    np.testing.assert_array_equal(got["scale"], ref["scale"])
    np.testing.assert_allclose(got["orientation"], ref["orientation"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(got["descriptor"], ref["descriptor"], rtol=0, atol=1e-5)


def test_features_without_color(ctx):
    d, _ = O.synth_render(K320)
    ctx.upload_frame(Frame(K320, d, None))
    got, nk = ctx.detect_features()
    assert len(got) == 0 and nk == 0


def backprojected(feats, fr, K):
    """world positions of features from the frame depth at the rounded pixel (z <= 0: invalid)"""
    out = feats.copy()
    px = np.rint(feats["pixel"]).astype(int)
    z = fr.depth[np.clip(px[:, 1], 0, K.height - 1), np.clip(px[:, 0], 0, K.width - 1)].astype(np.float64)
    x = (px[:, 0] - K.cx) * z / K.fx
    y = (px[:, 1] - K.cy) * z / K.fy
    out["world_pos"] = np.stack([x, y, np.where(z > 0, z, -1.0)], axis=1)
    return out


def history(K, n_frames, ids):
    """features of a short bend sequence, frame ids from `ids`, stored in that order"""
    st = []
    for f in range(n_frames):
        fr = frame(K, (0.004 * f, 0.0, 1.2), 0.3 * f)
        feats, _ = O.detect_features(fr)
        feats = backprojected(feats, fr, K)
        feats["canonical_pos"] = feats["world_pos"]
        feats["frame_id"] = ids[f]
        st.append(feats)
    return np.concatenate(st)


@pytest.mark.parametrize("ids,tau_px,tau_3d,keep,maxc", [
    ([0, 1, 2, 3], 48.0, 0.10, 64, 128),  # defaults
    ([5, 2, 5, 0], 48.0, 0.10, 64, 128),  # frame ids unsorted and repeated (groups not contiguous)
    ([0, 1, 2, 3], 3.0, 0.004, 64, 128),  # tight reprojection / 3-D prune
    ([0, 1, 2, 3], 48.0, 0.10, 7, 5),     # candidate cap and keep_best below the mutual count
])
def test_match_features_parity(ctx, ids, tau_px, tau_3d, keep, maxc):
    st = history(K320, 4, ids)
    fr = frame(K320, (0.02, 0.0, 1.2), 1.3)
    cur, _ = O.detect_features(fr)
    cur = backprojected(cur, fr, K320)
    pred = st["world_pos"].copy()
    pred[::9, 2] = -1.0  # some history features without a prediction
    p = FeatureParams.make()
    p.tau_pixels, p.tau_3d, p.keep_best, p.max_candidates = tau_px, tau_3d, keep, maxc
    ref = O.match_features(cur, st, pred, K320, p)
    got = ctx.match_features(cur, st, pred, K320, p)
    assert len(ref) >= (3 if keep < 10 else 6)
    np.testing.assert_array_equal(got["source_id"], ref["source_id"])
    np.testing.assert_array_equal(got["target_id"], ref["target_id"])
    np.testing.assert_array_equal(got["distance"], ref["distance"])  # sequential fp64 sum: bit-exact


def test_match_features_empty(ctx):
    st = history(K320, 1, [0])
    assert len(ctx.match_features(st[:0], st, st["world_pos"], K320)) == 0
    assert len(ctx.match_features(st, st[:0], np.zeros((0, 3)), K320)) == 0


def test_feature_store_round_trip(ctx):
    st = history(K320, 2, [0, 1])
    ctx.set_feature_store(st)
    back = ctx.feature_store()
    assert back.tobytes() == st.tobytes()
    ctx.set_feature_store(st[:0])
    assert len(ctx.feature_store()) == 0


def test_match_features_many_groups(ctx):
    """more frame groups than SMs: the matcher's blocks stride over the store"""
    base = history(K320, 2, [0, 1])
    rng = np.random.default_rng(3)
    groups = []
    for g in range(200):
        f = base.copy()
        f["frame_id"] = g
        f["descriptor"] = np.clip(f["descriptor"] + rng.normal(0, 0.01, f["descriptor"].shape), 0, None)
        groups.append(f)
    st = np.concatenate(groups)
    fr = frame(K320, (0.01, 0.0, 1.2), 0.4)
    cur, _ = O.detect_features(fr)
    cur = backprojected(cur, fr, K320)
    pred = st["world_pos"].copy()
    ref = O.match_features(cur, st, pred, K320)
    got = ctx.match_features(cur, st, pred, K320)
    assert len(ref) > 200
    np.testing.assert_array_equal(got["source_id"], ref["source_id"])
    np.testing.assert_array_equal(got["target_id"], ref["target_id"])
    np.testing.assert_array_equal(got["distance"], ref["distance"])


def test_match_features_large_group(ctx):
    """a frame group whose distance tile exceeds shared memory (the global fallback)"""
    st = history(K320, 10, [0] * 10)  # one group of ~10 frames of features
    fr = frame(K640, (0.01, 0.0, 1.2), 0.4)
    cur, _ = O.detect_features(fr)
    cur = backprojected(cur, fr, K640)
    assert len(st) * len(cur) > 16384
    pred = st["world_pos"].copy()
    p = FeatureParams.make()
    p.tau_pixels, p.tau_3d = 1e9, 1e9  # keep every mutual match
    ref = O.match_features(cur, st, pred, K640, p)
    got = ctx.match_features(cur, st, pred, K640, p)
    assert len(ref) > 5
    np.testing.assert_array_equal(got["source_id"], ref["source_id"])
    np.testing.assert_array_equal(got["target_id"], ref["target_id"])
    np.testing.assert_array_equal(got["distance"], ref["distance"])


@pytest.mark.parametrize("kw", [dict(max_keypoints=20), dict(max_orientations=1), dict(dog_levels=4, octaves=3),
                                dict(contrast_threshold=0.03, edge_ratio=5.0)])
def test_features_parity_params(ctx, kw):
    fr = frame(K640, (0.02, -0.01, 1.25), 1.0)
    p = FeatureParams.make(**kw)
    ref, nk_ref = O.detect_features(fr, p)
    ctx.upload_frame(fr)
    got, nk = ctx.detect_features(p)
    assert nk == nk_ref and len(got) == len(ref) and len(got) > 0
    np.testing.assert_array_equal(got["pixel"], ref["pixel"])
    np.testing.assert_array_equal(got["scale"], ref["scale"])
    np.testing.assert_allclose(got["orientation"], ref["orientation"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(got["descriptor"], ref["descriptor"], rtol=0, atol=1e-5)


def test_match_pruning_gates_device(ctx):  # test_features.cpp:135-181
    from tests.feature_kats import K as KK, pruning_cases
    for name, store, cur, pred, exp in pruning_cases():
        m = ctx.match_features(cur, store, pred, KK)
        assert [(int(a), int(b)) for a, b in zip(m["source_id"], m["target_id"])] == exp, name


def test_descriptors_match_across_translation_device(ctx):  # test_features.cpp:103-133
    from tests.feature_kats import K as KK, blob_frame, with_world
    ctx.upload_frame(blob_frame())
    f0, _ = ctx.detect_features()
    ctx.upload_frame(blob_frame(12, 8))
    f1, _ = ctx.detect_features()
    assert len(f0) >= 4 and len(f1) >= 4
    st = with_world(f0)
    st["frame_id"] = 0
    cur = with_world(f1)
    m = ctx.match_features(cur, st, st["world_pos"], KK)
    assert len(m) >= 4
    off = cur["pixel"][m["target_id"]] - st["pixel"][m["source_id"]]
    assert np.all(np.abs(off[:, 0] - 12) < 1.5) and np.all(np.abs(off[:, 1] - 8) < 1.5)


def test_blobs_detected_near_centers_device(ctx):  # test_features.cpp:82-101
    from tests.feature_kats import CENTERS, blob_frame
    fr = blob_frame()
    ctx.upload_frame(fr)
    f, nk = ctx.detect_features()
    assert nk > 0
    near = [np.min(np.linalg.norm(f["pixel"] - np.array(c), axis=1)) < 3.0 for c in CENTERS]
    assert sum(near) >= len(CENTERS) - 1  # features: one blob may fail the descriptor tests
    fr.depth[:] = 0
    ctx.upload_frame(fr)
    f, nk = ctx.detect_features()
    assert nk == 0 and len(f) == 0
