"""Oracle restatement of the feature front-end (features.cpp:12-433):
properties of the DoG pyramid, keypoints and descriptors on the textured
synthetic sphere, and of the mutual-best matching."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import FEATURE_DTYPE, FeatureParams, Frame, Intrinsics

K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)


def textured_frame(center=(0.0, 0.0, 1.2)):
    d, c = O.synth_render(K, center=center)
    return Frame(K, d, c)


def test_pyramid_shapes_and_dog():
    fr = textured_frame()
    g00 = O.pyramid_level(fr, 0, 0)
    g01 = O.pyramid_level(fr, 0, 1)
    d00 = O.pyramid_level(fr, 0, 0, dog=True)
    assert g00.shape == (240, 320)
    np.testing.assert_array_equal(d00, g01 - g00)  # float DoG, exact
    assert O.pyramid_level(fr, 1, 0).shape == (120, 160)
    assert O.pyramid_level(fr, 3, 3).shape == (30, 40)


def test_constant_image_blurs_to_itself():
    d = np.full((240, 320), 1.0, np.float32)
    c = np.full((240, 320, 3), 128.0, np.float32)
    fr = Frame(K, d, c)
    g = O.pyramid_level(fr, 2, 3)
    gray = (np.float32(0.299) * 128 + np.float32(0.587) * 128 + np.float32(0.114) * 128) / np.float32(255)
    assert np.allclose(g, gray, atol=1e-6)
    feats, nk = O.detect_features(fr)
    assert nk == 0 and len(feats) == 0  # flat: no extrema


def test_keypoints_and_descriptors_on_texture():
    fr = textured_frame()
    feats, nk = O.detect_features(fr)
    p = FeatureParams.make()
    assert 20 <= nk <= p.max_keypoints
    assert 0 < len(feats) <= nk
    dsc = feats["descriptor"].astype(np.float64)
    np.testing.assert_allclose(np.linalg.norm(dsc, axis=1), 1.0, atol=1e-6)
    assert dsc.max() <= 0.2 / 0.2 + 1e-6 and dsc.min() >= 0
    # every keypoint lies on valid depth (detect_keypoints' lift condition)
    px = feats["pixel"].astype(int)
    assert np.all(fr.depth[px[:, 1], px[:, 0]] > 0)


def test_matching_a_frame_against_itself():
    fr = textured_frame()
    feats, _ = O.detect_features(fr)
    cur = feats.copy()
    cur["world_pos"] = np.array([0.0, 0.0, 1.0])
    store = feats.copy()
    store["frame_id"] = 0
    pred = np.tile([0.0, 0.0, 1.0], (len(store), 1))
    pred[:, 0] = (store["pixel"][:, 0] - K.cx) / K.fx  # project back to the same pixel at z = 1
    pred[:, 1] = (store["pixel"][:, 1] - K.cy) / K.fy
    cur["world_pos"] = pred
    m = O.match_features(cur, store, pred, K)
    assert len(m) > 0 and np.all(m["distance"] < 1e-12)
    assert len(m) <= FeatureParams.make().keep_best
    assert np.all(m["source_id"] == m["target_id"])


def test_descriptor_distance():
    a = np.zeros(128, np.float32)
    b = np.zeros(128, np.float32)
    a[3], b[3] = 0.5, -0.5
    assert O.descriptor_distance(a, b) == pytest.approx(1.0)


def test_match_pruning_gates():  # test_features.cpp:135-181
    from tests.feature_kats import K as KK, pruning_cases
    for name, store, cur, pred, exp in pruning_cases():
        m = O.match_features(cur, store, pred, KK)
        assert [(int(a), int(b)) for a, b in zip(m["source_id"], m["target_id"])] == exp, name


def test_descriptors_match_across_translation():  # test_features.cpp:103-133
    from tests.feature_kats import K as KK, blob_frame, with_world
    f0, _ = O.detect_features(blob_frame())
    f1, _ = O.detect_features(blob_frame(12, 8))
    assert len(f0) >= 4 and len(f1) >= 4
    st = with_world(f0)
    st["frame_id"] = 0
    cur = with_world(f1)
    m = O.match_features(cur, st, st["world_pos"], KK)
    assert len(m) >= 4
    off = cur["pixel"][m["target_id"]] - st["pixel"][m["source_id"]]
    assert np.all(np.abs(off[:, 0] - 12) < 1.5) and np.all(np.abs(off[:, 1] - 8) < 1.5)
    assert np.all(m["distance"] <= FeatureParams.make().tau_descriptor)


def test_blobs_detected_near_centers():  # test_features.cpp:82-101
    from tests.feature_kats import CENTERS, blob_frame
    fr = blob_frame()
    f, nk = O.detect_features(fr)
    assert nk > 0
    px = f["pixel"]
    # the reference checks its keypoints; these are the features that survive
    # extract_descriptors, so one blob may lose its feature to the descriptor tests
    near = [np.min(np.linalg.norm(px - np.array(c), axis=1)) < 3.0 for c in CENTERS]
    assert sum(near) >= len(CENTERS) - 1
    for p, s in zip(px, f["scale"]):
        assert np.min(np.linalg.norm(np.array(CENTERS) - p, axis=1)) < 4.0 * s + 4.0
    fr.depth[:] = 0  # without valid depth nothing may be detected
    f, nk = O.detect_features(fr)
    assert nk == 0 and len(f) == 0
