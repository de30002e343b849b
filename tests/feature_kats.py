"""Shared fixtures restating test_features.cpp:103-181 (translation matching and
the pruning gates of match_frame_pair) for the oracle and the device tests."""
import numpy as np

from paper_1603_08161_b200.abi import FEATURE_DTYPE, FeatureParams, Frame, Intrinsics

K = Intrinsics.make(280.0, 280.0, 159.5, 119.5, 320, 240)
CENTERS = [(61.3, 52.8), (171.2, 48.1), (243.7, 101.5), (94.6, 140.2), (201.9, 176.4), (140.5, 93.7)]


def backproject(x, y, z):
    return np.array([(x - K.cx) * z / K.fx, (y - K.cy) * z / K.fy, z])


def blob_frame(shift_x=0.0, shift_y=0.0, z=1.3, sigma=3.0):
    """blob_image (test_features.cpp:8-22) as an RGB frame with r = g = b, depth z"""
    ys, xs = np.mgrid[0:240, 0:320].astype(np.float64)
    v = np.full((240, 320), 0.05)
    for cx, cy in CENTERS:
        v += 0.8 * np.exp(-((xs - (cx + shift_x)) ** 2 + (ys - (cy + shift_y)) ** 2) / (2 * sigma * sigma))
    g = np.minimum(v, 1.0).astype(np.float32)
    color = np.repeat((g * np.float32(255.0))[:, :, None], 3, axis=2).astype(np.float32)
    return Frame(K, np.full((240, 320), z, np.float32), color)


def with_world(feats, z=1.3):
    f = feats.copy()
    f["world_pos"] = np.stack([backproject(p[0], p[1], z) for p in f["pixel"]]) if len(f) else f["world_pos"]
    return f


def make_feature(desc, pixel, world, frame_id):
    f = np.zeros(1, FEATURE_DTYPE)
    f["descriptor"][0] = desc
    f["pixel"][0] = pixel
    f["world_pos"][0] = world
    f["canonical_pos"][0] = world
    f["frame_id"][0] = frame_id
    return f


def basis(i, v=1.0):
    d = np.zeros(128, np.float32)
    d[i] = v
    return d


def pruning_cases():
    """(name, store, current, predicted, expected [(source, target)]) per SUBCASE"""
    p = FeatureParams.make()
    w0 = backproject(100, 100, 1.3)
    store = np.concatenate([make_feature(basis(0), (100, 100), w0, 0),
                            make_feature(basis(1), (150, 100), backproject(150, 100, 1.3), 0)])
    pred = np.stack([w0, store["world_pos"][1]])
    far = np.zeros(128, np.float32)
    far[0] = np.float32(1.0 + p.tau_descriptor + 0.01)
    cases = [
        ("clean mutual best pair survives",
         make_feature(basis(0), (102, 101), backproject(102, 101, 1.3), 1), [(0, 0)]),
        ("descriptor distance beyond tau is rejected", make_feature(far, (100, 100), w0, 1), []),
        ("predicted reprojection too far in pixels is rejected",
         make_feature(basis(0), (100 + p.tau_pixels + 5, 100), w0, 1), []),
        ("3d displacement beyond tau is rejected",
         make_feature(basis(0), (100, 100), w0 + np.array([0, 0, p.tau_3d + 0.02]), 1), []),
        ("a history feature claimed better by another is not mutual best",
         np.concatenate([make_feature(basis(0, 0.5), (100, 100), w0, 1),
                         make_feature(basis(0, 0.9), (101, 100), w0, 1)]), [(0, 1)]),
    ]
    return [(name, store, cur, pred, exp) for name, cur, exp in cases]
