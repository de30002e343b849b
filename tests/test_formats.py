"""Snapshot and frame formats: DeformableVolume::save /
load (volume.cpp:150-217), FeatureStore::save / load (features.cpp:306-352),
save/load_depth_pgm and save/load_color_ppm (image.cpp:21-121).

CPU: the oracle restatement against the reference's layout (magic, header and
record sizes, big-endian PGM, header comments) and round trips.
GPU: libwfk's device codecs write the oracle's bytes exactly and read them back.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import FEATURE_DTYPE, Frame, Intrinsics, Volume
from tests.fixtures import active_sphere_volume

K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)


def random_volume(n=(9, 7, 6), seed=3):
    rng = np.random.default_rng(seed)
    v = Volume(n, 0.031, (-0.1, 0.2, 0.9))
    v.truncation = 0.123
    v.tsdf[:] = rng.uniform(-1, 1, v.num_points).astype(np.float32)
    v.weight[:] = rng.uniform(0, 64, v.num_points).astype(np.float32)
    v.color[:] = rng.uniform(0, 255, (v.num_points, 3)).astype(np.float32)
    v.deformed[:] += rng.normal(0, 1e-3, (v.num_points, 3))
    v.euler[:] = rng.normal(0, 0.1, (v.num_points, 3))
    v.age[:] = rng.integers(0, 100, v.num_points)
    v.active[:] = rng.integers(0, 2, v.num_points)
    return v


def same_volume(a, b):
    assert a.dims == b.dims and a.voxel_size == b.voxel_size and a.truncation == b.truncation
    assert np.array_equal(a.origin, b.origin)
    for f in ("tsdf", "weight", "color", "deformed", "euler", "age", "active"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f


def features(n=5):
    rng = np.random.default_rng(1)
    f = np.zeros(n, FEATURE_DTYPE)
    f["canonical_pos"] = rng.normal(size=(n, 3))
    f["world_pos"] = rng.normal(size=(n, 3))
    f["pixel"] = rng.uniform(0, 300, (n, 2))
    f["scale"] = rng.uniform(1, 5, n)
    f["orientation"] = rng.uniform(-3, 3, n)
    f["descriptor"] = rng.uniform(0, 0.2, (n, 128)).astype(np.float32)
    f["frame_id"] = np.arange(n) // 2
    return f


def test_volume_snapshot_layout_and_round_trip():
    v = random_volume()
    img = O.volume_save_bytes(v)
    assert img[:8] == b"WFVOL01\n"
    assert len(img) == 60 + 73 * v.num_points
    assert tuple(np.frombuffer(img[8:20], np.int32)) == v.dims
    assert tuple(np.frombuffer(img[20:60], np.float64)) == (v.voxel_size, *v.origin, v.truncation)
    rec = img[60:60 + 73]  # first record: tsdf, weight, color, deformed, euler, age, active
    assert np.frombuffer(rec[0:4], np.float32)[0] == v.tsdf[0]
    assert np.array_equal(np.frombuffer(rec[20:44], np.float64), v.deformed[0])
    assert rec[72] == v.active[0]
    same_volume(O.volume_load_bytes(img), v)


def test_feature_store_layout():
    f = features()
    img = O.feature_store_bytes(f)
    assert img[:8] == b"WFFEAT1\n" and np.frombuffer(img[8:12], np.int32)[0] == len(f)
    assert len(img) == 12 + len(f) * (80 + 512 + 4)
    r1 = img[12 + 596:12 + 2 * 596]
    assert np.array_equal(np.frombuffer(r1[:80], np.float64)[6:8], f["pixel"][1])
    assert np.frombuffer(r1[592:596], np.int32)[0] == f["frame_id"][1]


def test_pgm_ppm_kats_and_round_trip():
    d = np.array([[0.0, 1.2345, 65.6], [-1.0, 0.0005, 2.0]], np.float32)  # clamps and rounding
    img = O.pgm_encode(d)
    assert img.startswith(b"P5\n3 2\n65535\n")
    raster = np.frombuffer(img[len(b"P5\n3 2\n65535\n"):], ">u2").reshape(2, 3)
    assert raster.tolist() == [[0, 1235, 65535], [0, 1, 2000]]
    back = O.pnm_decode(img, 1)
    assert np.array_equal(back, raster.astype(np.float32) / np.float32(1000))
    c = np.array([[[0.4, 254.6, 300.0], [-3.0, 127.5, 12.0]]], np.float32)
    img = O.ppm_encode(c)
    assert img.startswith(b"P6\n2 1\n255\n")
    assert list(img[len(b"P6\n2 1\n255\n"):]) == [0, 255, 255, 0, 128, 12]
    # header comments and arbitrary whitespace (read_pnm_header, image.cpp:21-50)
    commented = b"P5 # depth\n# a comment line\n3\t2\n65535\n" + img[:0] + raster.astype(">u2").tobytes()
    assert np.array_equal(O.pnm_decode(commented, 1), back)


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


@pytest.mark.gpu
def test_device_volume_snapshot(ctx, tmp_path):
    v = random_volume((33, 17, 9))  # 5,049 points: a partial last block
    ctx.upload_volume(v)
    path = str(tmp_path / "v.wfvol")
    ctx.save_volume(path)
    img = open(path, "rb").read()
    assert img == O.volume_save_bytes(v)
    assert ctx.pack_volume() == img
    ctx.upload_volume(active_sphere_volume(8, 0.05))  # different lattice in between
    ctx.load_volume(path)
    back = Volume(v.dims, v.voxel_size, v.origin)
    ctx.download_volume(back)
    back.truncation = O.volume_load_bytes(ctx.pack_volume()).truncation
    same_volume(back, v)
    bad = bytearray(img)
    bad[3] = ord("X")
    with pytest.raises(Exception):
        ctx.unpack_volume(bytes(bad))
    with pytest.raises(Exception):
        ctx.unpack_volume(img[:-1])


@pytest.mark.gpu
def test_device_feature_store_files(ctx, tmp_path):
    f = features(7)
    ctx.set_feature_store(f)
    path = str(tmp_path / "f.wffeat")
    ctx.save_feature_store(path)
    assert open(path, "rb").read() == O.feature_store_bytes(f)
    ctx.set_feature_store(f[:0])
    ctx.load_feature_store(path)
    assert ctx.feature_store().tobytes() == f.tobytes()


@pytest.mark.gpu
def test_device_pnm(ctx, tmp_path):
    d, c = O.synth_render(K, amplitude=0.7)
    d = d.copy()
    d[5, 7] = 70.0   # clamps to 65535
    d[6, 8] = -2.0   # clamps to 0
    ctx.upload_frame(Frame(K, d, c))
    dp, cp = str(tmp_path / "d.pgm"), str(tmp_path / "c.ppm")
    ctx.save_frame_pnm(dp, cp)
    assert open(dp, "rb").read() == O.pgm_encode(d)
    assert open(cp, "rb").read() == O.ppm_encode(c)
    # the reference's own header variants decode the same
    raw = open(dp, "rb").read()
    alt = str(tmp_path / "alt.pgm")
    with open(alt, "wb") as fh:
        fh.write(b"P5\n# written elsewhere\n320 240\n65535\n" + raw[len(b"P5\n320 240\n65535\n"):])
    ctx.load_frame_pnm(alt, cp, K)
    gd, gc = ctx.download_frame(320, 240)
    assert np.array_equal(gd, O.pnm_decode(raw, 1))
    assert np.array_equal(gc, O.pnm_decode(open(cp, "rb").read(), 3))
    with pytest.raises(Exception):
        ctx.load_frame_pnm(dp, None, Intrinsics.make(280, 280, 159.5, 119.5, 640, 480))  # size mismatch
