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
