"""Batched DeformableVolume::invert_warp (volume.cpp:68-126) on the B200
against the oracle restatement: the same damped Gauss-Newton iterates with
-fmad=false on both sides, so success flags match exactly and points to
rounding."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Pose
from tests.test_oracle_invert_warp import field, inner_points

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("rot,t,jit", [((0.0, 0.0, 0.0), (0, 0, 0), 0.0),
                                       ((0.05, -0.03, 0.02), (0.01, -0.02, 0.005), 0.0),
                                       ((0.0, 0.02, 0.0), (0, 0, 0), 0.006)])
def test_invert_warp_parity(ctx, rot, t, jit):
    v = field(rot=rot, t=t, jitter=jit, seed=7)
    x = inner_points(v, k=500, seed=11)
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, -0.02)), (0.002, 0.001, -0.001))
    y = np.array([O.warp_point(v, pose, p) for p in x])
    seed = x + np.random.default_rng(2).uniform(-0.02, 0.02, x.shape)
    seed[:5] = 9.0  # outside the grid: nullopt
    ref, ok_ref = O.invert_warp(v, pose, y, seed)
    ctx.upload_volume(v)
    got, ok = ctx.invert_warp(pose, y, seed)
    assert np.array_equal(ok, ok_ref)
    assert not ok[:5].any() and ok.mean() > 0.9
    np.testing.assert_allclose(got[ok], ref[ok], rtol=0, atol=1e-12)
