"""tools/synthscene (the bench's and the tests' synthetic RGB-D generator)
against the reference's own SyntheticScene::render_frame
(proj/src/synthcam.cpp:252-316, built into oracle/_ref): depth and color
must be identical bit for bit, so both bench arms and every parity test
consume exactly the frames the reference would render.  CPU only."""
import ctypes as C

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Intrinsics
from tools import synthscene as S

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference here)")

K320 = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
K640 = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)


def ref_render(scene, frame):
    l = O.lib("ref")
    depth = np.zeros((scene.height, scene.width), np.float32)
    color = np.zeros((scene.height, scene.width, 3), np.float32)
    l.wfo_ref_render_scene.argtypes = [C.POINTER(S.Scene), C.c_int32, C.c_void_p, C.c_void_p]
    assert l.wfo_ref_render_scene(C.byref(scene), frame, depth.ctypes.data, color.ctypes.data) == 0
    return depth, color


def check(scene, frame):
    d, c = S.render(scene, frame)
    dr, cr = ref_render(scene, frame)
    assert (d > 0).sum() > 1000, "scene should cover the image"
    assert np.array_equal(d.view(np.uint32), dr.view(np.uint32)), f"{int((d != dr).sum())} depth pixels differ"
    assert np.array_equal(c.view(np.uint32), cr.view(np.uint32)), f"{int((c != cr).any(-1).sum())} color pixels differ"


@pytest.mark.parametrize("frame", [0, 37, 150])
def test_bend_sphere_oscillating(frame):  # BASELINE configs[1..2] scene
    check(S.bend_sphere(K320, frames=300, amplitude=2.0, frequency=2.0), frame)


def test_bend_sphere_640():
    check(S.bend_sphere(K640, frames=300, amplitude=2.0, frequency=2.0), 21)


def test_bend_sphere_linear_ramp():
    check(S.bend_sphere(K320, frames=10, amplitude=1.0, frequency=0.0), 6)


@pytest.mark.parametrize("frame,sphere", [(0, 0.0), (17, 0.0), (5, 0.12)])
def test_room_corner_moving_camera(frame, sphere):  # acceptance criterion 4, configs[4]
    check(S.room_corner(K320, sphere_radius=sphere), frame)


def test_bend_cylinder():  # acceptance criteria 5/6
    check(S.bend_cylinder(K320), 30)


def test_sliding_plane():  # acceptance criterion 7
    check(S.sliding_plane(K320), 10)


def test_twist_box_checker_noise_textures():
    s = S.Scene.make(K320, frames=20)
    s.add_shape(S.BOX, center=(0.0, 0.05, 1.3), half_extents=(0.2, 0.15, 0.1))
    s.add_shape(S.SPHERE, center=(0.15, -0.1, 1.1), radius=0.08)
    s.warp_type, s.driver_axis, s.amplitude, s.frequency = S.WARP_TWIST, 1, 1.5, 1.0
    s.pivot[:] = [0.0, 0.0, 1.3]
    s.tex_type = S.CHECKER
    check(s, 4)
    s.tex_type, s.tex_scale = S.NOISE, 0.05
    check(s, 9)


def test_depth_noise():
    s = S.bend_sphere(K320, frames=10, amplitude=0.5, frequency=0.0)
    s.noise_sigma, s.noise_seed = 0.002, 5
    check(s, 3)
