"""Synthetic RGB-D inputs for bench.py and the tests (not the product, not the
oracle): ctypes front end of tools/bin/libsynthscene.so (tools/synthscene.cpp),
a restatement of the reference's SyntheticScene that renders bit-identical
frames (tests/test_synthscene.py checks it against the reference build).

Scene presets follow the reference: the BASELINE sphere under the bend warp
(SURVEY.md 8(d)), the acceptance room corner (acceptance.cpp:463-481), the
bend cylinder (acceptance.cpp:507-527) and the sliding textured plane
(acceptance.cpp:616-633)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "bin", "libsynthscene.so")

SPHERE, BOX, PLANE, CYLINDER = 0, 1, 2, 3
CHECKER, NOISE, DOTS = 0, 1, 2
WARP_NONE, WARP_RIGID, WARP_BEND, WARP_TWIST = 0, 1, 2, 3
MAX_SHAPES = 8

D3 = C.c_double * 3


class Shape(C.Structure):
    _fields_ = [("type", C.c_int32), ("reserved_", C.c_int32), ("center", D3), ("radius", C.c_double),
                ("half_extents", D3), ("normal", D3), ("offset", C.c_double), ("axis", D3),
                ("half_height", C.c_double)]


class Scene(C.Structure):
    _fields_ = [("frames", C.c_int32), ("num_shapes", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32), ("height", C.c_int32),
                ("shapes", Shape * MAX_SHAPES),
                ("tex_type", C.c_int32), ("tex_seed", C.c_uint32), ("tex_scale", C.c_double),
                ("dot_radius", C.c_double),
                ("warp_type", C.c_int32), ("driver_axis", C.c_int32), ("rot_axis", C.c_int32),
                ("reserved2_", C.c_int32), ("amplitude", C.c_double), ("frequency", C.c_double),
                ("pivot", D3), ("rotation_axis", D3), ("deg_per_frame", C.c_double), ("trans_per_frame", D3),
                ("cam_rot_axis", D3), ("cam_deg_per_frame", C.c_double), ("cam_trans_per_frame", D3),
                ("t_min", C.c_double), ("t_max", C.c_double), ("noise_sigma", C.c_double),
                ("noise_seed", C.c_uint32), ("reserved3_", C.c_int32)]

    @classmethod
    def make(cls, intr, frames=10) -> "Scene":
        """SceneSpec defaults (synthcam.hpp:62-78) with the given intrinsics."""
        s = cls()
        s.frames = frames
        s.fx, s.fy, s.cx, s.cy = intr.fx, intr.fy, intr.cx, intr.cy
        s.width, s.height = intr.width, intr.height
        s.tex_type, s.tex_seed, s.tex_scale, s.dot_radius = DOTS, 7, 0.06, 0.3
        s.warp_type, s.driver_axis, s.rot_axis = WARP_NONE, 0, 2
        s.rotation_axis[:] = [0, 1, 0]
        s.cam_rot_axis[:] = [0, 1, 0]
        s.t_min, s.t_max = 0.05, 6.0
        s.noise_seed = 1
        return s

    def add_shape(self, type_, center=(0.0, 0.0, 1.2), radius=0.3, half_extents=(0.3, 0.3, 0.3),
                  normal=(0.0, 0.0, -1.0), offset=-1.2, axis=(0.0, 1.0, 0.0), half_height=0.4) -> "Scene":
        """ShapeSpec (synthcam.hpp:15-24), defaults included."""
        if self.num_shapes >= MAX_SHAPES:
            raise ValueError("too many shapes")
        sh = self.shapes[self.num_shapes]
        sh.type = type_
        sh.center[:] = list(center)
        sh.radius = radius
        sh.half_extents[:] = list(half_extents)
        sh.normal[:] = list(normal)
        sh.offset = offset
        sh.axis[:] = list(axis)
        sh.half_height = half_height
        self.num_shapes += 1
        return self


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE, "synthscene"], check=True)
        _lib = C.CDLL(LIB_PATH)
        _lib.ss_render.argtypes = [C.POINTER(Scene), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32]
        _lib.ss_warp_phase.restype = C.c_double
        _lib.ss_warp_phase.argtypes = [C.POINTER(Scene), C.c_int32]
        _lib.ss_inverse_warp.argtypes = [C.POINTER(Scene), C.c_int32, C.c_void_p, C.c_void_p]
    return _lib


def render(scene: Scene, frame: int, threads: int = 0):
    """SyntheticScene::render_frame: (depth HxW float32, color HxWx3 float32)."""
    depth = np.zeros((scene.height, scene.width), np.float32)
    color = np.zeros((scene.height, scene.width, 3), np.float32)
    rc = lib().ss_render(C.byref(scene), int(frame), depth.ctypes.data, color.ctypes.data, int(threads))
    if rc != 0:
        raise ValueError("invalid synthetic scene")
    return depth, color


def inverse_warp(scene: Scene, frame: int, world) -> np.ndarray:
    w = np.ascontiguousarray(world, np.float64).reshape(3).copy()
    out = np.zeros(3)
    lib().ss_inverse_warp(C.byref(scene), int(frame), w.ctypes.data, out.ctypes.data)
    return out


# ---- presets ------------------------------------------------------------------
def bend_sphere(intr, frames=300, amplitude=2.0, frequency=2.0, center=(0.0, 0.0, 1.2), radius=0.3) -> Scene:
    """The BASELINE configs' scene: sphere r 0.3 at z 1.2, Dots
    texture (scale 0.06, seed 7), bend warp driver x / rotation y about the
    sphere center; frequency 0 = linear ramp over the sequence."""
    s = Scene.make(intr, frames)
    s.add_shape(SPHERE, center=center, radius=radius)
    s.warp_type, s.driver_axis, s.rot_axis = WARP_BEND, 0, 1
    s.amplitude, s.frequency = amplitude, frequency
    s.pivot[:] = list(center)
    return s


def room_corner(intr, frames=30, sphere_radius=0.0) -> Scene:
    """Acceptance criterion 4's five-wall room (acceptance.cpp:463-481) with the
    rigidly moving camera; sphere_radius > 0 adds SURVEY.md 8(d) row 5's sphere
    at (0, 0, 1.2) (configs[4])."""
    s = Scene.make(intr, frames)
    for n, off in (((0, 0, -1), -1.45), ((1, 0, 0), -0.26), ((-1, 0, 0), -0.26), ((0, 1, 0), -0.26),
                   ((0, -1, 0), -0.26)):
        s.add_shape(PLANE, normal=n, offset=off)
    if sphere_radius > 0:
        s.add_shape(SPHERE, center=(0.0, 0.0, 1.2), radius=sphere_radius)
    s.cam_deg_per_frame = 0.25
    s.cam_rot_axis[:] = [0.2, 1, 0.1]
    s.cam_trans_per_frame[:] = [0.0015, 0.001, 0.001]
    return s


def bend_cylinder(intr, frames=60) -> Scene:
    """Acceptance criteria 5/6's bend cylinder (acceptance.cpp:507-527)."""
    s = Scene.make(intr, frames)
    s.add_shape(CYLINDER, center=(0.0, 0.0, 1.3), axis=(1.0, 0.0, 0.0), radius=0.1, half_height=0.22)
    s.tex_type, s.tex_scale = DOTS, 0.04
    s.warp_type, s.driver_axis, s.rot_axis, s.amplitude = WARP_BEND, 0, 1, 4.0
    s.pivot[:] = [0.0, 0.0, 1.3]
    return s


def sliding_plane(intr, frames=30) -> Scene:
    """Acceptance criterion 7's textured plane sliding 2 mm/frame (acceptance.cpp:616-633)."""
    s = Scene.make(intr, frames)
    s.add_shape(PLANE, normal=(0.0, 0.0, -1.0), offset=-1.3)
    s.tex_type, s.tex_scale = DOTS, 0.03
    s.warp_type = WARP_RIGID
    s.trans_per_frame[:] = [0.002, 0.0, 0.0]
    return s


def bend_amplitude(scene: Scene, frame: int) -> float:
    """the bend angle rate of a frame: amplitude * warp_phase (synthcam.cpp:138-149)"""
    return scene.amplitude * lib().ss_warp_phase(C.byref(scene), int(frame))

