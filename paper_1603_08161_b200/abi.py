"""ctypes images of include/wfk_types.h and the host-side data containers.

These mirror the reference's wf:: value types (proj/include/wf/*.hpp) so that
Python callers hold the same data a C++ caller of the reference would:

* ``Volume``          -- wf::DeformableVolume (volume.hpp:29-112), SoA numpy arrays
* ``CORR_DTYPE``      -- wf::Correspondence   (correspond.hpp:14-23), 184 B records
* ``Pose``            -- wf::GlobalPose       (core.hpp:20-31)
* ``Intrinsics``      -- wf::Intrinsics       (core.hpp:41-58)
* ``SolverParams``    -- wf::SolverParams     (solver.hpp:12-22)
* ``FusionParams``    -- wf::FusionParams     (fusion.hpp:10-15)
* ``CorrespondParams``-- wf::CorrespondenceParams (correspond.hpp:25-29)

Only plain data lives here; no compute.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

WFK_OK = 0
WFK_E_INVALID_ARG = -1
WFK_E_OUT_OF_RANGE = -2
WFK_E_LOGIC = -3
WFK_E_CUDA = -4
WFK_E_NCCL = -5
WFK_E_OOM = -6
WFK_E_CAPACITY = -7

EXEC_SERIAL = 0
EXEC_PARALLEL = 1
DENSE_PLANE = 0
SPARSE_POINT = 1

VOL_TSDF, VOL_WEIGHT, VOL_COLOR, VOL_DEFORMED, VOL_EULER, VOL_AGE, VOL_ACTIVE = (
    1 << i for i in range(7))
VOL_ALL = 0x7F

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint8)


class VolumeView(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("reserved_", C.c_int32),
                ("voxel_size", C.c_double), ("origin", C.c_double * 3),
                ("truncation", C.c_double),
                ("tsdf", _fp), ("weight", _fp), ("color", _fp),
                ("deformed", _dp), ("euler", _dp), ("age", _ip), ("active", _up)]


class Pose(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("translation", C.c_double * 3)]

    @staticmethod
    def make(rotation=None, translation=None) -> "Pose":
        p = Pose()
        r = np.eye(3) if rotation is None else np.asarray(rotation, dtype=np.float64)
        t = np.zeros(3) if translation is None else np.asarray(translation, dtype=np.float64)
        p.rotation[:] = [float(v) for v in r.reshape(9)]
        p.translation[:] = [float(v) for v in t.reshape(3)]
        return p

    def matrix(self) -> np.ndarray:
        return np.array(self.rotation[:], dtype=np.float64).reshape(3, 3)

    def vector(self) -> np.ndarray:
        return np.array(self.translation[:], dtype=np.float64)


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]

    @staticmethod
    def make(fx, fy, cx, cy, width, height) -> "Intrinsics":
        return Intrinsics(float(fx), float(fy), float(cx), float(cy), int(width), int(height))


class SolverParams(C.Structure):
    _fields_ = [("w_d", C.c_double), ("w_s", C.c_double), ("w_r", C.c_double),
                ("flip_flop_iters", C.c_int32), ("pcg_max_iters", C.c_int32),
                ("flip_flop_rel_tol", C.c_double), ("pcg_tol", C.c_double),
                ("levels", C.c_int32), ("exec", C.c_int32)]

    @staticmethod
    def make(**kw) -> "SolverParams":
        # defaults: solver.hpp:12-22
        d = dict(w_d=1.0, w_s=0.5, w_r=5.0, flip_flop_iters=4, pcg_max_iters=50,
                 flip_flop_rel_tol=1e-6, pcg_tol=1e-4, levels=3, exec=EXEC_PARALLEL)
        d.update(kw)
        return SolverParams(**d)


class Energy(C.Structure):
    _fields_ = [("total", C.c_double), ("sparse", C.c_double), ("dense", C.c_double),
                ("reg", C.c_double)]

    def as_dict(self):
        return dict(total=self.total, sparse=self.sparse, dense=self.dense, reg=self.reg)


class TraceEntry(C.Structure):
    _fields_ = [("level", C.c_int32), ("iteration", C.c_int32), ("energy", Energy),
                ("pcg_iterations", C.c_int32), ("anomaly", C.c_int32),
                ("pcg_residual", C.c_double)]


class PcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("reserved_", C.c_int32),
                ("relative_residual", C.c_double)]


class FusionParams(C.Structure):
    _fields_ = [("k_min", C.c_int32), ("bootstrap", C.c_int32), ("w_max", C.c_double),
                ("sample_weight", C.c_double)]

    @staticmethod
    def make(**kw) -> "FusionParams":
        d = dict(k_min=3, bootstrap=0, w_max=64.0, sample_weight=1.0)  # fusion.hpp:10-15
        d.update(kw)
        return FusionParams(**d)


class FusionStats(C.Structure):
    _fields_ = [("fused", C.c_int32), ("skipped_gate", C.c_int32),
                ("skipped_frustum", C.c_int32), ("skipped_occluded", C.c_int32)]

    def as_tuple(self):
        return (self.fused, self.skipped_gate, self.skipped_frustum, self.skipped_occluded)


class ExpansionStats(C.Structure):
    _fields_ = [("activated", C.c_int32), ("orphans", C.c_int32)]


class CorrespondParams(C.Structure):
    _fields_ = [("eps_d", C.c_double), ("eps_n", C.c_double), ("eps_v", C.c_double)]

    @staticmethod
    def make(eps_d=0.05, eps_n=0.5, eps_v=0.8) -> "CorrespondParams":  # correspond.hpp:25-29
        return CorrespondParams(eps_d, eps_n, eps_v)


class FeatureParams(C.Structure):
    """wf::FeatureParams (features.hpp:29-45)."""
    _fields_ = [("octaves", C.c_int32), ("dog_levels", C.c_int32), ("sigma0", C.c_double),
                ("contrast_threshold", C.c_double), ("edge_ratio", C.c_double), ("max_keypoints", C.c_int32),
                ("max_orientations", C.c_int32), ("orientation_peak_ratio", C.c_double),
                ("max_candidates", C.c_int32), ("keep_best", C.c_int32), ("tau_descriptor", C.c_double),
                ("tau_pixels", C.c_double), ("tau_3d", C.c_double)]

    @staticmethod
    def make(**kw) -> "FeatureParams":
        d = dict(octaves=4, dog_levels=3, sigma0=1.6, contrast_threshold=0.01, edge_ratio=10.0, max_keypoints=150,
                 max_orientations=2, orientation_peak_ratio=0.8, max_candidates=128, keep_best=64,
                 tau_descriptor=0.7, tau_pixels=48.0, tau_3d=0.10)
        d.update(kw)
        return FeatureParams(**d)


# wf::Feature (features.hpp:13-22)
FEATURE_DTYPE = np.dtype([("canonical_pos", np.float64, 3), ("world_pos", np.float64, 3), ("pixel", np.float64, 2),
                          ("scale", np.float64), ("orientation", np.float64), ("descriptor", np.float32, 128),
                          ("frame_id", np.int32), ("reserved_", np.int32)])
# wf::FeatureMatch
MATCH_DTYPE = np.dtype([("source_id", np.int32), ("target_id", np.int32), ("distance", np.float64)])


class IcpParams(C.Structure):
    """wf::IcpParams (solver.hpp:121-131)."""
    _fields_ = [("corr", CorrespondParams), ("max_iters", C.c_int32), ("min_correspondences", C.c_int32),
                ("rel_tol", C.c_double), ("min_improvement", C.c_double)]

    @staticmethod
    def make(max_iters=20, rel_tol=1e-6, min_improvement=0.0, min_correspondences=6, corr=None) -> "IcpParams":
        return IcpParams(corr or CorrespondParams.make(), max_iters, min_correspondences, rel_tol, min_improvement)


class IcpResult(C.Structure):
    """wf::IcpResult (solver.hpp:133-139)."""
    _fields_ = [("pose", Pose), ("converged", C.c_int32), ("degraded", C.c_int32), ("rms", C.c_double),
                ("iterations", C.c_int32), ("reserved_", C.c_int32)]


class FrameView(C.Structure):
    _fields_ = [("intrinsics", Intrinsics), ("depth", _fp), ("color", _fp)]


class PointNormalMapView(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("point", _dp), ("normal", _dp),
                ("point_valid", _up), ("normal_valid", _up)]


class GeometryBufferView(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("depth", _fp), ("point", _dp),
                ("normal", _dp), ("canonical", _dp)]


class MeshView(C.Structure):
    _fields_ = [("num_vertices", C.c_int64), ("num_triangles", C.c_int64),
                ("vertices_canonical", _dp), ("vertices_deformed", _dp),
                ("normals_deformed", _dp), ("colors", _fp), ("triangles", _ip)]


# wf::Correspondence, field-for-field (correspond.hpp:14-23)
CORR_DTYPE = np.dtype([
    ("kind", np.int32), ("reserved_", np.int32), ("canonical", np.float64, 3),
    ("anchor_index", np.int32, 8), ("anchor_weight", np.float64, 8),
    ("target", np.float64, 3), ("target_normal", np.float64, 3), ("confidence", np.float64)])
assert CORR_DTYPE.itemsize == 184


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the ABI must be C-contiguous"
    return a.ctypes.data_as(C.POINTER(ctype))


class Volume:
    """Host mirror of wf::DeformableVolume (volume.hpp:29-112, ctor volume.cpp:8-25)."""

    def __init__(self, dims, voxel_size: float, origin):
        dims = tuple(int(d) for d in dims)
        if min(dims) < 2:
            raise ValueError("DeformableVolume: each dim must be >= 2")
        if voxel_size <= 0:
            raise ValueError("DeformableVolume: voxel_size must be > 0")
        self.dims = dims
        self.voxel_size = float(voxel_size)
        self.origin = np.asarray(origin, dtype=np.float64).reshape(3).copy()
        self.truncation = 4.0 * self.voxel_size
        n = dims[0] * dims[1] * dims[2]
        self.tsdf = np.zeros(n, np.float32)
        self.weight = np.zeros(n, np.float32)
        self.color = np.zeros((n, 3), np.float32)
        self.deformed = self.canonical_positions()
        self.euler = np.zeros((n, 3), np.float64)
        self.age = np.zeros(n, np.int32)
        self.active = np.zeros(n, np.uint8)

    @property
    def num_points(self) -> int:
        return self.dims[0] * self.dims[1] * self.dims[2]

    def linear_index(self, x, y, z):
        return x + self.dims[0] * (y + self.dims[1] * z)

    def index3(self, i):
        nx, ny = self.dims[0], self.dims[1]
        i = np.asarray(i)
        return np.stack([i % nx, (i // nx) % ny, i // (nx * ny)], axis=-1)

    def canonical_positions(self) -> np.ndarray:
        idx = self.index3(np.arange(self.num_points))
        return self.origin[None, :] + self.voxel_size * idx.astype(np.float64)

    def canonical_position(self, i) -> np.ndarray:
        return self.origin + self.voxel_size * self.index3(i).astype(np.float64)

    def copy(self) -> "Volume":
        v = Volume.__new__(Volume)
        v.dims, v.voxel_size, v.origin, v.truncation = (
            self.dims, self.voxel_size, self.origin.copy(), self.truncation)
        for f in ("tsdf", "weight", "color", "deformed", "euler", "age", "active"):
            setattr(v, f, getattr(self, f).copy())
        return v

    def view(self) -> VolumeView:
        vv = VolumeView()
        vv.dims[:] = list(self.dims)
        vv.voxel_size = self.voxel_size
        vv.origin[:] = [float(o) for o in self.origin]
        vv.truncation = self.truncation
        vv.tsdf = ptr(self.tsdf, C.c_float)
        vv.weight = ptr(self.weight, C.c_float)
        vv.color = ptr(self.color, C.c_float)
        vv.deformed = ptr(self.deformed, C.c_double)
        vv.euler = ptr(self.euler, C.c_double)
        vv.age = ptr(self.age, C.c_int32)
        vv.active = ptr(self.active, C.c_uint8)
        vv._keep = self  # keep arrays alive while the view is
        return vv


class Frame:
    """Host mirror of wf::Frame (image.hpp:31-35)."""

    def __init__(self, intrinsics: Intrinsics, depth: np.ndarray, color: np.ndarray | None = None):
        self.intrinsics = intrinsics
        self.depth = np.ascontiguousarray(depth, dtype=np.float32).reshape(
            intrinsics.height, intrinsics.width)
        self.color = None if color is None else np.ascontiguousarray(
            color, dtype=np.float32).reshape(intrinsics.height, intrinsics.width, 3)

    def view(self) -> FrameView:
        f = FrameView()
        f.intrinsics = self.intrinsics
        f.depth = ptr(self.depth, C.c_float)
        f.color = ptr(self.color, C.c_float)
        f._keep = self
        return f


def trace_to_list(buf, n):
    return [dict(level=buf[i].level, iteration=buf[i].iteration,
                 energy=buf[i].energy.as_dict(), pcg_iterations=buf[i].pcg_iterations,
                 pcg_residual=buf[i].pcg_residual, anomaly=bool(buf[i].anomaly))
            for i in range(n)]
