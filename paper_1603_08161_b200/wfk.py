"""ctypes front end of libwfk.so (include/wfk.h) -- the B200 path.

``Context`` owns one device (its CUDA stream, the device-resident lattice and
work buffers).  Its methods are one-to-one with the C ABI; the reference's
stateless ``wf::`` functions are layered on top in C++ by
integration/wf_b200_adapter.cpp.

There is no CPU fallback: if libwfk.so is missing or no B200 is visible the
constructor raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .abi import (CORR_DTYPE, FEATURE_DTYPE, MATCH_DTYPE, FeatureParams, CorrespondParams, Energy, ExpansionStats, FrameView, FusionParams,
                  FusionStats, GeometryBufferView, IcpParams, IcpResult, Intrinsics, MeshView, PcgResult,
                  PointNormalMapView, Pose, SolverParams, TraceEntry, Volume, VolumeView, ptr,
                  trace_to_list, VOL_ALL, WFK_OK)

HERE = os.path.dirname(os.path.abspath(__file__))
# WFK_LIBRARY: an alternate build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("WFK_LIBRARY") or os.path.join(HERE, "_lib", "libwfk.so")
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int = 4) -> str:
    """Compile libwfk.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", f"-j{jobs}", "-C", CSRC], check=True)
    return LIB_PATH


class WfkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libwfk error {code}: {msg}")
        self.code = code


class PipelineConfig(C.Structure):
    _fields_ = [("solver", SolverParams), ("correspond", CorrespondParams), ("fusion", FusionParams),
                ("reassociations", C.c_int32), ("estimate_pose", C.c_int32), ("icp", IcpParams),
                ("use_features", C.c_int32), ("reserved_", C.c_int32), ("features", FeatureParams)]


class FrameRecord(C.Structure):
    _fields_ = [("energy", Energy), ("dense_count", C.c_int32), ("sparse_count", C.c_int32),
                ("anomalies", C.c_int32), ("trace_len", C.c_int32), ("pcg_iterations", C.c_int32),
                ("bootstrap", C.c_int32), ("fusion", FusionStats), ("expansion", ExpansionStats),
                ("pose", Pose), ("icp_degraded", C.c_int32), ("icp_iterations", C.c_int32),
                ("icp_rms", C.c_double), ("match_count", C.c_int32), ("features_added", C.c_int32)]


class NeHost(C.Structure):
    _fields_ = [("rows", C.c_void_p), ("node_row", C.c_void_p), ("blocks", C.c_void_p),
                ("cols", C.c_void_p), ("rhs", C.c_void_p), ("frozen", C.c_void_p)]


class Profile(C.Structure):
    _fields_ = [("flip_flop_launches", C.c_int64), ("pcg_iterations", C.c_int64), ("flip_flop_ms", C.c_double),
                ("flip_flop_bytes", C.c_double), ("flip_flop_bytes_impl", C.c_double),
                ("stage_ms", C.c_double * 8), ("launches", C.c_int64)]

    STAGES = ("maps_mesh_raster", "associate", "solve", "redeform", "fuse", "frame")

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "stage_ms"}
        d["stage_ms"] = {k: self.stage_ms[i] for i, k in enumerate(self.STAGES)}
        return d


class Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("precision", C.c_int32), ("reserved_", C.c_int32 * 6)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libwfk.so not built ({LIB_PATH}); run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        _lib.wfk_last_error.restype = C.c_char_p
        _lib.wfk_last_error.argtypes = [C.c_void_p]
        _lib.wfk_launch_count.restype = C.c_int64
        _lib.wfk_launch_count.argtypes = [C.c_void_p]
        _lib.wfk_pcg_iteration_count.restype = C.c_int64
        _lib.wfk_pcg_iteration_count.argtypes = [C.c_void_p]
        _lib.wfk_destroy.argtypes = [C.c_void_p]
        _lib.wfk_host_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
        _lib.wfk_host_free.argtypes = [C.c_void_p]
        _lib.wfk_host_free.restype = None
    return _lib


def _cptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def dist_unique_id() -> bytes:
    """An NCCL unique id for wfk_dist_init (rank 0 creates it and shares it)."""
    buf = (C.c_uint8 * 128)()
    rc = lib().wfk_dist_unique_id(buf)
    if rc != WFK_OK:
        raise WfkError(rc, "wfk_dist_unique_id failed (NCCL unavailable?)")
    return bytes(buf)


def dist_plan(cols, world: int):
    """The z-slab partition of a system's rows (host only, no GPU): ranges
    (world x 2: lo, hi) and the halo transfers (n x 4: src, dst, row_lo, row_hi)."""
    cols = np.ascontiguousarray(cols, np.int32).reshape(-1, 27)
    ranges = np.zeros((world, 2), np.int32)
    n = C.c_int32()
    rc = lib().wfk_dist_plan(C.c_int32(len(cols)), _cptr(cols), C.c_int32(world), _cptr(ranges), None, 0,
                             C.byref(n))
    if rc != WFK_OK:
        raise WfkError(rc, "wfk_dist_plan failed")
    xf = np.zeros((max(n.value, 1), 4), np.int32)
    rc = lib().wfk_dist_plan(C.c_int32(len(cols)), _cptr(cols), C.c_int32(world), _cptr(ranges), _cptr(xf),
                             C.c_int32(len(xf)), C.byref(n))
    if rc != WFK_OK:
        raise WfkError(rc, "wfk_dist_plan failed")
    return ranges, xf[: n.value]


def slab_plan(row_work, blocks: int, block_threads: int, ranks: int):
    """The in-kernel slab partition's host plan (wfk_slab_plan, no GPU): the
    tile row bounds (n_tiles + 1) and the rank tile bounds (ranks + 1)."""
    w = np.ascontiguousarray(row_work, np.int32)
    nt = C.c_int32()
    tr = np.zeros(8 * blocks + 1, np.int32)
    rt = np.zeros(ranks + 1, np.int32)
    rc = lib().wfk_slab_plan(C.c_int32(len(w)), _cptr(w), C.c_int32(blocks), C.c_int32(block_threads),
                             C.c_int32(ranks), C.byref(nt), _cptr(tr), _cptr(rt))
    if rc != WFK_OK:
        raise WfkError(rc, "wfk_slab_plan failed")
    return tr[: nt.value + 1], rt


class _Pinned:
    def __init__(self, nbytes):
        p = C.c_void_p()
        rc = lib().wfk_host_alloc(C.c_size_t(nbytes), C.byref(p))
        if rc != WFK_OK:
            raise WfkError(rc, "wfk_host_alloc failed")
        self.p = p

    def __del__(self):
        if getattr(self, "p", None):
            lib().wfk_host_free(self.p)
            self.p = None


def pinned_array(shape, dtype) -> np.ndarray:
    """numpy array over page-locked host memory (wfk_host_alloc)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    buf = _Pinned(n)
    raw = (C.c_uint8 * n).from_address(buf.p.value)
    arr = np.frombuffer(raw, dtype=dtype).reshape(shape)
    arr.setflags(write=True)
    _PINNED_KEEP.append(buf)  # lifetime tied to the process (bench buffers)
    return arr


_PINNED_KEEP = []


class Context:
    """One libwfk context on one CUDA device (wfk_create / wfk_destroy)."""

    def __init__(self, device: int = 0, precision: int = 0):
        cfg = Config()
        cfg.device = device
        cfg.precision = precision
        h = C.c_void_p()
        rc = lib().wfk_create(C.byref(cfg), C.byref(h))
        if rc != WFK_OK:
            raise WfkError(rc, "wfk_create failed (no B200 / CUDA device visible?)")
        self.h = h
        self.dims = None

    def set_precision(self, precision: int):
        """WFK_PRECISION_FP64 (0, default) or WFK_PRECISION_FAST (1)"""
        self._check(lib().wfk_set_precision(self.h, C.c_int32(precision)))

    def close(self):
        if getattr(self, "h", None):
            lib().wfk_destroy(self.h)
            self.h = None

    __del__ = close

    def _check(self, rc):
        if rc != WFK_OK:
            raise WfkError(rc, lib().wfk_last_error(self.h).decode())

    @property
    def launch_count(self) -> int:
        return int(lib().wfk_launch_count(self.h))

    @property
    def pcg_iteration_count(self) -> int:
        return int(lib().wfk_pcg_iteration_count(self.h))

    # ---- volume ------------------------------------------------------------
    def upload_volume(self, vol: Volume, fields: int = VOL_ALL):
        vv = vol.view()
        self._check(lib().wfk_volume_upload(self.h, C.byref(vv), C.c_uint32(fields)))
        self.dims = vol.dims

    def download_volume(self, vol: Volume, fields: int = VOL_ALL):
        vv = vol.view()
        self._check(lib().wfk_volume_download(self.h, C.byref(vv), C.c_uint32(fields)))

    def create_volume(self, dims, voxel: float, origin):
        """DeformableVolume(dims, voxel, origin) constructed on the device"""
        d = (C.c_int32 * 3)(*dims)
        o = (C.c_double * 3)(*origin)
        self._check(lib().wfk_volume_create(self.h, d, C.c_double(voxel), o))

    def checkpoint_volume(self, restore: bool = False):
        """device-side save / restore of deformed, euler, age and active"""
        self._check(lib().wfk_volume_checkpoint(self.h, C.c_int32(1 if restore else 0)))

    # ---- snapshot / frame formats -----------------------
    def save_volume(self, path: str):
        """DeformableVolume::save (volume.cpp:150-178) of the device lattice."""
        self._check(lib().wfk_volume_save(self.h, os.fsencode(path)))

    def load_volume(self, path: str):
        """DeformableVolume::load (volume.cpp:180-217) into the device lattice."""
        self._check(lib().wfk_volume_load(self.h, os.fsencode(path)))
        self.dims = self.volume_dims()

    def volume_dims(self):
        img = self.pack_volume(header_only=True)
        return tuple(int(d) for d in np.frombuffer(img[8:20], np.int32))

    def pack_volume(self, header_only: bool = False) -> bytes:
        n = C.c_int64()
        self._check(lib().wfk_volume_pack(self.h, None, C.c_int64(0), C.byref(n)))
        out = np.zeros(n.value, np.uint8)
        self._check(lib().wfk_volume_pack(self.h, _cptr(out), C.c_int64(n.value), C.byref(n)))
        return out[:60].tobytes() if header_only else out.tobytes()

    def unpack_volume(self, image: bytes):
        buf = np.frombuffer(image, np.uint8)
        self._check(lib().wfk_volume_unpack(self.h, _cptr(buf), C.c_int64(len(buf))))
        self.dims = self.volume_dims()

    def save_feature_store(self, path: str):
        self._check(lib().wfk_feature_store_save(self.h, os.fsencode(path)))

    def load_feature_store(self, path: str):
        self._check(lib().wfk_feature_store_load(self.h, os.fsencode(path)))

    def load_frame_pnm(self, depth_pgm: str, color_ppm, intr):
        self._check(lib().wfk_frame_load_pnm(self.h, os.fsencode(depth_pgm),
                                             None if color_ppm is None else os.fsencode(color_ppm), C.byref(intr)))

    def save_frame_pnm(self, depth_pgm, color_ppm):
        self._check(lib().wfk_frame_save_pnm(self.h, None if depth_pgm is None else os.fsencode(depth_pgm),
                                             None if color_ppm is None else os.fsencode(color_ppm)))

    def download_frame(self, width: int, height: int, color: bool = True):
        d = np.zeros((height, width), np.float32)
        c = np.zeros((height, width, 3), np.float32) if color else None
        self._check(lib().wfk_frame_download(self.h, _cptr(d), _cptr(c)))
        return d, c

    # ---- solver ------------------------------------------------------------
    def compute_active_set(self, want_list: bool = True):
        n = C.c_int64()
        if not want_list:
            self._check(lib().wfk_compute_active_set(self.h, None, C.c_int64(0), C.byref(n)))
            return n.value
        cap = int(np.prod(self.dims))
        out = np.zeros(cap, np.int32)
        self._check(lib().wfk_compute_active_set(self.h, _cptr(out), C.c_int64(cap), C.byref(n)))
        return out[: n.value].copy()

    def upload_constraints(self, cons):
        cons = np.ascontiguousarray(cons if cons is not None else np.zeros(0, CORR_DTYPE), dtype=CORR_DTYPE)
        self._check(lib().wfk_constraints_upload(self.h, _cptr(cons), C.c_int64(len(cons))))

    def append_constraints(self, cons, drop_inactive=True) -> int:
        cons = np.ascontiguousarray(cons, dtype=CORR_DTYPE)
        kept = C.c_int64()
        self._check(lib().wfk_constraints_append(self.h, _cptr(cons), C.c_int64(len(cons)),
                                                 C.c_int32(1 if drop_inactive else 0), C.byref(kept)))
        return kept.value

    def download_constraints(self):
        n = C.c_int64()
        self._check(lib().wfk_constraints_download(self.h, None, C.c_int64(0), C.byref(n)))
        out = np.zeros(max(n.value, 1), CORR_DTYPE)
        self._check(lib().wfk_constraints_download(self.h, _cptr(out), C.c_int64(len(out)), C.byref(n)))
        return out[: n.value].copy()

    def evaluate_energy(self, pose: Pose, params: SolverParams) -> dict:
        e = Energy()
        self._check(lib().wfk_evaluate_energy(self.h, C.byref(pose), C.byref(params), C.byref(e)))
        return e.as_dict()

    def update_rotations(self):
        self._check(lib().wfk_update_rotations(self.h, C.c_int32(1)))

    def _trace(self, fn, *args, cap=4096):
        buf = (TraceEntry * cap)()
        n = C.c_int32()
        self._check(fn(self.h, *args, buf, C.c_int32(cap), C.byref(n)))
        return trace_to_list(buf, n.value)

    def flip_flop_solve(self, pose: Pose, params: SolverParams, level: int = 0):
        return self._trace(lib().wfk_flip_flop_solve, C.byref(pose), C.byref(params), C.c_int32(level))

    def solve_coarse_to_fine(self, pose: Pose, params: SolverParams):
        return self._trace(lib().wfk_solve_coarse_to_fine, C.byref(pose), C.byref(params))

    def solve_coarse_to_fine_dist(self, pose: Pose, params: SolverParams):
        """solve_coarse_to_fine with each level's PCG on this rank's z-slab (wfk_dist_init first)."""
        return self._trace(lib().wfk_solve_coarse_to_fine_dist, C.byref(pose), C.byref(params))

    def solve_coarse_to_fine_slabs(self, slabs: int, pose: Pose, params: SolverParams):
        """The same partitioned solve with `slabs` slab states on this GPU."""
        return self._trace(lib().wfk_solve_coarse_to_fine_slabs, C.c_int32(slabs), C.byref(pose), C.byref(params))

    def hierarchy_info(self, levels: int):
        dims = np.zeros((levels, 3), np.int32)
        act = np.zeros(levels, np.int64)
        self._check(lib().wfk_hierarchy_info(self.h, C.c_int32(levels), _cptr(dims), _cptr(act)))
        return dims, act

    def build_normal_equations(self, pose: Pose, params: SolverParams) -> dict:
        rows = C.c_int32()
        self._check(lib().wfk_build_normal_equations(self.h, C.byref(pose), C.byref(params), None,
                                                     C.byref(rows)))
        n = rows.value
        npts = int(np.prod(self.dims))
        out = dict(rows=np.zeros(n, np.int32), node_row=np.zeros(npts, np.int32),
                   blocks=np.zeros((n, 27, 3, 3)), cols=np.zeros((n, 27), np.int32),
                   rhs=np.zeros((n, 3)), frozen=np.zeros(n, np.uint8))
        ne = NeHost(*(_cptr(out[k]) for k in ("rows", "node_row", "blocks", "cols", "rhs", "frozen")))
        self._check(lib().wfk_build_normal_equations(self.h, C.byref(pose), C.byref(params), C.byref(ne),
                                                     C.byref(rows)))
        return out

    def pcg_solve(self, blocks, cols, rhs, x, tol, max_iters):
        blocks = np.ascontiguousarray(blocks, np.float64)
        cols = np.ascontiguousarray(cols, np.int32)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.ascontiguousarray(x, np.float64).copy()
        res = PcgResult()
        self._check(lib().wfk_pcg_solve(self.h, C.c_int32(len(cols)), _cptr(blocks), _cptr(cols), _cptr(rhs),
                                        _cptr(x), C.c_double(tol), C.c_int32(max_iters), C.c_int32(1),
                                        C.byref(res)))
        return x, res.iterations, res.relative_residual

    # ---- slab-partitioned PCG ----------------------------------
    def dist_init(self, rank: int, world: int, nccl_id: bytes | None = None):
        """Join the NCCL communicator of a partitioned solve (world 1: no id needed)."""
        buf = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        self._check(lib().wfk_dist_init(self.h, C.c_int32(rank), C.c_int32(world), buf))

    def pcg_solve_dist(self, blocks, cols, rhs, x, tol, max_iters):
        """pcg_solve with this rank's z-slab of the rows; returns the full x."""
        blocks = np.ascontiguousarray(blocks, np.float64)
        cols = np.ascontiguousarray(cols, np.int32)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.ascontiguousarray(x, np.float64).copy()
        res = PcgResult()
        self._check(lib().wfk_pcg_solve_dist(self.h, C.c_int32(len(cols)), _cptr(blocks), _cptr(cols), _cptr(rhs),
                                             _cptr(x), C.c_double(tol), C.c_int32(max_iters), C.byref(res)))
        return x, res.iterations, res.relative_residual

    def pcg_solve_slabs(self, slabs, blocks, cols, rhs, x, tol, max_iters):
        """The same partition run on this GPU as `slabs` slab states (halo copies on the device)."""
        blocks = np.ascontiguousarray(blocks, np.float64)
        cols = np.ascontiguousarray(cols, np.int32)
        rhs = np.ascontiguousarray(rhs, np.float64)
        x = np.ascontiguousarray(x, np.float64).copy()
        res = PcgResult()
        self._check(lib().wfk_pcg_solve_slabs(self.h, C.c_int32(slabs), C.c_int32(len(cols)), _cptr(blocks),
                                              _cptr(cols), _cptr(rhs), _cptr(x), C.c_double(tol),
                                              C.c_int32(max_iters), C.byref(res)))
        return x, res.iterations, res.relative_residual

    def ne_multiply(self, blocks, cols, x):
        blocks = np.ascontiguousarray(blocks, np.float64)
        cols = np.ascontiguousarray(cols, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._check(lib().wfk_ne_multiply(self.h, C.c_int32(len(cols)), _cptr(blocks), _cptr(cols), _cptr(x),
                                          _cptr(y)))
        return y

    # ---- fusion ------------------------------------------------------------
    def upload_frame(self, frame):
        fv = frame.view()
        self._check(lib().wfk_frame_upload(self.h, C.byref(fv)))
        self._frame_wh = (frame.intrinsics.width, frame.intrinsics.height)

    def integrate_frame(self, pose: Pose, params: FusionParams) -> FusionStats:
        s = FusionStats()
        self._check(lib().wfk_integrate_frame(self.h, C.byref(pose), C.byref(params), C.c_int32(1), C.byref(s)))
        return s

    def expand_grid(self) -> ExpansionStats:
        s = ExpansionStats()
        self._check(lib().wfk_expand_grid(self.h, C.byref(s)))
        return s

    def advance_ages(self, idx):
        idx = np.ascontiguousarray(idx, np.int32)
        self._check(lib().wfk_advance_ages(self.h, _cptr(idx), C.c_int64(idx.size)))

    def advance_active_ages(self):
        self._check(lib().wfk_advance_active_ages(self.h))

    # ---- association -------------------------------------------------------
    def backproject_depth(self, download: bool = True):
        from types import SimpleNamespace
        if not download:
            self._check(lib().wfk_backproject_depth(self.h, C.c_int32(1), None))
            return None
        # sizes come from the uploaded frame; caller passes dims via last upload
        w, h = self._frame_wh
        m = SimpleNamespace(width=w, height=h, point=np.zeros((w * h, 3)), normal=np.zeros((w * h, 3)),
                            point_valid=np.zeros(w * h, np.uint8), normal_valid=np.zeros(w * h, np.uint8))
        v = PointNormalMapView(w, h, ptr(m.point, C.c_double), ptr(m.normal, C.c_double),
                               ptr(m.point_valid, C.c_uint8), ptr(m.normal_valid, C.c_uint8))
        self._check(lib().wfk_backproject_depth(self.h, C.c_int32(1), C.byref(v)))
        return m

    def extract_mesh(self, pose: Pose):
        nv, nt = C.c_int64(), C.c_int64()
        self._check(lib().wfk_extract_mesh(self.h, C.byref(pose), C.byref(nv), C.byref(nt)))
        return nv.value, nt.value

    def mesh_warp(self, pose: Pose):
        self._check(lib().wfk_mesh_warp(self.h, C.byref(pose)))

    def compute_normals(self):
        self._check(lib().wfk_compute_normals(self.h))

    def download_mesh(self):
        from types import SimpleNamespace
        mv = MeshView()
        self._check(lib().wfk_mesh_download(self.h, C.byref(mv)))
        V, T = mv.num_vertices, mv.num_triangles
        m = SimpleNamespace(vertices_canonical=np.zeros((V, 3)), vertices_deformed=np.zeros((V, 3)),
                            normals_deformed=np.zeros((V, 3)), colors=np.zeros((V, 3), np.float32),
                            triangles=np.zeros((T, 3), np.int32))
        mv = MeshView(V, T, ptr(m.vertices_canonical, C.c_double), ptr(m.vertices_deformed, C.c_double),
                      ptr(m.normals_deformed, C.c_double), ptr(m.colors, C.c_float), ptr(m.triangles, C.c_int32))
        self._check(lib().wfk_mesh_download(self.h, C.byref(mv)))
        return m

    def upload_mesh(self, m):
        def a(x, dt):
            return None if x is None else np.ascontiguousarray(x, dt)
        can, de = a(m.vertices_canonical, np.float64), a(m.vertices_deformed, np.float64)
        nr = a(getattr(m, "normals_deformed", None), np.float64)
        col, tri = a(m.colors, np.float32), a(m.triangles, np.int32)
        mv = MeshView(len(can), len(tri), ptr(can, C.c_double), ptr(de, C.c_double), ptr(nr, C.c_double),
                      ptr(col, C.c_float), ptr(tri, C.c_int32))
        self._check(lib().wfk_mesh_upload(self.h, C.byref(mv)))

    def rasterize(self, intr: Intrinsics, download: bool = True):
        from types import SimpleNamespace
        if not download:
            self._check(lib().wfk_rasterize(self.h, C.byref(intr), C.c_int32(1), None))
            return None
        w, h = intr.width, intr.height
        b = SimpleNamespace(width=w, height=h, depth=np.zeros(w * h, np.float32), point=np.zeros((w * h, 3)),
                            normal=np.zeros((w * h, 3)), canonical=np.zeros((w * h, 3)))
        v = GeometryBufferView(w, h, ptr(b.depth, C.c_float), ptr(b.point, C.c_double), ptr(b.normal, C.c_double),
                               ptr(b.canonical, C.c_double))
        self._check(lib().wfk_rasterize(self.h, C.byref(intr), C.c_int32(1), C.byref(v)))
        return b

    def upload_gbuffer(self, b):
        v = GeometryBufferView(b.width, b.height, ptr(np.ascontiguousarray(b.depth, np.float32), C.c_float),
                               ptr(np.ascontiguousarray(b.point), C.c_double),
                               ptr(np.ascontiguousarray(b.normal), C.c_double),
                               ptr(np.ascontiguousarray(b.canonical), C.c_double))
        self._check(lib().wfk_gbuffer_upload(self.h, C.byref(v)))

    def find_dense_correspondences(self, intr: Intrinsics, params: CorrespondParams, drop_inactive=False) -> int:
        n = C.c_int64()
        self._check(lib().wfk_find_dense_correspondences(self.h, C.byref(intr), C.byref(params),
                                                         C.c_int32(1 if drop_inactive else 0), C.byref(n)))
        return n.value

    # ---- per-frame pipeline --------------------------------------------------
    def process_frame(self, frame, pose: Pose, cfg: PipelineConfig, frame_index: int, sparse=None) -> FrameRecord:
        rec = FrameRecord()
        s = None if sparse is None or len(sparse) == 0 else np.ascontiguousarray(sparse, CORR_DTYPE)
        fv = frame.view()
        self._check(lib().wfk_process_frame(self.h, C.byref(fv), C.byref(pose), C.byref(cfg), _cptr(s),
                                            C.c_int64(0 if s is None else len(s)), C.c_int32(frame_index),
                                            C.byref(rec)))
        return rec

    def detect_features(self, params=None):
        """build_pyramid + detect_keypoints + extract_descriptors of the uploaded frame;
        returns (features[FEATURE_DTYPE], n_keypoints)."""
        p = params or FeatureParams.make()
        cap = 4 * max(p.max_keypoints, 1)
        out = np.zeros(cap, FEATURE_DTYPE)
        n, nk = C.c_int32(), C.c_int32()
        self._check(lib().wfk_detect_features(self.h, C.byref(p), _cptr(out), C.c_int32(cap), C.byref(n),
                                              C.byref(nk)))
        return out[: n.value].copy(), nk.value

    def match_features(self, current, store, predicted_world, intr, params=None):
        """match_features (features.cpp:416-433) on the device; returns MATCH_DTYPE records."""
        p = params or FeatureParams.make()
        cur = np.ascontiguousarray(current, FEATURE_DTYPE)
        st = np.ascontiguousarray(store, FEATURE_DTYPE)
        pw = np.ascontiguousarray(predicted_world, np.float64).reshape(-1, 3)
        cap = max(len(st), 1)
        out = np.zeros(cap, MATCH_DTYPE)
        n = C.c_int32()
        self._check(lib().wfk_match_features(self.h, _cptr(cur), C.c_int32(len(cur)), _cptr(st), C.c_int32(len(st)),
                                             ptr(pw, C.c_double), C.byref(intr), C.byref(p), _cptr(out),
                                             C.c_int32(cap), C.byref(n)))
        return out[: n.value].copy()

    def feature_store(self):
        """The context's FeatureStore (FEATURE_DTYPE records)."""
        n = C.c_int64()
        self._check(lib().wfk_feature_store_download(self.h, None, C.c_int64(0), C.byref(n)))
        out = np.zeros(max(n.value, 1), FEATURE_DTYPE)
        self._check(lib().wfk_feature_store_download(self.h, _cptr(out), C.c_int64(len(out)), C.byref(n)))
        return out[: n.value].copy()

    def set_feature_store(self, features):
        f = np.ascontiguousarray(features, FEATURE_DTYPE)
        self._check(lib().wfk_feature_store_upload(self.h, _cptr(f) if len(f) else None, C.c_int64(len(f))))

    def feature_pyramid_level(self, o, l, dog=False):
        w, h = C.c_int32(), C.c_int32()
        self._check(lib().wfk_feature_pyramid_level(self.h, o, l, int(dog), None, C.byref(w), C.byref(h)))
        out = np.zeros((h.value, w.value), np.float32)
        self._check(lib().wfk_feature_pyramid_level(self.h, o, l, int(dog), _cptr(out), C.byref(w), C.byref(h)))
        return out

    def invert_warp(self, pose: Pose, y, seed, max_iters=20, tol=1e-6):
        """DeformableVolume::invert_warp (volume.cpp:95-126) for each row; returns (x, ok)."""
        y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
        seed = np.ascontiguousarray(seed, np.float64).reshape(-1, 3)
        n = y.shape[0]
        x = np.zeros((n, 3), np.float64)
        ok = np.zeros(n, np.uint8)
        self._check(lib().wfk_invert_warp(self.h, C.byref(pose), C.c_int64(n), ptr(y, C.c_double),
                                          ptr(seed, C.c_double), C.c_int32(max_iters), C.c_double(tol),
                                          ptr(x, C.c_double), ptr(ok, C.c_uint8)))
        return x, ok.astype(bool)

    def upload_maps(self, maps):
        """A host PointNormalMap (e.g. the oracle's) as the context's frame maps."""
        mv = maps.view()
        self._check(lib().wfk_maps_upload(self.h, C.byref(mv)))

    def estimate_global_pose(self, intr, initial: Pose, params=None) -> IcpResult:
        """estimate_global_pose (solver.cpp:536-614) on the context's geometry
        buffer, frame maps and volume."""
        res = IcpResult()
        p = params or IcpParams.make()
        self._check(lib().wfk_estimate_global_pose(self.h, C.byref(intr), C.byref(initial), C.byref(p),
                                                   C.byref(res)))
        return res

    def stage_frame(self, slot: int, frame):
        fv = frame.view()
        self._check(lib().wfk_frame_stage(self.h, C.c_int32(slot), C.byref(fv)))

    def process_staged_frame(self, slot: int, pose: Pose, cfg: PipelineConfig, frame_index: int,
                             sparse=None) -> FrameRecord:
        rec = FrameRecord()
        s = None if sparse is None or len(sparse) == 0 else np.ascontiguousarray(sparse, CORR_DTYPE)
        self._check(lib().wfk_process_staged_frame(self.h, C.c_int32(slot), C.byref(pose), C.byref(cfg), _cptr(s),
                                                   C.c_int64(0 if s is None else len(s)),
                                                   C.c_int32(frame_index), C.byref(rec)))
        return rec

    # ---- measurement ---------------------------------------------------------
    def profile_enable(self, on: bool = True):
        self._check(lib().wfk_profile_enable(self.h, C.c_int32(1 if on else 0)))

    def profile_read(self) -> Profile:
        p = Profile()
        self._check(lib().wfk_profile_read(self.h, C.byref(p)))
        return p

    def timer_mark(self, slot: int):
        self._check(lib().wfk_timer_mark(self.h, C.c_int32(slot)))

    def timer_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        self._check(lib().wfk_timer_elapsed_ms(self.h, C.c_int32(a), C.c_int32(b), C.byref(ms)))
        return ms.value

    def flush_l2(self):
        self._check(lib().wfk_flush_l2(self.h))

    def debug_overrun(self, past_end: int):
        """Checked-mode self-test (include/wfk.h): a kernel writes `past_end`
        bytes beyond a scratch buffer; raises WfkError when WFK_CHECK caught it."""
        self._check(lib().wfk_debug_overrun(self.h, C.c_int32(past_end)))


def check_enabled() -> bool:
    """True when the library runs in checked mode (WFK_CHECK=1 at load)."""
    return bool(lib().wfk_check_enabled())

def pipeline_config(solver=None, correspond=None, fusion=None, reassociations=3, estimate_pose=True,
                    icp=None, use_features=True, features=None) -> PipelineConfig:
    """ReconstructorConfig defaults (config.hpp:30-46): ICP on, features on, 3 reassociations."""
    cfg = PipelineConfig()
    cfg.solver = solver or SolverParams.make()
    cfg.correspond = correspond or CorrespondParams.make()
    cfg.fusion = fusion or FusionParams.make()
    cfg.reassociations = reassociations
    cfg.estimate_pose = 1 if estimate_pose else 0
    cfg.icp = icp or IcpParams.make()
    cfg.use_features = 1 if use_features else 0
    cfg.features = features or FeatureParams.make()
    return cfg
