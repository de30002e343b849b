"""ORACLE -- test infrastructure only (tests/, __graft_entry__.smoke(), bench.py's
CPU-baseline leg).  ctypes front end of the wfo_* C ABI (oracle/wfo.h), served
by one of two CPU backends:

* "ref"  -- oracle/_ref/libwfref.so: the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled against the Eigen/doctest shims
  (oracle/ref/Makefile), behind a conversion-only C ABI (oracle/ref/capi.cpp);
* "port" -- oracle/_build/liboracle.so: the line-by-line restatement
  (oracle/wf_oracle.cpp), kept as the checker where the reference has no
  public entry point and as a cross-check of the reference build.

WF_ORACLE=ref|port picks the backend (default: "ref" when libwfref.so is
built, else "port"); set_backend() switches it at run time.  Never imported by
the product package."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1603_08161_b200.abi import (
    CORR_DTYPE, FEATURE_DTYPE, MATCH_DTYPE, CorrespondParams, Energy, ExpansionStats, FeatureParams, FusionParams,
    FusionStats,
    GeometryBufferView, IcpParams, IcpResult, Intrinsics, MeshView, PcgResult, PointNormalMapView, Pose,
    SolverParams, TraceEntry, VolumeView, FrameView, Volume, ptr, trace_to_list,
    WFK_OK, WFK_E_CAPACITY, WFK_E_INVALID_ARG, WFK_E_OUT_OF_RANGE, WFK_E_LOGIC,
    EXEC_PARALLEL)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libwfref.so")
REFERENCE_SRC = "/root/reference/proj"


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def build_ref(force: bool = False) -> str | None:
    """Compile the reference into oracle/_ref (only where /root/reference is
    mounted; the GPU box uses the prebuilt files)."""
    if (force or not os.path.exists(REF_LIB_PATH)) and os.path.isdir(REFERENCE_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "ref")], check=True)
    return REF_LIB_PATH if os.path.exists(REF_LIB_PATH) else None


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


_libs: dict = {}
_backend = os.environ.get("WF_ORACLE") or ("ref" if os.path.exists(REF_LIB_PATH) else "port")


def backend() -> str:
    return _backend


def set_backend(kind: str) -> str:
    """Switch the wfo_* backend ("ref" or "port"); returns the previous one.
    Handles (normal equations, meshes, reconstructors) belong to the backend
    that made them."""
    global _backend
    if kind not in ("ref", "port"):
        raise ValueError(kind)
    prev, _backend = _backend, kind
    return prev


def lib(kind: str | None = None):
    kind = kind or _backend
    if kind not in _libs:
        if kind == "ref":
            path = build_ref()
            if path is None:
                raise OracleError(WFK_E_INVALID_ARG, "reference build oracle/_ref/libwfref.so is missing")
        else:
            path = build()
        l = C.CDLL(path)
        _declare(l)
        _libs[kind] = l
    return _libs[kind]


def _declare(l):
    vp = C.POINTER(VolumeView)
    cp = C.c_void_p
    l.wfo_last_error.restype = C.c_char_p
    l.wfo_ne_symmetry_error.restype = C.c_double
    l.wfo_dense_confidence.restype = C.c_double
    l.wfo_dense_confidence.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(CorrespondParams)]
    l.wfo_rng_new.restype = cp
    l.wfo_rng_new.argtypes = [C.c_uint32]
    l.wfo_rng_free.argtypes = [cp]
    l.wfo_rng_uniform.restype = C.c_double
    l.wfo_rng_uniform.argtypes = [cp, C.c_double, C.c_double]
    l.wfo_rng_vec3.argtypes = [cp, C.c_double, C.c_double, C.POINTER(C.c_double)]
    l.wfo_rng_int.argtypes = [cp, C.c_int, C.c_int]
    l.wfo_rng_vec3_array.argtypes = [cp, C.c_double, C.c_double, C.c_int64, C.POINTER(C.c_double)]
    l.wfo_ne_num_rows.restype = C.c_int32
    l.wfo_ne_num_rows.argtypes = [cp]
    l.wfo_ne_free.argtypes = [cp]
    l.wfo_mesh_free.argtypes = [cp]
    l.wfo_recon_free.argtypes = [cp]
    l.wfo_ne_export.argtypes = [cp] + [C.c_void_p] * 6
    l.wfo_ne_multiply.argtypes = [cp, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32]
    l.wfo_ne_symmetry_error.argtypes = [cp]
    l.wfo_ne_pcg_solve.argtypes = [cp, C.POINTER(C.c_double), C.c_double, C.c_int32, C.c_int32,
                                   C.POINTER(PcgResult)]
    l.wfo_mesh_sizes.argtypes = [cp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    l.wfo_mesh_export.argtypes = [cp, C.POINTER(MeshView)]
    l.wfo_mesh_warp.argtypes = [cp, vp, C.POINTER(Pose)]
    l.wfo_compute_normals.argtypes = [cp]
    l.wfo_rasterize.argtypes = [cp, C.POINTER(Intrinsics), C.c_int32, C.POINTER(GeometryBufferView)]
    l.wfo_recon_volume.argtypes = [cp, vp]
    l.wfo_recon_process_frame.argtypes = [cp, C.POINTER(FrameView), C.c_void_p, C.c_int64, C.c_void_p]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != WFK_OK:
        raise OracleError(rc, lib().wfo_last_error().decode())


def _cptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# --- seeded streams (oracle/fixtures.cpp) ----------------------------------
class Rng:
    """std::mt19937 + uniform_real_distribution<double>, as the reference tests draw."""

    def __init__(self, seed: int):
        self.h = lib().wfo_rng_new(int(seed))

    def __del__(self):
        if getattr(self, "h", None):
            lib().wfo_rng_free(self.h)
            self.h = None

    def uniform(self, lo, hi) -> float:
        return lib().wfo_rng_uniform(self.h, float(lo), float(hi))

    def vec3(self, lo, hi) -> np.ndarray:
        out = np.zeros(3)
        lib().wfo_rng_vec3(self.h, float(lo), float(hi), ptr(out, C.c_double))
        return out

    def vec3_array(self, lo, hi, n) -> np.ndarray:
        out = np.zeros((n, 3))
        lib().wfo_rng_vec3_array(self.h, float(lo), float(hi), int(n), ptr(out, C.c_double))
        return out

    def randint(self, lo, hi) -> int:
        return lib().wfo_rng_int(self.h, int(lo), int(hi))


# --- core / volume ------------------------------------------------------------
def euler_to_matrix(abc) -> np.ndarray:
    a = np.asarray(abc, np.float64).reshape(3).copy()
    r = np.zeros(9)
    lib().wfo_euler_to_matrix(ptr(a, C.c_double), ptr(r, C.c_double))
    return r.reshape(3, 3)


def matrix_to_euler(r) -> np.ndarray:
    m = np.ascontiguousarray(r, np.float64).reshape(9).copy()
    e = np.zeros(3)
    lib().wfo_matrix_to_euler(ptr(m, C.c_double), ptr(e, C.c_double))
    return e


def svd3(a):
    m = np.ascontiguousarray(a, np.float64).reshape(9).copy()
    u, s, v = np.zeros(9), np.zeros(3), np.zeros(9)
    lib().wfo_svd3(*(ptr(x, C.c_double) for x in (m, u, s, v)))
    return u.reshape(3, 3), s, v.reshape(3, 3)


def contains(vol: Volume, x) -> bool:
    p = np.asarray(x, np.float64).reshape(3).copy()
    vv = vol.view()
    return bool(lib().wfo_contains(C.byref(vv), ptr(p, C.c_double)))


def trilinear_anchors(vol: Volume, x):
    p = np.asarray(x, np.float64).reshape(3).copy()
    idx = np.zeros(8, np.int32)
    w = np.zeros(8)
    vv = vol.view()
    _check(lib().wfo_trilinear_anchors(C.byref(vv), ptr(p, C.c_double), ptr(idx, C.c_int32),
                                       ptr(w, C.c_double)))
    return idx, w


def warp_point(vol: Volume, pose: Pose, x):
    p = np.asarray(x, np.float64).reshape(3).copy()
    out = np.zeros(3)
    vv = vol.view()
    _check(lib().wfo_warp_point(C.byref(vv), C.byref(pose), ptr(p, C.c_double), ptr(out, C.c_double)))
    return out


# --- solver -------------------------------------------------------------------
def compute_active_set(vol: Volume) -> np.ndarray:
    out = np.zeros(vol.num_points, np.int32)
    n = C.c_int64()
    vv = vol.view()
    _check(lib().wfo_compute_active_set(C.byref(vv), ptr(out, C.c_int32), C.c_int64(out.size), C.byref(n)))
    return out[: n.value].copy()


def _cons(cons):
    if cons is None or len(cons) == 0:
        return None, 0
    cons = np.ascontiguousarray(cons, dtype=CORR_DTYPE)
    return cons, len(cons)


class NormalEquations:
    """wf::NormalEquations (solver.hpp:46-60) materialised from the oracle."""

    def __init__(self, vol: Volume, pose: Pose, cons, params: SolverParams):
        c, n = _cons(cons)
        h = C.c_void_p()
        vv = vol.view()
        _check(lib().wfo_build_normal_equations(C.byref(vv), C.byref(pose), _cptr(c), C.c_int64(n),
                                                C.byref(params), C.byref(h)))
        self.h = h
        self._l = lib()  # handles belong to the backend that made them
        nr = self._l.wfo_ne_num_rows(h)
        self.rows = np.zeros(nr, np.int32)
        self.node_row = np.zeros(vol.num_points, np.int32)
        self.blocks = np.zeros((nr, 27, 3, 3))
        self.cols = np.zeros((nr, 27), np.int32)
        self.rhs = np.zeros((nr, 3))
        self.frozen = np.zeros(nr, np.uint8)
        self._l.wfo_ne_export(h, *(_cptr(a) for a in (self.rows, self.node_row, self.blocks, self.cols,
                                                     self.rhs, self.frozen)))

    def __del__(self):
        if getattr(self, "h", None):
            self._l.wfo_ne_free(self.h)
            self.h = None

    @property
    def num_rows(self):
        return len(self.rows)

    def multiply(self, x, exec_=EXEC_PARALLEL):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._l.wfo_ne_multiply(self.h, ptr(x, C.c_double), ptr(y, C.c_double), exec_)
        return y

    def symmetry_error(self):
        return self._l.wfo_ne_symmetry_error(self.h)

    def pcg_solve(self, x, tol, max_iters, exec_=EXEC_PARALLEL):
        x = np.ascontiguousarray(x, np.float64)
        res = PcgResult()
        _check(self._l.wfo_ne_pcg_solve(self.h, ptr(x, C.c_double), float(tol), int(max_iters), exec_,
                                      C.byref(res)))
        return x, res.iterations, res.relative_residual


def evaluate_energy(vol, pose, cons, params) -> dict:
    c, n = _cons(cons)
    e = Energy()
    vv = vol.view()
    _check(lib().wfo_evaluate_energy(C.byref(vv), C.byref(pose), _cptr(c), C.c_int64(n),
                                     C.byref(params), C.byref(e)))
    return e.as_dict()


def update_rotations(vol, exec_=EXEC_PARALLEL):
    vv = vol.view()
    _check(lib().wfo_update_rotations(C.byref(vv), exec_))


def _trace_call(fn, *args, cap=4096):
    buf = (TraceEntry * cap)()
    n = C.c_int32()
    _check(fn(*args, buf, C.c_int32(cap), C.byref(n)))
    return trace_to_list(buf, n.value)


def flip_flop_solve(vol, pose, cons, params, level=0):
    c, n = _cons(cons)
    vv = vol.view()
    return _trace_call(lib().wfo_flip_flop_solve, C.byref(vv), C.byref(pose), _cptr(c), C.c_int64(n),
                       C.byref(params), C.c_int32(level))


def solve_coarse_to_fine(vol, pose, cons, params):
    c, n = _cons(cons)
    vv = vol.view()
    return _trace_call(lib().wfo_solve_coarse_to_fine, C.byref(vv), C.byref(pose), _cptr(c), C.c_int64(n),
                       C.byref(params))


def hierarchy_info(vol, cons, levels, want_level=-1):
    c, n = _cons(cons)
    dims = np.zeros((levels, 3), np.int32)
    act = np.zeros(levels, np.int64)
    out = np.zeros(max(n, 1), CORR_DTYPE) if want_level >= 0 else None
    vv = vol.view()
    _check(lib().wfo_hierarchy_info(C.byref(vv), _cptr(c), C.c_int64(n), C.c_int32(levels), _cptr(dims),
                                    _cptr(act), C.c_int32(want_level), _cptr(out)))
    return dims, act, (out[:n] if out is not None else None)


# --- fusion -------------------------------------------------------------------
def integrate_frame(vol, frame, pose, params: FusionParams, exec_=EXEC_PARALLEL):
    s = FusionStats()
    vv, fv = vol.view(), frame.view()
    _check(lib().wfo_integrate_frame(C.byref(vv), C.byref(fv), C.byref(pose), C.byref(params), exec_,
                                     C.byref(s)))
    return s


def expand_grid(vol):
    s = ExpansionStats()
    vv = vol.view()
    _check(lib().wfo_expand_grid(C.byref(vv), C.byref(s)))
    return s


def advance_ages(vol, idx):
    idx = np.ascontiguousarray(idx, np.int32)
    vv = vol.view()
    _check(lib().wfo_advance_ages(C.byref(vv), ptr(idx, C.c_int32), C.c_int64(idx.size)))


# --- correspondence -----------------------------------------------------------
class PointNormalMap:
    def __init__(self, w, h):
        self.width, self.height = w, h
        self.point = np.zeros((h * w, 3))
        self.normal = np.zeros((h * w, 3))
        self.point_valid = np.zeros(h * w, np.uint8)
        self.normal_valid = np.zeros(h * w, np.uint8)

    def view(self):
        m = PointNormalMapView(self.width, self.height, ptr(self.point, C.c_double),
                               ptr(self.normal, C.c_double), ptr(self.point_valid, C.c_uint8),
                               ptr(self.normal_valid, C.c_uint8))
        m._keep = self
        return m


class GeometryBuffer:
    def __init__(self, w, h):
        self.width, self.height = w, h
        self.depth = np.full(h * w, np.inf, np.float32)
        self.point = np.zeros((h * w, 3))
        self.normal = np.zeros((h * w, 3))
        self.canonical = np.zeros((h * w, 3))

    def view(self):
        g = GeometryBufferView(self.width, self.height, ptr(self.depth, C.c_float),
                               ptr(self.point, C.c_double), ptr(self.normal, C.c_double),
                               ptr(self.canonical, C.c_double))
        g._keep = self
        return g

    def valid(self):
        return np.isfinite(self.depth)


def backproject_depth(frame, exec_=EXEC_PARALLEL) -> PointNormalMap:
    k = frame.intrinsics
    m = PointNormalMap(k.width, k.height)
    fv, mv = frame.view(), m.view()
    _check(lib().wfo_backproject_depth(C.byref(fv), exec_, C.byref(mv)))
    return m


def dense_confidence(dist, nd, vd, params=None) -> float:
    p = params or CorrespondParams.make()
    return lib().wfo_dense_confidence(dist, nd, vd, C.byref(p))


def sample_point_normal(maps: PointNormalMap, uv):
    u = np.asarray(uv, np.float64).reshape(2).copy()
    p, n = np.zeros(3), np.zeros(3)
    mv = maps.view()
    ok = lib().wfo_sample_point_normal(C.byref(mv), ptr(u, C.c_double), ptr(p, C.c_double),
                                       ptr(n, C.c_double))
    return bool(ok), p, n


def find_dense_correspondences(buf, maps, intr, params, vol):
    cap = buf.width * buf.height
    out = np.zeros(max(cap, 1), CORR_DTYPE)
    n = C.c_int64()
    bv, mv, vv = buf.view(), maps.view(), vol.view()
    _check(lib().wfo_find_dense_correspondences(C.byref(bv), C.byref(mv), C.byref(intr), C.byref(params),
                                                C.byref(vv), _cptr(out), C.c_int64(cap), C.byref(n)))
    return out[: n.value].copy()


def estimate_global_pose(buf, maps, intr, vol, initial=None, params=None) -> IcpResult:
    """estimate_global_pose (solver.cpp:536-614)."""
    res = IcpResult()
    bv, mv, vv = buf.view(), maps.view(), vol.view()
    p = params or IcpParams.make()
    ini = initial or Pose.make()
    _check(lib().wfo_estimate_global_pose(C.byref(bv), C.byref(mv), C.byref(intr), C.byref(vv), C.byref(ini),
                                          C.byref(p), C.byref(res)))
    return res


# --- feature front-end (features.cpp) ---------------------------------------------
def detect_features(frame, params=None):
    """build_pyramid + detect_keypoints + extract_descriptors of a frame
    (pipeline.cpp:97-101); returns (features[FEATURE_DTYPE], n_keypoints)."""
    p = params or FeatureParams.make()
    cap = 4 * max(p.max_keypoints, 1)
    out = np.zeros(cap, FEATURE_DTYPE)
    n = C.c_int32()
    nk = C.c_int32()
    fv = frame.view()
    _check(lib().wfo_detect_features(C.byref(fv), C.byref(p), _cptr(out), C.c_int32(cap), C.byref(n), C.byref(nk)))
    return out[: n.value].copy(), nk.value


def pyramid_level(frame, o, l, dog=False, params=None):
    p = params or FeatureParams.make()
    w, h = C.c_int32(), C.c_int32()
    fv = frame.view()
    _check(lib().wfo_pyramid_level(C.byref(fv), C.byref(p), o, l, int(dog), None, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value), np.float32)
    _check(lib().wfo_pyramid_level(C.byref(fv), C.byref(p), o, l, int(dog), _cptr(out), C.byref(w), C.byref(h)))
    return out


def descriptor_distance(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    lib().wfo_descriptor_distance.restype = C.c_double
    return lib().wfo_descriptor_distance(ptr(a, C.c_float), ptr(b, C.c_float))


def match_features(current, store, predicted_world, intr, params=None):
    """match_features (features.cpp:416-433)."""
    p = params or FeatureParams.make()
    cur = np.ascontiguousarray(current, FEATURE_DTYPE)
    st = np.ascontiguousarray(store, FEATURE_DTYPE)
    pw = np.ascontiguousarray(predicted_world, np.float64).reshape(-1, 3)
    cap = max(len(st), 1)
    out = np.zeros(cap, MATCH_DTYPE)
    n = C.c_int32()
    _check(lib().wfo_match_features(_cptr(cur), C.c_int32(len(cur)), _cptr(st), C.c_int32(len(st)),
                                    ptr(pw, C.c_double), C.byref(intr), C.byref(p), _cptr(out), C.c_int32(cap),
                                    C.byref(n)))
    return out[: n.value].copy()


def invert_warp(vol, pose, y, seed, max_iters=20, tol=1e-6):
    """DeformableVolume::invert_warp (volume.cpp:95-126) for each row of y / seed;
    returns (x, ok)."""
    y = np.ascontiguousarray(y, np.float64).reshape(-1, 3)
    seed = np.ascontiguousarray(seed, np.float64).reshape(-1, 3)
    n = y.shape[0]
    x = np.zeros((n, 3), np.float64)
    ok = np.zeros(n, np.uint8)
    vv = vol.view()
    p = pose or Pose.make()
    _check(lib().wfo_invert_warp(C.byref(vv), C.byref(p), C.c_int64(n), ptr(y, C.c_double), ptr(seed, C.c_double),
                                 C.c_int32(max_iters), C.c_double(tol), ptr(x, C.c_double), ptr(ok, C.c_uint8)))
    return x, ok.astype(bool)


def ldlt_solve(a, b):
    """Eigen LDLT (symmetric pivoting) restated: solve a x = b, a symmetric n x n, n <= 8."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64).reshape(-1)
    n = b.shape[0]
    x = np.zeros(n, np.float64)
    _check(lib().wfo_ldlt_solve(C.c_int(n), ptr(a, C.c_double), ptr(b, C.c_double), ptr(x, C.c_double)))
    return x


def sparse_to_constraints(canonical, target, vol):
    canonical = np.ascontiguousarray(canonical, np.float64).reshape(-1, 3)
    target = np.ascontiguousarray(target, np.float64).reshape(-1, 3)
    out = np.zeros(max(len(canonical), 1), CORR_DTYPE)
    n = C.c_int64()
    vv = vol.view()
    _check(lib().wfo_sparse_to_constraints(ptr(canonical, C.c_double), ptr(target, C.c_double),
                                           C.c_int64(len(canonical)), C.byref(vv), _cptr(out), C.byref(n)))
    return out[: n.value].copy()


class Mesh:
    """wf::SurfaceMesh from the oracle, copied into numpy."""

    def __init__(self, handle):
        self.h = handle
        self._l = lib()  # handles belong to the backend that made them
        self.refresh()

    def refresh(self):
        nv, nt = C.c_int64(), C.c_int64()
        self._l.wfo_mesh_sizes(self.h, C.byref(nv), C.byref(nt))
        V, T = nv.value, nt.value
        self.vertices_canonical = np.zeros((V, 3))
        self.vertices_deformed = np.zeros((V, 3))
        self.normals_deformed = np.zeros((V, 3))
        self.colors = np.zeros((V, 3), np.float32)
        self.triangles = np.zeros((T, 3), np.int32)
        mv = MeshView(V, T, ptr(self.vertices_canonical, C.c_double), ptr(self.vertices_deformed, C.c_double),
                      ptr(self.normals_deformed, C.c_double), ptr(self.colors, C.c_float),
                      ptr(self.triangles, C.c_int32))
        self._l.wfo_mesh_export(self.h, C.byref(mv))

    def __del__(self):
        if getattr(self, "h", None):
            self._l.wfo_mesh_free(self.h)
            self.h = None

    def compute_normals(self):
        self._l.wfo_compute_normals(self.h)
        self.refresh()

    def warp(self, vol, pose):
        vv = vol.view()
        _check(self._l.wfo_mesh_warp(self.h, C.byref(vv), C.byref(pose)))
        self.refresh()

    def rasterize(self, intr, exec_=EXEC_PARALLEL) -> GeometryBuffer:
        b = GeometryBuffer(intr.width, intr.height)
        bv = b.view()
        _check(self._l.wfo_rasterize(self.h, C.byref(intr), exec_, C.byref(bv)))
        return b


def extract_mesh(vol, pose=None) -> Mesh:
    h = C.c_void_p()
    vv = vol.view()
    p = pose or Pose.make()
    _check(lib().wfo_extract_mesh(C.byref(vv), C.byref(p), C.byref(h)))
    return Mesh(h)


def synth_render(intr, center=(0.0, 0.0, 1.2), radius=0.3, pivot=(0.0, 0.0, 1.2), amplitude=0.0,
                 driver_axis=0, rot_axis=1, tex_seed=7, tex_scale=0.06, dot_radius=0.3):
    """SyntheticScene::render_frame for a sphere under the bend warp (test-bed)."""
    depth = np.zeros((intr.height, intr.width), np.float32)
    color = np.zeros((intr.height, intr.width, 3), np.float32)
    c = np.asarray(center, np.float64).copy()
    pv = np.asarray(pivot, np.float64).copy()
    l = lib()
    l.wfo_synth_render.argtypes = [C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double), C.c_double,
                                   C.c_int, C.c_int, C.c_uint32, C.c_double, C.c_double,
                                   C.POINTER(Intrinsics), C.c_void_p, C.c_void_p]
    _check(l.wfo_synth_render(ptr(c, C.c_double), radius, ptr(pv, C.c_double), amplitude, driver_axis,
                              rot_axis, tex_seed, tex_scale, dot_radius, C.byref(intr), _cptr(depth),
                              _cptr(color)))
    return depth, color


# --- per-frame pipeline (pipeline.cpp:143-262, hot-path subset) -------------------
class ReconConfig(C.Structure):
    _fields_ = [("dims", C.c_int32 * 3), ("reassociations", C.c_int32), ("voxel_size", C.c_double),
                ("origin", C.c_double * 3), ("solver", SolverParams), ("correspond", CorrespondParams),
                ("fusion", FusionParams), ("estimate_pose", C.c_int32), ("reserved_", C.c_int32),
                ("icp", IcpParams), ("use_features", C.c_int32), ("reserved2_", C.c_int32),
                ("features", FeatureParams)]


class FrameRecord(C.Structure):
    _fields_ = [("energy", Energy), ("dense_count", C.c_int32), ("sparse_count", C.c_int32),
                ("anomalies", C.c_int32), ("trace_len", C.c_int32), ("pcg_iterations", C.c_int32),
                ("reserved_", C.c_int32), ("fusion", FusionStats), ("expansion", ExpansionStats),
                ("pose", Pose), ("icp_degraded", C.c_int32), ("icp_iterations", C.c_int32),
                ("icp_rms", C.c_double), ("match_count", C.c_int32), ("features_added", C.c_int32)]


class Reconstructor:
    def __init__(self, dims, voxel, origin, solver=None, correspond=None, fusion=None, reassociations=3,
                 estimate_pose=True, icp=None, use_features=True, features=None):
        cfg = ReconConfig()
        cfg.dims[:] = list(dims)
        cfg.voxel_size = voxel
        cfg.origin[:] = list(origin)
        cfg.reassociations = reassociations
        cfg.solver = solver or SolverParams.make()
        cfg.correspond = correspond or CorrespondParams.make()
        cfg.fusion = fusion or FusionParams.make()
        cfg.estimate_pose = 1 if estimate_pose else 0
        cfg.icp = icp or IcpParams.make()
        cfg.use_features = 1 if use_features else 0
        cfg.features = features or FeatureParams.make()
        self.cfg = cfg
        h = C.c_void_p()
        self._l = lib()  # handles belong to the backend that made them
        _check(self._l.wfo_recon_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self._l.wfo_recon_free(self.h)
            self.h = None

    def volume_view(self) -> VolumeView:
        v = VolumeView()
        self._l.wfo_recon_volume(self.h, C.byref(v))
        return v

    def volume_arrays(self) -> dict:
        v = self.volume_view()
        n = v.dims[0] * v.dims[1] * v.dims[2]
        def arr(p, shape, dt):
            return np.ctypeslib.as_array(p, shape=shape).astype(dt, copy=True)
        return dict(tsdf=arr(v.tsdf, (n,), np.float32), weight=arr(v.weight, (n,), np.float32),
                    color=arr(v.color, (n, 3), np.float32), deformed=arr(v.deformed, (n, 3), np.float64),
                    euler=arr(v.euler, (n, 3), np.float64), age=arr(v.age, (n,), np.int32),
                    active=arr(v.active, (n,), np.uint8))

    def feature_store(self):
        n = C.c_int64()
        _check(self._l.wfo_recon_feature_store(self.h, None, C.c_int64(0), C.byref(n)))
        out = np.zeros(max(n.value, 1), FEATURE_DTYPE)
        _check(self._l.wfo_recon_feature_store(self.h, _cptr(out), C.c_int64(len(out)), C.byref(n)))
        return out[: n.value].copy()

    def process_frame(self, frame, sparse=None) -> FrameRecord:
        rec = FrameRecord()
        s, n = _cons(sparse)
        fv = frame.view()
        _check(self._l.wfo_recon_process_frame(self.h, C.byref(fv), _cptr(s), C.c_int64(n), C.byref(rec)))
        return rec


# ---- snapshot / frame formats (wf_formats.cpp) ------------------------------------
def _bytes_call(fn, *args):
    n = C.c_int64()
    _check(fn(*args, None, C.c_int64(0), C.byref(n)))
    out = np.zeros(n.value, np.uint8)
    _check(fn(*args, _cptr(out), C.c_int64(n.value), C.byref(n)))
    return out.tobytes()


def volume_save_bytes(vol) -> bytes:
    """DeformableVolume::save (volume.cpp:150-178) as bytes."""
    vv = vol.view()
    return _bytes_call(lib().wfo_volume_save_bytes, C.byref(vv))


def volume_load_bytes(image: bytes):
    """DeformableVolume::load (volume.cpp:180-217) from bytes."""
    from paper_1603_08161_b200.abi import Volume as _V, VolumeView as _VV
    buf = np.frombuffer(image, np.uint8)
    hv = _VV()
    _check(lib().wfo_volume_load_bytes(_cptr(buf), C.c_int64(len(buf)), C.byref(hv)))
    v = _V(tuple(hv.dims), hv.voxel_size, tuple(hv.origin))
    vv = v.view()
    _check(lib().wfo_volume_load_bytes(_cptr(buf), C.c_int64(len(buf)), C.byref(vv)))
    v.truncation = vv.truncation
    return v


def feature_store_bytes(features) -> bytes:
    """FeatureStore::save (features.cpp:306-323) as bytes."""
    f = np.ascontiguousarray(features, FEATURE_DTYPE)
    return _bytes_call(lib().wfo_feature_store_bytes, _cptr(f), C.c_int32(len(f)))


def pgm_encode(depth) -> bytes:
    d = np.ascontiguousarray(depth, np.float32)
    return _bytes_call(lib().wfo_pgm_encode, _cptr(d), C.c_int32(d.shape[1]), C.c_int32(d.shape[0]))


def ppm_encode(color) -> bytes:
    c = np.ascontiguousarray(color, np.float32)
    return _bytes_call(lib().wfo_ppm_encode, _cptr(c), C.c_int32(c.shape[1]), C.c_int32(c.shape[0]))


def pnm_decode(image: bytes, channels: int):
    buf = np.frombuffer(image, np.uint8)
    w, h = C.c_int32(), C.c_int32()
    _check(lib().wfo_pnm_decode(_cptr(buf), C.c_int64(len(buf)), C.c_int32(channels), C.byref(w), C.byref(h), None))
    shape = (h.value, w.value) if channels == 1 else (h.value, w.value, 3)
    out = np.zeros(shape, np.float32)
    _check(lib().wfo_pnm_decode(_cptr(buf), C.c_int64(len(buf)), C.c_int32(channels), C.byref(w), C.byref(h),
                                _cptr(out)))
    return out
