"""Restatements of the reference's seeded test fixtures.

* active_sphere_volume      proj/tests/test_solver.cpp:14-24 (radius 0.2) and
                            proj/tests/acceptance.cpp:100-110 (radius 0.3*voxel*(n-1))
* sparse_constraint         test_solver.cpp:26-37 / acceptance.cpp:112-125
* rigid_motion_constraints  test_solver.cpp:40-57
* node_constraints          acceptance.cpp:127-142
* make_volume               proj/bench/kernel_bench.cpp:15-29
* plane_frame               test_fusion.cpp:10-16, test_correspond.cpp:10-15
* sphere_volume             test_isosurface.cpp:12-20
Random draws come from oracle/fixtures.cpp (std::mt19937 + uniform_real_distribution).
"""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import (CORR_DTYPE, DENSE_PLANE, SPARSE_POINT, Frame, Intrinsics,
                                       Volume)

K320 = Intrinsics.make(280.0, 280.0, 159.5, 119.5, 320, 240)


def sphere_tsdf(v: Volume, center, radius, clamp_mu=False):
    c = v.canonical_positions()
    d = np.sqrt(np.sum((c - np.asarray(center)[None, :]) ** 2, axis=1)) - radius
    if clamp_mu:
        d = np.clip(d, -v.truncation, v.truncation)
    v.tsdf[:] = d.astype(np.float32)
    v.weight[:] = 1.0


def active_sphere_volume(n=12, voxel=0.05, radius=0.2) -> Volume:
    v = Volume((n, n, n), voxel, (-0.5 * voxel * (n - 1), -0.5 * voxel * (n - 1), 1.0))
    center = v.origin + 0.5 * voxel * (n - 1) * np.ones(3)
    sphere_tsdf(v, center, radius)
    O.compute_active_set(v)
    return v


def acceptance_sphere_volume(n, voxel) -> Volume:
    return active_sphere_volume(n, voxel, 0.3 * voxel * (n - 1))


def sparse_constraint(v: Volume, canonical, target):
    rec = np.zeros(1, CORR_DTYPE)
    idx, w = O.trilinear_anchors(v, canonical)
    rec["kind"] = SPARSE_POINT
    rec["canonical"] = canonical
    rec["anchor_index"] = idx
    rec["anchor_weight"] = w
    rec["target"] = target
    rec["confidence"] = 1.0
    return rec


def node_constraints(v: Volume, stride: int, target_fn):
    out = []
    eps = 1e-9 * np.ones(3)
    for i in range(0, v.num_points, stride):
        if not v.active[i]:
            continue
        c = v.canonical_position(i)
        if not (O.contains(v, c + eps) and O.contains(v, c - eps)):
            continue
        idx, _ = O.trilinear_anchors(v, c)
        if not all(v.active[j] for j in idx):
            continue
        out.append(sparse_constraint(v, c, target_fn(c)))
    return np.concatenate(out) if out else np.zeros(0, CORR_DTYPE)


def rigid_motion_constraints(v: Volume, r, t):
    r = np.asarray(r)
    t = np.asarray(t)
    return node_constraints(v, 3, lambda c: r @ c + t)


def make_volume(n: int) -> Volume:
    vol = Volume((n, n, n), 1.0 / (n - 1), (-0.5, -0.5, 0.7))
    sphere_tsdf(vol, (0, 0, 1.2), 0.35, clamp_mu=True)
    O.compute_active_set(vol)
    rng = O.Rng(11)
    vol.deformed += rng.vec3_array(-0.002, 0.002, vol.num_points)
    return vol


def plane_frame(z, gray=None, k=K320) -> Frame:
    depth = np.full((k.height, k.width), np.float32(z), np.float32)
    color = None if gray is None else np.full((k.height, k.width, 3), np.float32(gray), np.float32)
    return Frame(k, depth, color)


def sphere_volume(n, voxel, center, radius) -> Volume:
    center = np.asarray(center, np.float64)
    v = Volume((n, n, n), voxel, center - 0.5 * voxel * (n - 1) * np.ones(3))
    sphere_tsdf(v, center, radius)
    return v


def random_dense_constraints(v: Volume, count: int, seed: int, normal_jitter=0.3):
    """Dense point-to-plane constraints at random canonical points of fully
    active cells (same record layout find_dense_correspondences emits)."""
    rng = np.random.default_rng(seed)
    out = []
    tries = 0
    pos = v.canonical_positions()
    act = np.nonzero(v.active)[0]
    while len(out) < count and tries < 50 * count:
        tries += 1
        i = act[rng.integers(len(act))]
        c = pos[i] + rng.uniform(0.0, 1.0, 3) * v.voxel_size
        if not O.contains(v, c):
            continue
        idx, w = O.trilinear_anchors(v, c)
        if not all(v.active[j] for j in idx):
            continue
        n = np.array([0.0, 0.0, -1.0]) + rng.uniform(-normal_jitter, normal_jitter, 3)
        n /= np.linalg.norm(n)
        rec = np.zeros(1, CORR_DTYPE)
        rec["kind"] = DENSE_PLANE
        rec["canonical"] = c
        rec["anchor_index"] = idx
        rec["anchor_weight"] = w
        rec["target"] = c + rng.uniform(-0.01, 0.01, 3)
        rec["target_normal"] = n
        rec["confidence"] = rng.uniform(0.3, 1.0)
        out.append(rec)
    return np.concatenate(out) if out else np.zeros(0, CORR_DTYPE)
