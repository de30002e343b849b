"""Parity of the B200 solver (libwfk.so via its C ABI) against the oracle.

Integer and index work must be bit-exact (rows, node_row, stencil columns,
frozen rows, active sets).  Floating-point work is compared against the oracle
with the tolerances of BASELINE.json's north_star: <= 1e-4 relative on final
energy and <= 1e-3 voxel on deformed positions; the assembled quantities that
are computed in the reference's own operation order are held to 1e-12."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200.abi import CORR_DTYPE, Pose, SolverParams, Volume
from tests.fixtures import (acceptance_sphere_volume, active_sphere_volume, make_volume, node_constraints,
                            random_dense_constraints, rigid_motion_constraints)

pytestmark = pytest.mark.gpu

ENERGY_RTOL = 1e-4     # north_star: final energy
POS_TOL_VOXEL = 1e-3   # north_star: deformed positions, in voxels


@pytest.fixture(scope="module")
def ctx():
    from paper_1603_08161_b200.wfk import Context
    c = Context(0)
    yield c
    c.close()


def jittered_sphere(n=12, voxel=0.05, seed=21, amp=0.02, euler_amp=0.0):
    v = active_sphere_volume(n, voxel)
    rng = O.Rng(seed)
    for i in range(v.num_points):
        v.deformed[i] += rng.vec3(-amp, amp)
        if euler_amp:
            v.euler[i] = euler_amp * rng.vec3(-1, 1)
    return v


def test_active_set_bit_exact(ctx):
    v = Volume((20, 20, 20), 0.05, (-0.475, -0.475, 1.0))
    from tests.fixtures import sphere_tsdf
    sphere_tsdf(v, v.origin + 0.475, 0.31)
    v.weight[::7] = 0  # unobserved corners
    ref = v.copy()
    exp = O.compute_active_set(ref)
    ctx.upload_volume(v)
    got = ctx.compute_active_set()
    assert np.array_equal(got, exp)
    ctx.download_volume(v)
    assert np.array_equal(v.active, ref.active)
    # grow-only
    v.tsdf += np.float32(0.05)
    ref.tsdf += np.float32(0.05)
    ctx.upload_volume(v)
    assert np.array_equal(ctx.compute_active_set(), O.compute_active_set(ref))


def test_normal_equations_match_reference_layout(ctx):
    v = jittered_sphere(euler_amp=0.05)
    cons = np.concatenate([rigid_motion_constraints(v, np.eye(3), (0.01, 0, 0)),
                           random_dense_constraints(v, 150, seed=3)])
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.01, -0.02, 0.03)), (0.01, 0.0, -0.02))
    ref = O.NormalEquations(v, pose, cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    got = ctx.build_normal_equations(pose, p)
    assert np.array_equal(got["rows"], ref.rows)
    assert np.array_equal(got["node_row"], ref.node_row)
    assert np.array_equal(got["cols"], ref.cols)
    assert np.array_equal(got["frozen"], ref.frozen)
    scale = np.max(np.abs(ref.blocks))
    assert np.max(np.abs(got["blocks"] - ref.blocks)) <= 1e-12 * scale
    assert np.max(np.abs(got["rhs"] - ref.rhs)) <= 1e-12 * np.max(np.abs(ref.rhs))


def test_frozen_component_detection(ctx):
    # two disjoint shells; constraints only on one -> the other is frozen
    v = Volume((24, 12, 12), 0.05, (0, 0, 1.0))
    c = v.canonical_positions()
    d1 = np.linalg.norm(c - (0.275, 0.275, 1.275), axis=1) - 0.15
    d2 = np.linalg.norm(c - (0.875, 0.275, 1.275), axis=1) - 0.15
    v.tsdf[:] = np.minimum(d1, d2).astype(np.float32)
    v.weight[:] = 1
    O.compute_active_set(v)
    cons = node_constraints(v, 3, lambda x: x + 0.01)
    cons = cons[cons["canonical"][:, 0] < 0.55]
    ref = O.NormalEquations(v, Pose.make(), cons, SolverParams.make())
    assert 0 < ref.frozen.sum() < ref.num_rows
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    got = ctx.build_normal_equations(Pose.make(), SolverParams.make())
    assert np.array_equal(got["frozen"], ref.frozen)


def test_assembled_pcg_and_multiply(ctx):
    v = active_sphere_volume(8, 0.07)
    r = O.euler_to_matrix((0.02, -0.03, 0.05))
    cons = rigid_motion_constraints(v, r, (0.02, -0.01, 0.005))
    ref = O.NormalEquations(v, Pose.make(), cons, SolverParams.make())
    x = np.random.default_rng(1).uniform(-1, 1, (ref.num_rows, 3))
    y = ctx.ne_multiply(ref.blocks, ref.cols, x)
    assert np.max(np.abs(y - ref.multiply(x))) <= 1e-12 * np.max(np.abs(y))
    # PCG against a dense solve (test_solver.cpp:98-130)
    xg, it, res = ctx.pcg_solve(ref.blocks, ref.cols, ref.rhs, np.zeros((ref.num_rows, 3)), 1e-12, 4000)
    n = ref.num_rows
    a = np.zeros((3 * n, 3 * n))
    e = np.zeros((n, 3))
    for j in range(3 * n):
        e[j // 3, j % 3] = 1
        a[:, j] = ref.multiply(e).reshape(-1)
        e[j // 3, j % 3] = 0
    xd = np.linalg.solve(a, ref.rhs.reshape(-1))
    assert np.sqrt(np.sum((xg.reshape(-1) - xd) ** 2) / np.sum(xd ** 2)) < 1e-8
    xo, ito, reso = ref.pcg_solve(np.zeros((n, 3)), 1e-12, 4000)
    assert abs(it - ito) <= 2


def test_energy_parity(ctx):
    v = jittered_sphere(euler_amp=0.1)
    cons = np.concatenate([rigid_motion_constraints(v, np.eye(3), (0.01, 0, 0)),
                           random_dense_constraints(v, 200, seed=4)])
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.01, 0.0, 0.02)), (0.0, 0.01, 0.0))
    exp = O.evaluate_energy(v, pose, cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    got = ctx.evaluate_energy(pose, p)
    for k in ("total", "sparse", "dense", "reg"):
        assert got[k] == pytest.approx(exp[k], rel=1e-11, abs=1e-300)


def test_energy_identity_field_is_zero(ctx):  # test_solver.cpp:213-221
    v = active_sphere_volume()
    cons = rigid_motion_constraints(v, np.eye(3), np.zeros(3))
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    e = ctx.evaluate_energy(Pose.make(), SolverParams.make())
    assert e["reg"] == 0.0 and e["total"] < 1e-28


def test_energy_rejects_inactive_anchor(ctx):  # solver.cpp:352-353
    from paper_1603_08161_b200.wfk import WfkError
    v = active_sphere_volume()
    cons = rigid_motion_constraints(v, np.eye(3), np.zeros(3))
    v.active[cons["anchor_index"][0][0]] = 0
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    with pytest.raises(WfkError) as ei:
        ctx.evaluate_energy(Pose.make(), SolverParams.make())
    assert ei.value.code == -3


def test_bad_anchor_layout_rejected(ctx):
    from paper_1603_08161_b200.wfk import WfkError
    v = active_sphere_volume()
    cons = rigid_motion_constraints(v, np.eye(3), np.zeros(3)).copy()
    ctx.upload_volume(v)
    bad = cons[:1].copy()
    bad["anchor_index"][0][3] += 1
    with pytest.raises(WfkError) as ei:
        ctx.upload_constraints(bad)
    assert ei.value.code == -1
    bad = cons[:1].copy()
    bad["anchor_index"][0][:] = v.num_points + 5
    with pytest.raises(WfkError) as ei:
        ctx.upload_constraints(bad)
    assert ei.value.code == -2


def test_update_rotations_parity(ctx):
    v = jittered_sphere(amp=0.01)
    r = O.euler_to_matrix((0.3, -0.2, 0.5))
    v.deformed[:] = (v.canonical_positions() + np.random.default_rng(2).uniform(-0.003, 0.003, (v.num_points, 3))) @ r.T
    ref = v.copy()
    O.update_rotations(ref)
    ctx.upload_volume(v)
    ctx.update_rotations()
    ctx.download_volume(v)
    act = v.active.astype(bool)
    d = np.abs(v.euler[act] - ref.euler[act])
    assert np.max(d) < 1e-11
    assert np.array_equal(v.euler[~act], ref.euler[~act])


def test_rotation_fit_recovers_rigid_motion(ctx):  # test_solver.cpp:144-162
    v = active_sphere_volume()
    r = O.euler_to_matrix((0.3, -0.2, 0.5))
    v.deformed[:] = v.canonical_positions() @ r.T + (0.1, 0.05, -0.07)
    ctx.upload_volume(v)
    ctx.update_rotations()
    ctx.download_volume(v)
    for i in np.nonzero(v.active)[0]:
        assert np.linalg.norm(O.euler_to_matrix(v.euler[i]) - r) < 1e-12


def compare_solves(v_gpu, v_ref, trace_gpu, trace_ref):
    assert len(trace_gpu) == len(trace_ref)
    for a, b in zip(trace_gpu, trace_ref):
        assert a["level"] == b["level"] and a["iteration"] == b["iteration"]
        assert a["energy"]["total"] == pytest.approx(b["energy"]["total"], rel=ENERGY_RTOL)
        assert a["anomaly"] == b["anomaly"]
    act = v_ref.active.astype(bool)
    assert np.array_equal(v_gpu.active, v_ref.active)
    dev = np.max(np.linalg.norm(v_gpu.deformed[act] - v_ref.deformed[act], axis=1)) / v_ref.voxel_size
    assert dev <= POS_TOL_VOXEL, dev


def test_flip_flop_parity(ctx):
    v = jittered_sphere(amp=0.015, seed=24)
    r = O.euler_to_matrix((0.05, -0.08, 0.1))
    t = np.array([0.02, 0.01, -0.015])
    cons = np.concatenate([rigid_motion_constraints(v, r, t), random_dense_constraints(v, 300, seed=5)])
    p = SolverParams.make(flip_flop_iters=6, flip_flop_rel_tol=0.0)
    ref = v.copy()
    tr = O.flip_flop_solve(ref, Pose.make(), cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.flip_flop_solve(Pose.make(), p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)
    # the descent property of test_solver.cpp:224-251
    for a, b in zip(tg, tg[1:]):
        assert b["energy"]["total"] <= a["energy"]["total"] * (1 + 1e-9)


def test_flip_flop_defaults_parity(ctx):
    v = jittered_sphere(n=16, voxel=0.04, amp=0.01, seed=7, euler_amp=0.02)
    cons = random_dense_constraints(v, 600, seed=8, normal_jitter=0.5)
    p = SolverParams.make()
    ref = v.copy()
    tr = O.flip_flop_solve(ref, Pose.make(), cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.flip_flop_solve(Pose.make(), p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)


def test_hierarchy_shape(ctx):  # test_solver.cpp:253-262
    v = active_sphere_volume()
    cons = rigid_motion_constraints(v, O.euler_to_matrix((0, 0.06, -0.04)), (0.015, -0.01, 0.02))
    dims_ref, act_ref, _ = O.hierarchy_info(v, cons, 3)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    dims, act = ctx.hierarchy_info(3)
    assert np.array_equal(dims, dims_ref)
    assert np.array_equal(act, act_ref)


def test_coarse_to_fine_parity(ctx):  # test_solver.cpp:253-272
    v = active_sphere_volume()
    r = O.euler_to_matrix((0, 0.06, -0.04))
    t = np.array([0.015, -0.01, 0.02])
    cons = rigid_motion_constraints(v, r, t)
    p = SolverParams.make(flip_flop_iters=20, pcg_tol=1e-8, pcg_max_iters=500)
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, Pose.make(), cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(Pose.make(), p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)
    for c in cons:
        assert np.linalg.norm(O.warp_point(v, Pose.make(), c["canonical"]) - c["target"]) < 1e-3


def test_coarse_to_fine_bench_fixture(ctx):
    # kernel_bench.cpp:15-29 fixture with dense constraints, default params
    v = make_volume(32)
    cons = random_dense_constraints(v, 2000, seed=9)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(pose, p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)


def test_solve_is_deterministic(ctx):
    v = jittered_sphere(amp=0.015, seed=24)
    cons = random_dense_constraints(v, 300, seed=5)
    p = SolverParams.make()
    out = []
    for _ in range(2):
        w = v.copy()
        ctx.upload_volume(w)
        ctx.upload_constraints(cons)
        tr = ctx.solve_coarse_to_fine(Pose.make(), p)
        ctx.download_volume(w)
        out.append((w.deformed.copy(), w.euler.copy(), [e["energy"]["total"] for e in tr]))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


def test_pipelined_pcg_spill_matches_shared(ctx, monkeypatch):
    """Large lattices keep the pipelined PCG's row state in a global spill
    area instead of shared memory (WFK_PIPE_SPILL forces it): same
    arithmetic, so the same result bit for bit."""
    v = make_volume(32)
    cons = random_dense_constraints(v, 2000, seed=9)
    p = SolverParams.make()
    out = []
    for spill in (None, "full"):
        if spill:
            monkeypatch.setenv("WFK_PIPE_SPILL", spill)
        w = v.copy()
        ctx.upload_volume(w)
        ctx.upload_constraints(cons)
        tr = ctx.solve_coarse_to_fine(Pose.make(), p)
        ctx.download_volume(w)
        out.append((w.deformed.copy(), [e["energy"]["total"] for e in tr]))
    monkeypatch.delenv("WFK_PIPE_SPILL", raising=False)
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


@pytest.mark.parametrize("slabs", [1, 3])
def test_coarse_to_fine_slab_partition_parity(ctx, slabs):
    """solve_coarse_to_fine with every level's PCG partitioned into z-slabs
    (slab states on one GPU) against the oracle"""
    v = make_volume(32)
    cons = random_dense_constraints(v, 2000, seed=9)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine_slabs(slabs, pose, p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)
    assert all(e["pcg_iterations"] > 0 for e in tg)


def test_chronopoulos_gear_variant_parity(ctx, monkeypatch):
    """WFK_PCG=cg forces the Chronopoulos-Gear PCG (the variant chosen when
    the pipelined PCG's row state does not fit shared memory): parity
    against the oracle at the north-star tolerances."""
    v = make_volume(32)
    cons = random_dense_constraints(v, 2000, seed=9)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    monkeypatch.setenv("WFK_PCG", "cg")
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(pose, p)
    ctx.download_volume(v)
    monkeypatch.delenv("WFK_PCG", raising=False)
    compare_solves(v, ref, tg, tr)


def test_frame_solve_determinism_stress(ctx):
    """The reference's race proxy is Serial == Parallel bitwise
    (test_solver.cpp:132-142); the device has no serial mode, so the stand-in
    is run-to-run identity under the persistent kernel's hand-rolled grid
    barrier and split reduction: 50 repeats of one frame's coarse-to-fine solve
    (a configs[2]-sized system: 640x480 dense association against a 128^3
    bootstrap, 3 levels) must produce bit-identical traces and fields."""
    from paper_1603_08161_b200.abi import CorrespondParams, Frame, Intrinsics
    from paper_1603_08161_b200.wfk import pipeline_config
    from tools import synthscene as S
    K = Intrinsics.make(560, 560, 319.5, 239.5, 640, 480)
    sc = S.bend_sphere(K, frames=300, amplitude=2.0, frequency=2.0)
    f0, f1 = (Frame(K, *S.render(sc, f)) for f in (0, 7))
    n = 128
    ctx.create_volume((n, n, n), 0.7 / (n - 1), (-0.35, -0.35, 0.85))
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=1)
    ctx.process_frame(f0, Pose.make(), cfg, 0)
    ctx.checkpoint_volume()
    ctx.upload_frame(f1)
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(Pose.make())
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    assert ctx.find_dense_correspondences(K, CorrespondParams.make(), drop_inactive=True) > 50000
    p = SolverParams.make()
    ref_trace, ref_field = None, None
    v = Volume((n, n, n), 0.7 / (n - 1), (-0.35, -0.35, 0.85))
    for rep in range(50):
        ctx.checkpoint_volume(restore=True)
        tr = ctx.solve_coarse_to_fine(Pose.make(), p)
        ctx.download_volume(v, 1 << 3)  # WFK_VOL_DEFORMED
        if ref_trace is None:
            ref_trace, ref_field = tr, v.deformed.copy()
            continue
        assert tr == ref_trace, rep
        assert np.array_equal(v.deformed, ref_field), rep


def test_fast_precision_cg_parity(ctx, monkeypatch):
    """WFK_PRECISION_FAST (fp32 Krylov vectors in the Chronopoulos-Gear PCG of
    matrix-free levels; fp64 arithmetic, dots, initial residual, x = x0 + d):
    parity by tolerance against the reference -- the north-star bars, 1e-4
    relative energy and 1e-3 voxel (measured at configs[4]: 9e-7, 1.5e-5)."""
    v = make_volume(32)
    cons = random_dense_constraints(v, 3000, seed=13)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    monkeypatch.setenv("WFK_PCG", "cg")  # below 500 K rows the CG variant (and so FAST) must be forced
    ctx.set_precision(1)
    try:
        ctx.upload_volume(v)
        ctx.upload_constraints(cons)
        tg = ctx.solve_coarse_to_fine(pose, p)
        ctx.download_volume(v)
    finally:
        ctx.set_precision(0)
    assert len(tg) == len(tr)
    for a, b in zip(tg, tr):
        assert a["energy"]["total"] == pytest.approx(b["energy"]["total"], rel=1e-4)
    act = ref.active.astype(bool)
    dev = np.max(np.linalg.norm(v.deformed[act] - ref.deformed[act], axis=1)) / v.voxel_size
    assert dev <= 1e-3, dev


@pytest.mark.parametrize("pack", ["1", "0"])
def test_packed_fp64_cg_parity(ctx, monkeypatch, pack):
    """The Chronopoulos-Gear PCG of matrix-free levels in both fp64 storages --
    packed 24-byte xyz vectors (the default, WFK_PACK unset or 1) and 32-byte
    padded ones (WFK_PACK=0) -- against the reference: fp64 throughout, so the
    fp64 parity bars apply."""
    v = make_volume(32)
    cons = random_dense_constraints(v, 3000, seed=13)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    monkeypatch.setenv("WFK_PCG", "cg")
    monkeypatch.setenv("WFK_PACK", pack)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(pose, p)
    ctx.download_volume(v)
    compare_solves(v, ref, tg, tr)


# ---- the slab-partitioned CG inside the persistent kernel ----
def _slab_solve(ctx, monkeypatch, slabs, n=48, ncons=6000):
    v = make_volume(n)
    cons = random_dense_constraints(v, ncons, seed=13)
    p = SolverParams.make()
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    monkeypatch.setenv("WFK_SLABS", str(slabs))
    monkeypatch.setenv("WFK_SLAB_MIN_ROWS", "0")  # partition every matrix-free level of the small fixture
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(pose, p)
    ctx.download_volume(v)
    return v, tg, cons, pose, p


def test_slab_cg_bitwise_across_ranks(ctx, monkeypatch):
    """pcg_slab with S = 1, 2, 4, 8 virtual ranks (block groups of one
    cooperative launch, each with its own u window filled by the neighbours'
    pushes, rank barriers, a rank-ordered all-reduce): block b always owns the
    same rows and every sum runs over block partials in block order, so the
    partitioned solve is bit-identical to the unpartitioned one."""
    base_v, base_t, _, _, _ = _slab_solve(ctx, monkeypatch, 1)
    for s in (2, 4, 8):
        v, t, _, _, _ = _slab_solve(ctx, monkeypatch, s)
        assert np.array_equal(v.deformed, base_v.deformed), s
        assert np.array_equal(v.euler, base_v.euler), s
        assert [e["energy"]["total"] for e in t] == [e["energy"]["total"] for e in base_t], s
        assert [e["pcg_iterations"] for e in t] == [e["pcg_iterations"] for e in base_t], s


def test_slab_cg_parity(ctx, monkeypatch):
    """The slab-partitioned solve (4 ranks) against the reference at the fp64 bars."""
    v, tg, cons, pose, p = _slab_solve(ctx, monkeypatch, 4)
    ref = make_volume(48)
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    compare_solves(v, ref, tg, tr)


def test_slab_partition_skips_small_levels(ctx, monkeypatch):
    """Under WFK_SLABS only matrix-free levels of >= kSlabMinRows (100 K) rows
    are partitioned; the fixture's levels are all smaller, so the solve is the
    fused one, bit for bit."""
    base_v, base_t, _, _, _ = _slab_solve(ctx, monkeypatch, 0)
    monkeypatch.delenv("WFK_SLAB_MIN_ROWS")
    v = make_volume(48)
    cons = random_dense_constraints(v, 6000, seed=13)
    pose = Pose.make(O.euler_to_matrix((0.0, 0.01, 0.0)), (0.005, 0, 0))
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    monkeypatch.setenv("WFK_SLABS", "4")
    t = ctx.solve_coarse_to_fine(pose, SolverParams.make())
    ctx.download_volume(v)
    assert np.array_equal(v.deformed, base_v.deformed)
    assert [e["energy"]["total"] for e in t] == [e["energy"]["total"] for e in base_t]


def test_slab_too_thin_is_rejected(ctx, monkeypatch):
    """A slab thinner than the stencil / constraint halo (here: one block's rows
    per rank) cannot be served by its two neighbours alone: invalid argument."""
    from paper_1603_08161_b200.wfk import WfkError
    with pytest.raises(WfkError):
        _slab_solve(ctx, monkeypatch, 148)
