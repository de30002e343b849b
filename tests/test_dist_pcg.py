"""The slab partition of the PCG (paper_1603_08161_b200/csrc/dist.cu).

CPU: the partition plan (`wfk_dist_plan`, host code of libwfk) on the
reference's own normal equations (built by the oracle), and the partitioned
iteration orchestrated over two gloo processes -- each rank applies the
operator to its slab only, receives exactly the halo rows the plan lists from
their owners and all-gathers its partial dots, summed in rank order.  The
per-rank arithmetic in that test is a numpy stand-in for the device kernels;
the point is that the plan's halo is sufficient and the rank-ordered
reductions reproduce the single-process PCG.
GPU (`-m gpu`): `wfk_pcg_solve_slabs` runs the same kernels and plan with
1-4 slab states on one B200 and matches `wfk_pcg_solve` / the oracle;
`wfk_pcg_solve_dist` at world 1.
"""
import os
import socket
import sys

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1603_08161_b200 import wfk
from paper_1603_08161_b200.abi import Pose, SolverParams
from tests.fixtures import active_sphere_volume, rigid_motion_constraints

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def system(n=10, voxel=0.06):
    v = active_sphere_volume(n, voxel)
    r = O.euler_to_matrix((0.02, -0.03, 0.05))
    cons = rigid_motion_constraints(v, r, (0.02, -0.01, 0.005))
    return v, O.NormalEquations(v, Pose.make(), cons, SolverParams.make())


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7])
def test_plan_covers_every_referenced_row(world):
    v, ne = system()
    cols = ne.cols
    ranges, xf = wfk.dist_plan(cols, world)
    n = len(cols)
    assert ranges[0, 0] == 0 and ranges[-1, 1] == n
    assert np.all(ranges[1:, 0] == ranges[:-1, 1])
    owner = np.zeros(n, np.int32)
    for k, (lo, hi) in enumerate(ranges):
        owner[lo:hi] = k
    for k, (lo, hi) in enumerate(ranges):
        ref = cols[lo:hi].reshape(-1)
        need = np.unique(ref[(ref >= 0) & ((ref < lo) | (ref >= hi))])
        got = np.zeros(n, bool)
        for src, dst, a, b in xf:
            if dst == k:
                assert src != k and np.all(owner[a:b] == src)  # sent by the owner
                assert not got[a:b].any()                      # at most once
                got[a:b] = True
        assert got[need].all(), f"rank {k} misses halo rows"


def test_plan_halo_is_adjacent_planes():
    """rows are in lattice order: a slab's halo lies within one z-plane of it"""
    v, ne = system()
    nx, ny, _ = v.dims
    plane = nx * ny
    z = ne.rows // plane
    ranges, xf = wfk.dist_plan(ne.cols, 3)
    for src, dst, a, b in xf:
        lo, hi = ranges[dst]
        assert z[a:b].min() >= z[lo] - 1 and z[a:b].max() <= z[hi - 1] + 1


def _pcg_rank(rank, world, port, blocks, cols, rhs, tol, max_iters, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_1603_08161_b200 import wfk as W

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ranges, xf = W.dist_plan(cols, world)
        lo, hi = ranges[rank]
        n = len(cols)
        A = blocks  # (n, 27, 3, 3)

        def apply(v, r0, r1):  # rows r0..r1 of A v
            out_ = np.zeros((r1 - r0, 3))
            for s in range(27):
                c = cols[r0:r1, s]
                m = c >= 0
                out_[m] += np.einsum("rij,rj->ri", A[r0:r1, s][m], v[c[m]])
            return out_

        def exchange(v):  # the plan's halo transfers, point to point
            reqs = []
            for src, dst, a, b in xf:
                if src == rank:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(v[a:b])), dst))
            for src, dst, a, b in xf:
                if dst == rank:
                    buf = torch.zeros((b - a, 3), dtype=torch.float64)
                    dist.recv(buf, src)
                    v[a:b] = buf.numpy()
            for q in reqs:
                q.wait()

        def gsum(vals):  # all-gather the partials, sum in rank order
            t = torch.tensor(vals, dtype=torch.float64)
            g = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(g, t)
            acc = np.zeros(len(vals))
            for q in range(world):
                acc = acc + g[q].numpy()
            return acc

        x = np.zeros((n, 3))
        d = np.stack([np.diagonal(A[:, 13], axis1=1, axis2=2)], 0)[0]
        dinv = np.where(d > 1e-300, 1.0 / np.where(d > 1e-300, d, 1.0), 1.0)
        r = np.zeros((n, 3))
        p = np.zeros((n, 3))
        r[lo:hi] = rhs[lo:hi] - apply(x, lo, hi)
        z = dinv * r
        p[lo:hi] = z[lo:hi]
        rz, rr, bb = gsum([np.sum(r[lo:hi] * z[lo:hi]), np.sum(r[lo:hi] ** 2), np.sum(rhs[lo:hi] ** 2)])
        rnorm, bnorm = np.sqrt(rr), np.sqrt(bb)
        stop = max(tol * rnorm, 1e-13 * bnorm)
        exchange(p)
        it = 0
        while it < max_iters and rnorm > stop:
            ap = apply(p, lo, hi)
            (pap,) = gsum([np.sum(p[lo:hi] * ap)])
            if pap <= 0:
                break
            alpha = rz / pap
            x[lo:hi] += alpha * p[lo:hi]
            r[lo:hi] -= alpha * ap
            z[lo:hi] = dinv[lo:hi] * r[lo:hi]
            rz_new, rr = gsum([np.sum(r[lo:hi] * z[lo:hi]), np.sum(r[lo:hi] ** 2)])
            beta = rz_new / rz
            rz = rz_new
            p[lo:hi] = z[lo:hi] + beta * p[lo:hi]
            exchange(p)
            rnorm = np.sqrt(rr)
            it += 1
        out.put((rank, it, x[lo:hi].copy(), lo, hi))
    finally:
        dist.destroy_process_group()


def test_partitioned_pcg_gloo_world2():
    import multiprocessing as mp

    v, ne = system()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_pcg_rank, args=(r, 2, port, ne.blocks, ne.cols, ne.rhs, 1e-10, 500, q))
          for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]  # identical scalars on both ranks: same iteration count
    x = np.zeros((ne.num_rows, 3))
    for _, _, xs, lo, hi in res:
        x[lo:hi] = xs
    xo, ito, _ = ne.pcg_solve(np.zeros((ne.num_rows, 3)), 1e-10, 500)
    assert abs(res[0][1] - ito) <= 2
    assert np.max(np.abs(x - xo)) <= 1e-7 * np.max(np.abs(xo))


@pytest.mark.gpu
@pytest.mark.parametrize("slabs", [1, 2, 3, 4])
def test_slab_pcg_matches_single(slabs):
    c = wfk.Context(0)
    try:
        v, ne = system(12, 0.05)
        x0 = np.zeros((ne.num_rows, 3))
        xs, its, ress = c.pcg_solve(ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        xd, itd, resd = c.pcg_solve_slabs(slabs, ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        assert abs(itd - its) <= 1
        assert np.max(np.abs(xd - xs)) <= 1e-8 * np.max(np.abs(xs))
        xo, ito, _ = ne.pcg_solve(np.zeros((ne.num_rows, 3)), 1e-10, 500)
        assert abs(itd - ito) <= 2
        # fixed work: the same number of iterations whatever the partition
        xf, itf, _ = c.pcg_solve_slabs(slabs, ne.blocks, ne.cols, ne.rhs, x0, 0.0, 25)
        x1, it1, _ = c.pcg_solve_slabs(1, ne.blocks, ne.cols, ne.rhs, x0, 0.0, 25)
        assert itf == it1 == 25
        assert np.max(np.abs(xf - x1)) <= 1e-10 * np.max(np.abs(x1))
    finally:
        c.close()


@pytest.mark.gpu
def test_dist_pcg_world1():
    c = wfk.Context(0)
    try:
        c.dist_init(0, 1)
        v, ne = system(12, 0.05)
        x0 = np.zeros((ne.num_rows, 3))
        xs, its, _ = c.pcg_solve_slabs(1, ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        xd, itd, _ = c.pcg_solve_dist(ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        assert itd == its and np.array_equal(xd, xs)
    finally:
        c.close()


@pytest.mark.gpu
def test_dist_pcg_nccl_world1():
    """the NCCL transport (dlopen'd libnccl, all-gather / broadcast) on a 1-rank communicator"""
    c = wfk.Context(0)
    try:
        c.dist_init(0, 1, wfk.dist_unique_id())
        v, ne = system(12, 0.05)
        x0 = np.zeros((ne.num_rows, 3))
        xs, its, _ = c.pcg_solve_slabs(1, ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        xd, itd, _ = c.pcg_solve_dist(ne.blocks, ne.cols, ne.rhs, x0, 1e-10, 500)
        assert itd == its and np.array_equal(xd, xs)
    finally:
        c.close()


def test_plan_more_ranks_than_rows():
    cols = -np.ones((3, 27), np.int32)
    for r in range(3):
        cols[r, 13] = r
        if r > 0:
            cols[r, 12] = r - 1
        if r < 2:
            cols[r, 14] = r + 1
    ranges, xf = wfk.dist_plan(cols, 5)
    assert ranges[0, 0] == 0 and ranges[-1, 1] == 3 and np.all(ranges[:, 1] >= ranges[:, 0])
    for src, dst, a, b in xf:
        assert ranges[src, 0] <= a < b <= ranges[src, 1]


def chain_system(n=10, seed=2):
    """an SPD 1-D chain: 4 I on the diagonal, -I to each neighbour"""
    cols = -np.ones((n, 27), np.int32)
    blocks = np.zeros((n, 27, 3, 3))
    for r in range(n):
        cols[r, 13] = r
        blocks[r, 13] = 4 * np.eye(3)
        if r > 0:
            cols[r, 12] = r - 1
            blocks[r, 12] = -np.eye(3)
        if r < n - 1:
            cols[r, 14] = r + 1
            blocks[r, 14] = -np.eye(3)
    rhs = np.random.default_rng(seed).normal(size=(n, 3))
    return blocks, cols, rhs


@pytest.mark.gpu
def test_slab_pcg_more_slabs_than_rows():
    c = wfk.Context(0)
    try:
        blocks, cols, rhs = chain_system(10)
        x0 = np.zeros((10, 3))
        xs, its, _ = c.pcg_solve(blocks, cols, rhs, x0, 1e-12, 200)
        xd, itd, _ = c.pcg_solve_slabs(13, blocks, cols, rhs, x0, 1e-12, 200)
        assert abs(itd - its) <= 1
        assert np.max(np.abs(xd - xs)) <= 1e-9 * np.max(np.abs(xs))
    finally:
        c.close()
