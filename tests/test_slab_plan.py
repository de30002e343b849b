"""The in-kernel slab partition of the matrix-free CG (pcg_slab, WFK_SLABS;
SURVEY.md 8(e)) on the CPU.

The device kernel runs the ranks as block groups of one cooperative launch;
what makes it a multi-GPU design is its plan and its protocol, and those are
what these tests exercise across real process boundaries:
  * the host plan (`wfk_slab_plan`, libwfk's own code): tiles of about equal
    work and the rank split into contiguous, equal tile ranges;
  * each rank's u window (its rows plus the rows its rows' stencil reaches)
    lies within its two neighbours' rows;
  * the per-iteration protocol over two gloo processes: a rank updates only
    its rows, pushes the rows a neighbour's window covers to that neighbour,
    applies A to its rows from its window, and every dot product is summed per
    tile and then over all tiles in tile order -- so the iterates are
    bit-identical to the single-rank run.
The per-rank arithmetic is numpy on the oracle's explicit normal equations
(the same Chronopoulos-Gear recurrences as pcg_slab); the GPU tests
(tests/test_gpu_solver.py::test_slab_cg_*) check the kernel itself.
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
BLOCKS, THREADS = 16, 32   # a small virtual grid: 16 x clamp(N / 512, 1, 8) tiles


def system(n=12, voxel=0.05):
    v = active_sphere_volume(n, voxel)
    r = O.euler_to_matrix((0.02, -0.03, 0.05))
    cons = rigid_motion_constraints(v, r, (0.02, -0.01, 0.005))
    return O.NormalEquations(v, Pose.make(), cons, SolverParams.make())


def row_work(cols):
    return (12 + (cols >= 0).sum(1)).astype(np.int32)


def windows(cols, lo):
    """rank s's u window: [min, max] of the rows its rows reference"""
    S = len(lo) - 1
    out = []
    for s in range(S):
        ref = cols[lo[s]:lo[s + 1]]
        ref = ref[ref >= 0]
        out.append((min(lo[s], int(ref.min())) if ref.size else lo[s],
                    max(lo[s + 1], int(ref.max()) + 1) if ref.size else lo[s + 1]))
    return out


def plan(cols, ranks):
    tr, rt = wfk.slab_plan(row_work(cols), BLOCKS, THREADS, ranks)
    lo = [int(tr[t]) for t in rt]
    return tr, rt, lo, windows(cols, lo)


@pytest.mark.parametrize("ranks", [1, 2, 3, 4])
def test_plan_split_and_windows(ranks):
    ne = system()
    cols = ne.cols
    n = len(cols)
    tr, rt, lo, win = plan(cols, ranks)
    ntiles = len(tr) - 1
    assert ntiles % BLOCKS == 0 and BLOCKS <= ntiles <= 8 * BLOCKS
    assert tr[0] == 0 and tr[-1] == n and np.all(np.diff(tr) >= 0)
    assert rt[0] == 0 and rt[-1] == ntiles and np.all(np.diff(rt) >= 1)
    # tiles of about equal work: within one row's work of the mean
    w = row_work(cols)
    tw = np.array([int(w[tr[t]:tr[t + 1]].sum()) for t in range(ntiles)])
    assert tw.max() - tw.min() <= 2 * int(w.max())
    for s, (a, b) in enumerate(win):
        assert a >= (lo[s - 1] if s > 0 else 0), "halo beyond the lower neighbour"
        assert b <= (lo[s + 2] if s + 2 <= ranks else n), "halo beyond the upper neighbour"


def test_plan_rejects_bad_arguments():
    with pytest.raises(wfk.WfkError):
        wfk.slab_plan(np.full(64, 12, np.int32), 4, 32, 5)   # more ranks than blocks


def _apply(blocks, cols, v_of, r0, r1):
    """rows r0..r1 of A v, v given through the rank's window accessor"""
    out = np.zeros((r1 - r0, 3))
    for s in range(27):
        c = cols[r0:r1, s]
        m = c >= 0
        if m.any():
            out[m] += np.einsum("rij,rj->ri", blocks[r0:r1, s][m], v_of(c[m]))
    return out


def slab_cg(ne, ranks, rank, comm, iters):
    """pcg_slab's recurrences for rank `rank` of `ranks`; comm: (push, gather)
    callbacks (None for a single rank).  Returns (d of own rows, lo, hi)."""
    blocks, cols, rhs = ne.blocks, ne.cols, ne.rhs
    n = len(cols)
    tr, rt, lo_all, win = plan(cols, ranks)
    lo, hi = lo_all[rank], lo_all[rank + 1]
    wlo, whi = win[rank]
    ntiles = len(tr) - 1
    my_tiles = range(rt[rank], rt[rank + 1])
    u_win = np.zeros((whi - wlo, 3))            # own rows + halo
    u_of = lambda idx: u_win[idx - wlo]          # noqa: E731
    diag = np.stack([np.diagonal(blocks[:, 13], axis1=1, axis2=2)], 0)[0]
    dinv = np.where(diag > 1e-300, 1.0 / np.where(diag > 1e-300, diag, 1.0), 1.0)
    r = np.zeros((n, 3))
    p = np.zeros((n, 3))
    s_ = np.zeros((n, 3))
    d = np.zeros((n, 3))
    w = np.zeros((n, 3))

    def tile_sums(terms):  # terms[j] : (n,) per-row values of own rows
        part = np.zeros((ntiles, len(terms)))
        for t in my_tiles:
            a, b = tr[t], tr[t + 1]
            for j, v in enumerate(terms):
                part[t, j] = np.sum(v[a:b])
        if comm is not None:
            part = comm[1](part)                  # every rank's tiles
        tot = np.zeros(len(terms))
        for t in range(ntiles):                   # tile order
            tot = tot + part[t]
        return tot

    def push():
        if comm is not None:
            comm[0](u_win, lo, hi, wlo, win)

    def matvec():
        w[lo:hi] = _apply(blocks, cols, u_of, lo, hi)

    # x0 = 0: r0 = b, u0 = D r0
    r[lo:hi] = rhs[lo:hi]
    u_win[lo - wlo:hi - wlo] = dinv[lo:hi] * r[lo:hi]
    ru = np.zeros(n)
    rr = np.zeros(n)
    bb = np.zeros(n)
    uu = u_win[lo - wlo:hi - wlo]
    ru[lo:hi] = np.sum(r[lo:hi] * uu, 1)
    rr[lo:hi] = np.sum(r[lo:hi] ** 2, 1)
    bb[lo:hi] = np.sum(rhs[lo:hi] ** 2, 1)
    push()
    matvec()
    wu = np.zeros(n)
    wu[lo:hi] = np.sum(w[lo:hi] * uu, 1)
    gamma, delta, rsq, bsq = tile_sums([ru, wu, rr, bb])
    gamma_prev = alpha_prev = 0.0
    for it in range(iters):
        beta = 0.0 if it == 0 else gamma / gamma_prev
        pap = delta if it == 0 else delta - beta * gamma / alpha_prev
        alpha = gamma / pap
        u_own = u_win[lo - wlo:hi - wlo].copy()
        p[lo:hi] = u_own + beta * p[lo:hi]
        s_[lo:hi] = w[lo:hi] + beta * s_[lo:hi]
        d[lo:hi] = d[lo:hi] + alpha * p[lo:hi]
        r[lo:hi] = r[lo:hi] - alpha * s_[lo:hi]
        u_win[lo - wlo:hi - wlo] = dinv[lo:hi] * r[lo:hi]
        uu = u_win[lo - wlo:hi - wlo]
        ru[lo:hi] = np.sum(r[lo:hi] * uu, 1)
        rr[lo:hi] = np.sum(r[lo:hi] ** 2, 1)
        push()
        matvec()
        wu[lo:hi] = np.sum(w[lo:hi] * uu, 1)
        gamma_prev, alpha_prev = gamma, alpha
        gamma, delta, rsq = tile_sums([ru, wu, rr])
    return d[lo:hi].copy(), lo, hi


def _rank_main(rank, world, port, ne_arrays, iters, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    class NE:
        pass

    ne = NE()
    ne.blocks, ne.cols, ne.rhs = ne_arrays
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def push(u_win, lo, hi, wlo, win):
            # rows of my range that a neighbour's window covers go to it;
            # the neighbour's rows my window covers come from it
            reqs = []
            for nb in (rank - 1, rank + 1):
                if 0 <= nb < world:
                    a, b = max(lo, win[nb][0]), min(hi, win[nb][1])
                    if b > a:
                        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(u_win[a - wlo:b - wlo])), nb))
            for nb in (rank - 1, rank + 1):
                if 0 <= nb < world:
                    _, _, lo_all, _ = plan(ne.cols, world)
                    a, b = max(lo_all[nb], win[rank][0]), min(lo_all[nb + 1], win[rank][1])
                    if b > a:
                        buf = torch.zeros((b - a, 3), dtype=torch.float64)
                        dist.recv(buf, nb)
                        u_win[a - wlo:b - wlo] = buf.numpy()
            for q in reqs:
                q.wait()

        def gather(part):
            t = torch.from_numpy(np.ascontiguousarray(part))
            g = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(g, t)
            full = np.zeros_like(part)
            for q in range(world):
                full += g[q].numpy()    # each tile is non-zero on exactly one rank
            return full

        out.put((rank,) + slab_cg(ne, world, rank, (push, gather), iters))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_cg_gloo_bit_identical(world):
    import multiprocessing as mp

    ne = system()
    iters = 25
    d1, lo1, hi1 = slab_cg(ne, 1, 0, None, iters)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, (ne.blocks, ne.cols, ne.rhs), iters, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    d = np.zeros_like(d1)
    for _, dr, lo, hi in res:
        d[lo:hi] = dr
    assert np.array_equal(d, d1)   # bit-identical to the single-rank run
    # the same Krylov iterate as the reference's PCG after the same number of
    # iterations (solver.cpp:282-343; equal in exact arithmetic)
    x_ref, it_ref, _ = ne.pcg_solve(np.zeros((ne.num_rows, 3)), 0.0, iters)
    assert it_ref == iters
    assert np.max(np.abs(d - x_ref)) <= 1e-8 * np.max(np.abs(x_ref))
