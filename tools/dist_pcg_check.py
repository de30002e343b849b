"""Multi-GPU check of the slab-partitioned PCG over NCCL (one process per GPU):

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
      --master-addr 127.0.0.1 --master-port 29511 tools/dist_pcg_check.py [n]

Every rank builds the same normal equations (oracle, n^3 sphere lattice),
rank 0 creates the NCCL id and shares it through torch.distributed (gloo),
each rank solves its z-slab with wfk_pcg_solve_dist, and rank 0 compares the
gathered x with the single-GPU wfk_pcg_solve and reports the time per
iteration (CUDA-synchronised wall clock around the solve, max over ranks).
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O  # noqa: E402  (builds the test system)
from paper_1603_08161_b200 import wfk  # noqa: E402
from paper_1603_08161_b200.abi import Pose, SolverParams  # noqa: E402
from tests.fixtures import active_sphere_volume, rigid_motion_constraints  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    v = active_sphere_volume(n, 0.6 / n, 0.25)
    cons = rigid_motion_constraints(v, O.euler_to_matrix((0.02, -0.03, 0.05)), (0.02, -0.01, 0.005))
    ne = O.NormalEquations(v, Pose.make(), cons, SolverParams.make())
    idt = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        idt[:] = torch.frombuffer(bytearray(wfk.dist_unique_id()), dtype=torch.uint8)
    dist.broadcast(idt, 0)
    c = wfk.Context(local)
    c.dist_init(rank, world, bytes(idt.tolist()))
    x0 = np.zeros((ne.num_rows, 3))
    c.pcg_solve_dist(ne.blocks, ne.cols, ne.rhs, x0, 0.0, 5)  # warm-up
    dist.barrier()
    t0 = time.perf_counter()
    x, it, res = c.pcg_solve_dist(ne.blocks, ne.cols, ne.rhs, x0, 0.0, 50)
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    if rank == 0:
        xs, its, _ = c.pcg_solve(ne.blocks, ne.cols, ne.rhs, x0, 0.0, 50)
        err = float(np.max(np.abs(x - xs)) / max(np.max(np.abs(xs)), 1e-300))
        print(f"rows {ne.num_rows} world {world}: iterations {it} (single {its}), max rel diff {err:.2e}, "
              f"{dt.item() * 1e3:.2f} ms per solve incl. the system upload")
    c.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
