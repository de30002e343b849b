"""bench.py's multi-process plumbing on CPU (gloo, world_size 2).

The 128^3 workload runs as independent replicas per GPU;
the only collectives are the timing reductions.  These tests run the same Dist
class with the gloo backend in two processes and check the reductions and the
whole-job ms/frame aggregation the driver's scaling numbers are computed from.
"""
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench

    d = bench.Dist(world, backend="gloo")
    try:
        assert d.world == world and d.rank == rank
        d.barrier()
        res = {
            "max": d.max(float(rank + 1)),
            "sum": d.sum(float(rank + 1)),
            # rank r timed 100 (r + 1) ms over 10 frames
            "job": d.whole_job_ms_per_frame(100.0 * (rank + 1), 10),
        }
        out.put((rank, res))
    finally:
        d.close()


@pytest.mark.timeout(180)
def test_dist_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=150) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert got[r]["max"] == 2.0
        assert got[r]["sum"] == 3.0
        # slowest rank 200 ms for 10 frames, 20 frames in the whole job
        assert got[r]["job"] == pytest.approx(10.0)


def test_dist_single_process_is_identity():
    sys.path.insert(0, ROOT)
    import bench

    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        os.environ.pop(k, None)
    d = bench.Dist(1, backend="gloo")
    assert d.world == 1 and d.max(3.5) == 3.5 and d.sum(2.0) == 2.0
    assert d.whole_job_ms_per_frame(50.0, 10) == 5.0
