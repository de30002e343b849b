"""Small workload for compute-sanitizer (memcheck / initcheck / racecheck /
synccheck, where offered) and for libwfk's checked mode (WFK_CHECK=1,
tests/test_gpu_checked.py): one coarse-to-fine flip-flop solve on a 12^3 jittered sphere
(pipelined PCG, and the Chronopoulos-Gear variant when WFK_PCG=cg), one
fusion step, and one 32^3 process_frame (association, ICP, features, solve,
fusion).  Run by tools/sanitize.sh; exits non-zero on a parity failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import pyoracle as O  # noqa: E402
from paper_1603_08161_b200.abi import FusionParams, Pose, SolverParams  # noqa: E402
from paper_1603_08161_b200.wfk import Context  # noqa: E402
from tests.fixtures import active_sphere_volume, plane_frame, random_dense_constraints  # noqa: E402


def main():
    ctx = Context(0)
    v = active_sphere_volume(12, 0.05)
    rng = O.Rng(21)
    for i in range(v.num_points):
        v.deformed[i] += rng.vec3(-0.02, 0.02)
    cons = random_dense_constraints(v, 300, seed=5)
    p = SolverParams.make()
    ref = v.copy()
    tr = O.solve_coarse_to_fine(ref, Pose.make(), cons, p)
    ctx.upload_volume(v)
    ctx.upload_constraints(cons)
    tg = ctx.solve_coarse_to_fine(Pose.make(), p)
    ctx.download_volume(v)
    e_g, e_r = tg[-1]["energy"]["total"], tr[-1]["energy"]["total"]
    assert abs(e_g - e_r) <= 1e-4 * abs(e_r), (e_g, e_r)
    fr = plane_frame(1.3, 90.0)
    ctx.upload_frame(fr)
    ctx.integrate_frame(Pose.make(), FusionParams.make(bootstrap=1))
    if os.environ.get("SAN_PIPELINE", "1") == "1":
        from paper_1603_08161_b200.abi import Intrinsics, Volume
        from paper_1603_08161_b200.wfk import pipeline_config
        n, voxel, origin = 32, 0.7 / 31, (-0.35, -0.35, 0.85)
        K = Intrinsics.make(280, 280, 159.5, 119.5, 320, 240)
        vol = Volume((n, n, n), voxel, origin)
        ctx.upload_volume(vol)
        from paper_1603_08161_b200.abi import Frame
        cfg = pipeline_config(solver=SolverParams.make(levels=2), reassociations=1)
        pose = Pose.make()
        for f in range(2):
            d, c = O.synth_render(K, amplitude=0.3 * f)
            pose = ctx.process_frame(Frame(K, d, c), pose, cfg, f).pose
    ctx.close()
    print("sanitize fixture OK", flush=True)


if __name__ == "__main__":
    main()
