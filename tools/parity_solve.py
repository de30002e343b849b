"""Parity of one frame-1 coarse-to-fine solve at a BASELINE solve config
(configs[3] 256^3 or configs[4] 512^3 / 1280x720 room + sphere, bench.py
--solve-config): the device solve (wfk_solve_coarse_to_fine) against the
reference's own solve_coarse_to_fine (oracle/_ref, unmodified sources, OpenMP)
on the same volume state (downloaded after the bootstrap frame) and the same
constraints (the device association, bit-exact with the reference's by the
kernel tests).  Too slow for the test suite at 512^3 (the reference takes
minutes and ~40 GB of host memory); run by hand on the GPU box:

    python tools/parity_solve.py 4 > profiles/r02_parity_config4.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(cfg_id: int):
    import bench
    from oracle import pyoracle as O
    from paper_1603_08161_b200.abi import CorrespondParams, Frame, Intrinsics, Pose, SolverParams, Volume
    from paper_1603_08161_b200.wfk import Context, pipeline_config
    from tools import synthscene as S
    c = bench.SOLVE_CONFIGS[cfg_id]
    n = c["n"]
    K = Intrinsics.make(*c["K"])
    if c["scene"] == "room":
        sc, idx = S.room_corner(K, frames=30, sphere_radius=0.12), [0, 1]
    else:
        sc, idx = S.bend_sphere(K, frames=bench.FRAMES_TOTAL, amplitude=bench.AMPLITUDE,
                                frequency=bench.FREQUENCY), [3, 4]
    frames = [Frame(K, *S.render(sc, f)) for f in idx]
    ctx = Context(0)
    if os.environ.get("WF_FAST"):
        ctx.set_precision(1)  # WFK_PRECISION_FAST
    ctx.create_volume((n, n, n), c["voxel"], c["origin"])
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=1)
    ctx.process_frame(frames[0], Pose.make(), cfg, 0)
    ctx.checkpoint_volume()
    pose = ctx.process_frame(frames[1], Pose.make(), cfg, 1).pose
    ctx.checkpoint_volume(restore=True)
    ctx.upload_frame(frames[1])
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(pose)
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    n_cons = ctx.find_dense_correspondences(K, CorrespondParams.make(), drop_inactive=True)
    cons = ctx.download_constraints()
    vol = Volume((n, n, n), c["voxel"], c["origin"])
    ctx.download_volume(vol)
    p = SolverParams.make()
    t0 = time.perf_counter()
    tg = ctx.solve_coarse_to_fine(pose, p)
    t_gpu = time.perf_counter() - t0
    ref = vol.copy()
    ctx.download_volume(vol)
    ctx.close()
    t0 = time.perf_counter()
    tr = O.solve_coarse_to_fine(ref, pose, cons, p)
    t_ref = time.perf_counter() - t0
    act = ref.active.astype(bool)
    dev = float(np.max(np.linalg.norm(vol.deformed[act] - ref.deformed[act], axis=1)) / c["voxel"])
    e_rel = [abs(a["energy"]["total"] - b["energy"]["total"]) / abs(b["energy"]["total"]) for a, b in zip(tg, tr)]
    out = {"config": c["desc"], "checker": O.backend(), "dense_constraints": int(n_cons),
           "active_nodes": int(act.sum()), "trace_len": [len(tg), len(tr)],
           "pcg_iterations": [sum(e["pcg_iterations"] for e in tg), sum(e["pcg_iterations"] for e in tr)],
           "worst_energy_rel": max(e_rel), "final_energy": [tg[-1]["energy"]["total"], tr[-1]["energy"]["total"]],
           "deformation_dev_voxel": dev, "gpu_solve_s_incl_sync": t_gpu, "reference_solve_s": t_ref,
           "reference_threads": int(O.lib().wfo_num_threads()),
           "precision": "fast" if os.environ.get("WF_FAST") else "fp64",
           "env": {k: v for k, v in os.environ.items() if k.startswith("WFK_")}}
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
