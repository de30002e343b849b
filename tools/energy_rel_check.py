import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import pyoracle as O
from paper_1603_08161_b200.abi import Intrinsics, Pose, SolverParams, Volume
from paper_1603_08161_b200.wfk import Context, pipeline_config
from tests.test_gpu_pipeline import bend_frames
ctx = Context(0)
for (n, W, H, f, nf, tot, solver, feats, re) in [
    (32, 320, 240, 280, 10, 10, SolverParams.make(levels=1, flip_flop_iters=5, flip_flop_rel_tol=0.0, pcg_max_iters=10, pcg_tol=0.0), False, 1),
    (64, 640, 480, 560, 4, 60, SolverParams.make(), True, 3),
    (128, 640, 480, 560, 3, 300, SolverParams.make(), True, 3)]:
    K = Intrinsics.make(f, f, (W - 1) / 2, (H - 1) / 2, W, H)
    voxel = 0.7 / (n - 1); origin = (-0.35, -0.35, 0.85)
    frames = bend_frames(ctx, K, nf, 1.0 if n == 32 else 2.0, frames_total=tot)
    ref = O.Reconstructor((n, n, n), voxel, origin, solver=solver, reassociations=re, use_features=feats)
    vol = Volume((n, n, n), voxel, origin); ctx.upload_volume(vol)
    cfg = pipeline_config(solver=solver, reassociations=re, use_features=feats)
    pose = Pose.make(); out = []
    for i, fr in enumerate(frames):
        rr = ref.process_frame(fr); rg = ctx.process_frame(fr, pose, cfg, i); pose = rg.pose
        if i: out.append(abs(rg.energy.total - rr.energy.total) / abs(rr.energy.total))
    print(n, ["%.1e" % x for x in out])
