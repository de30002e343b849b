"""Per-frame device time over the WHOLE BASELINE configs[2] sequence (300 frames),
not just bench.py's early window: same scene, lattice, parameters and timing
rule as bench.py's `value` (frames staged in HBM, L2 flushed before every
frame, CUDA events on the context stream).  Reports ms/frame over the early,
middle and late thirds plus the sizes that grow with the sequence (sparse
constraints, feature matches, feature-store entries) and the per-stage split
(wfk_profile: maps_mesh_raster = back-projection, mesh, raster, ICP and the
feature detection + matching; associate; solve; redeform; fuse = fusion,
expansion and the feature-store update).

    python tools/sequence_timing.py [--frames 300] [--out gpurun_out/sequence_timing.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=bench.FRAMES_TOTAL)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sequence_timing.json"))
    a = ap.parse_args()

    from paper_1603_08161_b200.abi import Intrinsics, Pose, SolverParams, Volume
    from paper_1603_08161_b200.wfk import Context, pipeline_config

    ctx = Context(0)
    K = Intrinsics.make(bench.FX, bench.FY, bench.CX, bench.CY, bench.W_PX, bench.H_PX)
    frames = bench.render_frames(K, range(a.frames), pinned=True)
    dims, voxel, origin = bench.lattice_geometry()
    ctx.upload_volume(Volume(dims, voxel, origin))
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=3)
    for f in range(1, a.frames):
        ctx.stage_frame(f, frames[f])
    pose = Pose.make()
    rec0 = ctx.process_frame(frames[0], pose, cfg, 0)
    assert rec0.bootstrap == 1
    store = int(rec0.features_added)
    rows = []
    ctx.profile_enable(True)
    prev = dict(ctx.profile_read().as_dict()["stage_ms"])
    for f in range(1, a.frames):
        ctx.flush_l2()
        ctx.timer_mark(0)
        r = ctx.process_staged_frame(f, pose, cfg, f)
        ctx.timer_mark(1)
        pose = r.pose
        store += int(r.features_added)
        cur = dict(ctx.profile_read().as_dict()["stage_ms"])
        stages = {k: round(cur[k] - prev[k], 4) for k in cur}
        prev = cur
        rows.append({"frame": f, "ms": round(ctx.timer_elapsed_ms(0, 1), 4), "stage_ms": stages,
                     "dense": int(r.dense_count),
                     "sparse": int(r.sparse_count), "matches": int(r.match_count), "store": store,
                     "pcg_iterations": int(r.pcg_iterations)})
    store_dev = int(len(ctx.feature_store()))
    ctx.close()

    def window(lo, hi):
        sel = [x for x in rows if lo <= x["frame"] <= hi]
        if not sel:
            return None
        ms = np.array([x["ms"] for x in sel])
        return {"frames": [lo, min(hi, sel[-1]["frame"])], "mean_ms": float(ms.mean()),
                "median_ms": float(np.median(ms)), "max_ms": float(ms.max()),
                "sparse_mean": float(np.mean([x["sparse"] for x in sel])),
                "matches_mean": float(np.mean([x["matches"] for x in sel])),
                "store_at_end": sel[-1]["store"],
                "stage_ms": {k: float(np.mean([x["stage_ms"][k] for x in sel])) for k in sel[0]["stage_ms"]}}

    third = a.frames // 3
    out = {"workload": "BASELINE configs[2] (bench.py scene / lattice / parameters), every frame of the sequence",
           "timing": "CUDA events on the context stream, frames staged in HBM, L2 flushed before each frame",
           "frames_timed": len(rows),
           "all": window(1, a.frames - 1),
           # frame 1 is the context's first solve (allocations, stream / module
           # first use): reported alone and left out of this summary
           "first_frame_ms": rows[0]["ms"] if rows else None,
           "all_after_first": window(2, a.frames - 1),
           "early": window(1, third - 1), "middle": window(third, 2 * third - 1),
           "late": window(2 * third, a.frames - 1),
           "bench_window": window(4, 23),
           "feature_store_device": store_dev,
           "per_frame": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "per_frame"}))


if __name__ == "__main__":
    main()
