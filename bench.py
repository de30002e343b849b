#!/usr/bin/env python
"""Benchmark of the VolumeDeform hot path on B200 (BASELINE.json metric:
"non-rigid solve ms/frame & PCG iters/s at named lattice; HBM GB/s vs peak").

Workload (BASELINE.json configs[2], concrete form in SURVEY.md 8(d) row 3):
640x480 depth, 128^3 deformation lattice, 3-level coarse-to-fine flip-flop
solve + deformed-TSDF fusion + association ("raycast") per frame, on a synthetic
deforming sphere (r 0.3 m at z 1.2 m, bend 2.0 rad/m oscillating with
frequency 2 over a 300-frame sequence).  One step = one
Reconstructor::process_frame (pipeline.cpp:143-262) with the reference's
default solver / correspondence / fusion parameters and 3 re-associations.
The global-pose ICP runs before the solve and the feature front-end (DoG
detection, matching against the FeatureStore, sparse constraints, store
update) runs around it, as in the reference's default configuration
(config.hpp:44-45, pipeline.cpp:95-141, 174-217, 257) -- on in both arms.

  python bench.py [--gpus N --steps K --warmup W]        B200 arm (libwfk.so)
  python bench.py --impl reference [...]                  CPU arm (the reference's own code,
                                                          oracle/_ref, on the host cores)

Frame 0 bootstraps the volume (untimed); W warm-up frames follow; K frames
are timed.  `value` times K frames whose inputs are staged in HBM beforehand;
`e2e` re-runs the same K frames from the same checkpointed volume through
wfk_process_frame with pinned HOST frame buffers (H2D of depth + color and
the D2H of the frame record inside the timed region).  L2 is flushed (256 MB
write) before every timed frame.  All times are CUDA events on the context's
stream.  With --gpus N > 1 (torchrun) every rank runs an independent replica
(the 128^3 path does not shard) and the timing is the max over
ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "non-rigid solve ms/frame & PCG iters/s at named lattice; HBM GB/s vs peak"
N_LATTICE = 128
W_PX, H_PX = 640, 480
FX, FY, CX, CY = 560.0, 560.0, 319.5, 239.5
FRAMES_TOTAL = 300
AMPLITUDE = 2.0
FREQUENCY = 2.0


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def workload_config(n_gpus):
    return {
        "workload": (f"VolumeDeform per-frame hot path, BASELINE configs[2]: 640x480 depth, 128^3 lattice, "
                     "3-level coarse-to-fine flip-flop GN/PCG + deformed-TSDF fusion + association"
                     if N_LATTICE == 128 else
                     f"VolumeDeform per-frame hot path on the BASELINE configs[3] lattice ({N_LATTICE}^3, "
                     "one GPU), 640x480 depth, 3-level coarse-to-fine flip-flop GN/PCG + fusion + association"),
        "lattice": [N_LATTICE] * 3,
        "depth_resolution": [W_PX, H_PX],
        "levels": 3, "flip_flop_iters": 4, "pcg_tol": 1e-4, "pcg_max_iters": 50, "reassociations": 3,
        "scene": "sphere r=0.3 m @ z=1.2 m, bend 2.0 rad/m, oscillating freq 2 over 300 frames",
        "icp": "on (global-pose ICP before the solve, config.hpp:45 default)",
        "sparse_features": "on (DoG features matched against the feature store, config.hpp:44 default)",
        "l2": "flushed (256 MB write) before every timed frame",
        "parallelism": f"replicas x{n_gpus}" if n_gpus > 1 else "single GPU",
    }


def scene(K):
    """The configs' synthetic sequence: tools/synthscene, the
    reference's SyntheticScene restated bit for bit (tests/test_synthscene.py),
    rendered on the host -- both arms consume identical frames."""
    from tools import synthscene as S
    return S.bend_sphere(K, frames=FRAMES_TOTAL, amplitude=AMPLITUDE, frequency=FREQUENCY)


def render_frames(K, indices, pinned=False):
    from tools import synthscene as S
    from paper_1603_08161_b200.abi import Frame
    sc = scene(K)
    out = []
    for f in indices:
        depth, color = S.render(sc, f)
        if pinned:
            from paper_1603_08161_b200.wfk import pinned_array
            pd = pinned_array(depth.shape, np.float32)
            pc = pinned_array(color.shape, np.float32)
            pd[:] = depth
            pc[:] = color
            depth, color = pd, pc
        out.append(Frame(K, depth, color))
    return out


REF_DESC = ("the reference itself: unmodified /root/reference/proj/src compiled with -O3 -fopenmp "
            "-ffp-contract=off against the Eigen/doctest subset shims (oracle/_ref/libwfref.so)")
DATA = ("synthetic (tools/synthscene: the reference's SyntheticScene restated and checked bit for bit against it; "
        "host-rendered, identical frames in both arms)")


def lattice_geometry():
    voxel = 0.7 / (N_LATTICE - 1)
    return (N_LATTICE,) * 3, voxel, (-0.35, -0.35, 0.85)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md "clocks" line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per flip-flop launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_flip_flop.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


# ---------------------------------------------------------------------------
# distributed plumbing (torchrun; replicas only)
# ---------------------------------------------------------------------------
class Dist:
    """One process per GPU (torchrun env).  The 128^3 workload runs as
    independent replicas, so the only collectives are the
    timing reductions: max over ranks of the device-timed region, sum of PCG
    iterations.  backend "gloo" (CPU tensors) is what the CPU tests use."""

    def __init__(self, n_gpus, backend="nccl"):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.device = "cuda" if backend == "nccl" else "cpu"
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.torch, self.dist = torch, dist

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return float(t.item())

    def whole_job_ms_per_frame(self, total_ms, frames_per_rank):
        """Whole-job ms/frame: the slowest rank's timed region over every
        rank's frames (each rank processes frames_per_rank frames)."""
        return self.max(total_ms) / (frames_per_rank * self.world)

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args):
    from paper_1603_08161_b200.abi import Intrinsics, Pose, SolverParams, Volume
    from paper_1603_08161_b200.wfk import Context, pipeline_config

    d = Dist(args.gpus)
    ctx = Context(d.local)
    K = Intrinsics.make(FX, FY, CX, CY, W_PX, H_PX)
    n_frames = 1 + args.warmup + args.steps

    # synthetic input sequence, rendered on the host, kept in pinned host memory
    frames = render_frames(K, range(n_frames), pinned=True)
    log(f"rendered {n_frames} frames; valid depth px of frame 1: {int((frames[min(1, n_frames - 1)].depth > 0).sum())}")

    dims, voxel, origin = lattice_geometry()
    vol = Volume(dims, voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=3)
    pose = Pose.make()
    for f in range(1, n_frames):
        ctx.stage_frame(f, frames[f])

    log("staged frames")
    rec0 = ctx.process_frame(frames[0], pose, cfg, 0)  # bootstrap
    log(f"bootstrap: fused {rec0.fusion.fused}")
    assert rec0.bootstrap == 1
    for f in range(1, 1 + args.warmup):
        pose = ctx.process_staged_frame(f, pose, cfg, f).pose  # the Reconstructor's pose_, refined by ICP

    # checkpoint (volume + pose + feature store) so the e2e pass repeats exactly the same K frames
    log("warm-up done")
    ckpt = Volume(dims, voxel, origin)
    ctx.download_volume(ckpt)
    ckpt_pose = pose
    ckpt_store = ctx.feature_store()
    timed = list(range(1 + args.warmup, n_frames))

    # ---- value: inputs resident in HBM ---------------------------------------
    ctx.profile_enable(True)
    launches0 = ctx.launch_count
    recs = []
    total_ms = 0.0
    frame_ms = []
    d.barrier()
    with ClockSampler(d.local) as clocks:
        for f in timed:
            ctx.flush_l2()
            ctx.timer_mark(0)
            recs.append(ctx.process_staged_frame(f, pose, cfg, f))
            ctx.timer_mark(1)
            pose = recs[-1].pose
            frame_ms.append(ctx.timer_elapsed_ms(0, 1))
            total_ms += frame_ms[-1]
    d.barrier()
    launches = ctx.launch_count - launches0
    prof = ctx.profile_read()
    ctx.profile_enable(False)

    log(f"timed: {total_ms / len(timed):.3f} ms/frame")
    # ---- e2e: same frames through the public call with host buffers -----------
    ctx.upload_volume(ckpt)
    ctx.set_feature_store(ckpt_store)
    pose = ckpt_pose
    e2e_ms = 0.0
    e2e_frame_ms = []
    d.barrier()
    for f in timed:
        ctx.flush_l2()
        ctx.timer_mark(2)
        r = ctx.process_frame(frames[f], pose, cfg, f)   # H2D frame + D2H record inside
        ctx.timer_mark(3)
        e2e_frame_ms.append(ctx.timer_elapsed_ms(2, 3))
        e2e_ms += e2e_frame_ms[-1]
        pose = r.pose
        _ = (r.energy.total, r.dense_count)
    d.barrier()

    k = len(timed)
    ms_frame = d.max(total_ms) / k          # per-rank ms/frame (slowest rank)
    e2e_frame = d.max(e2e_ms) / k
    job_ms_frame = d.whole_job_ms_per_frame(total_ms, k)
    job_e2e_frame = d.whole_job_ms_per_frame(e2e_ms, k)
    pcg_iters = sum(r.pcg_iterations for r in recs)
    pcg_iters_all = d.sum(pcg_iters)
    peak, peak_src = measured_peak()
    achieved = prof.flip_flop_bytes / (prof.flip_flop_ms * 1e-3) / 1e9 if prof.flip_flop_ms > 0 else 0.0
    achieved_impl = prof.flip_flop_bytes_impl / (prof.flip_flop_ms * 1e-3) / 1e9 if prof.flip_flop_ms > 0 else 0.0
    traffic, ncu_doc = ncu_traffic()
    clk = clocks.summary()

    cpu = None
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(frames, args.cpu_frames)

    if d.rank == 0:
        out = {
            "metric": METRIC,
            "value": job_ms_frame,
            "unit": "ms/frame",
            "n_gpus": d.world,
            "steps": k,
            "warmup": args.warmup,
            "ms_per_step": ms_frame,
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": DATA,
            "config": workload_config(d.world),
            "pcg_iters_per_s": pcg_iters_all / (d.max(total_ms) * 1e-3),
            "pcg_iterations_per_frame": pcg_iters / k,
            "frame_breakdown_ms": {kk: v / k for kk, v in prof.as_dict()["stage_ms"].items()},
            "frame_ms": [round(x, 3) for x in frame_ms],
            "e2e_frame_ms": [round(x, 3) for x in e2e_frame_ms],
            "dense_constraints_per_frame": float(np.mean([r.dense_count for r in recs])),
            "sparse_constraints_per_frame": float(np.mean([r.sparse_count for r in recs])),
            "feature_matches_per_frame": float(np.mean([r.match_count for r in recs])),
            "feature_store_size": int(len(ctx.feature_store())),
            "gpu_launches": int(launches),
            "roofline": {
                "bound": "hbm",
                "kernel": "k_flip_flop (cooperative flip-flop solve: energy, rhs/diag, matrix-free Jacobi-PCG, "
                          "write-back, Procrustes, energy)",
                "achieved": achieved,
                "peak": peak,
                "peak_source": peak_src,
                "unit": "GB/s",
                "frac": achieved / peak,
                "traffic": traffic,
                "bytes_model": "SURVEY.md 8(d): PCG 160 N + 32 C_d + 20 C_s per iteration, rhs/diag 52 N, "
                               "rotation 28 N, energy 28 N + 44 C",
                "achieved_fp64_layout": achieved_impl,
                "launches": prof.flip_flop_launches,
                "avg_launch_ms": prof.flip_flop_ms / max(prof.flip_flop_launches, 1),
                "share_of_frame": prof.flip_flop_ms / max(total_ms, 1e-9),
            },
            "e2e": {
                "value": job_e2e_frame,
                "unit": "ms/frame",
                "h2d_bytes_per_step": int(frames[0].depth.nbytes + frames[0].color.nbytes),
                "d2h_bytes_per_step": int(__import__("ctypes").sizeof(type(recs[0]))),
            },
            "clocks": clk,
        }
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    ctx.close()
    d.close()


def run_partitioned(args):
    """BASELINE configs[3]: the frame-1 solve on a 256^3
    lattice with every level's PCG slab-partitioned across the N ranks
    (wfk_solve_coarse_to_fine_dist, NCCL halos + all-gathered dots), repeated
    from the same checkpoint.  One step = one coarse-to-fine solve; `value` =
    ms per solve (max over ranks, CUDA events on the context stream);
    "scaling": "strong" (the lattice is fixed as N grows)."""
    from paper_1603_08161_b200.abi import CorrespondParams, Intrinsics, Pose, SolverParams, Volume
    from paper_1603_08161_b200.wfk import Context, dist_unique_id, pipeline_config

    d = Dist(args.gpus)
    ctx = Context(d.local)
    if d.world > 1:
        idt = d.torch.zeros(128, dtype=d.torch.uint8, device=d.device)
        if d.rank == 0:
            idt[:] = d.torch.frombuffer(bytearray(dist_unique_id()), dtype=d.torch.uint8).to(d.device)
        d.dist.broadcast(idt, 0)
        ctx.dist_init(d.rank, d.world, bytes(idt.cpu().tolist()))
    else:
        ctx.dist_init(0, 1)
    K = Intrinsics.make(FX, FY, CX, CY, W_PX, H_PX)
    frames = render_frames(K, [3, 4])  # a visible bend between the two frames
    dims, voxel, origin = lattice_geometry()
    vol = Volume(dims, voxel, origin)
    ctx.upload_volume(vol)
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=1, estimate_pose=False, use_features=False)
    pose = Pose.make()
    ctx.process_frame(frames[0], pose, cfg, 0)  # bootstrap
    # frame 1's dense constraints against the bootstrap surface
    ctx.upload_frame(frames[1])
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(pose)
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    n_cons = ctx.find_dense_correspondences(K, CorrespondParams.make(), drop_inactive=True)
    ckpt = Volume(dims, voxel, origin)
    ctx.download_volume(ckpt)
    p = SolverParams.make()
    for _ in range(args.warmup):
        ctx.upload_volume(ckpt)
        ctx.solve_coarse_to_fine_dist(pose, p)
    total_ms, pcg = 0.0, 0
    for _ in range(args.steps):
        ctx.upload_volume(ckpt)
        ctx.flush_l2()
        d.barrier()
        ctx.timer_mark(0)
        tr = ctx.solve_coarse_to_fine_dist(pose, p)
        ctx.timer_mark(1)
        total_ms += ctx.timer_elapsed_ms(0, 1)
        pcg += sum(e["pcg_iterations"] for e in tr)
    d.barrier()
    ms = d.max(total_ms) / args.steps
    fused = None
    if d.world == 1:  # the fused single-GPU solve of the same system, for reference
        fms = 0.0
        for _ in range(max(args.steps, 2)):
            ctx.upload_volume(ckpt)
            ctx.flush_l2()
            ctx.timer_mark(0)
            ctx.solve_coarse_to_fine(pose, p)
            ctx.timer_mark(1)
            fms += ctx.timer_elapsed_ms(0, 1)
        fused = fms / max(args.steps, 2)
    _, act = ctx.hierarchy_info(3)
    if d.rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": ms, "unit": "ms/solve", "n_gpus": d.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": DATA + ", frames 3-4",
            "config": {"workload": f"BASELINE configs[3]: {N_LATTICE}^3 lattice, frame-1 coarse-to-fine solve, "
                                   "every level's PCG slab-partitioned (z-slabs, NCCL halos + all-gathered dots)",
                       "lattice": [N_LATTICE] * 3, "rows_per_level": [int(a) for a in act],
                       "dense_constraints": int(n_cons), "parallelism": f"z-slab x{d.world}",
                       "l2": "flushed before every solve"},
            "pcg_iters_per_s": pcg / (d.max(total_ms) * 1e-3),
            "fused_single_gpu_ms_per_solve": fused,
            "gpu_launches": int(ctx.launch_count),
        }), flush=True)
    ctx.close()
    d.close()


# ---------------------------------------------------------------------------
# BASELINE configs[3] / configs[4] on one GPU: the frame-1 solve, repeated
# ---------------------------------------------------------------------------
SOLVE_CONFIGS = {
    # 256^3 sphere, 640x480, frame-1 solve (bend), levels 3
    3: dict(n=256, K=(560.0, 560.0, 319.5, 239.5, 640, 480), voxel=0.7 / 255, origin=(-0.35, -0.35, 0.85),
            scene="sphere", desc="BASELINE configs[3]: 256^3 lattice, 640x480, bend sphere, frame-1 coarse-to-fine "
                                 "solve (3 levels) on one GPU"),
    # 512^3, 1280x720, acceptance C4 five-wall room + sphere r 0.12 at (0, 0, 1.2),
    # voxel 0.63/511, origin (-0.315, -0.315, 0.95) (acceptance.cpp:466-486 scaled), frame-1 solve
    4: dict(n=512, K=(1120.0, 1120.0, 639.5, 359.5, 1280, 720), voxel=0.63 / 511, origin=(-0.315, -0.315, 0.95),
            scene="room", desc="BASELINE configs[4] (north-star stress): 512^3 lattice, 1280x720, five-wall room + "
                               "sphere, frame-1 coarse-to-fine solve (3 levels) on one GPU"),
}


def run_solve(args):
    """One step = the frame-1 solve_coarse_to_fine of a BASELINE solve config,
    from identical state every time (device-side checkpoint of the volume
    after the bootstrap frame): constraints from the frame-1 association at
    the ICP pose, as process_frame builds them (pipeline.cpp:174-240).  Inputs
    are HBM-resident; `value` = ms per solve (CUDA events, L2 flushed before
    each solve).  The roofline is the SURVEY.md 8(d) byte model of every
    k_flip_flop launch of the timed solves."""
    from paper_1603_08161_b200.abi import CorrespondParams, Frame, Intrinsics, Pose, SolverParams
    from paper_1603_08161_b200.wfk import Context, pipeline_config
    from tools import synthscene as S
    cfg_s = SOLVE_CONFIGS[args.solve_config]
    n = cfg_s["n"]
    K = Intrinsics.make(*cfg_s["K"])
    if cfg_s["scene"] == "room":
        sc = S.room_corner(K, frames=30, sphere_radius=0.12)
        frames_idx = [0, 1]
    else:
        sc = S.bend_sphere(K, frames=FRAMES_TOTAL, amplitude=AMPLITUDE, frequency=FREQUENCY)
        frames_idx = [3, 4]  # a visible bend between the two frames
    frames = [Frame(K, *S.render(sc, f)) for f in frames_idx]
    if args.slabs:
        # the matrix-free levels' CG cut into z-slab ranks inside the persistent
        # kernel (pcg_slab; virtual ranks on this GPU; read per solve call)
        os.environ["WFK_SLABS"] = str(args.slabs)
    ctx = Context(0)
    if args.fast:
        ctx.set_precision(1)  # WFK_PRECISION_FAST: fp32 Krylov vectors on levels that run the CG variant
    t0 = time.perf_counter()
    ctx.create_volume((n, n, n), cfg_s["voxel"], cfg_s["origin"])
    cfg = pipeline_config(solver=SolverParams.make(), reassociations=1)
    rec0 = ctx.process_frame(frames[0], Pose.make(), cfg, 0)  # bootstrap: fusion + active set
    ctx.checkpoint_volume()
    rec1 = ctx.process_frame(frames[1], Pose.make(), cfg, 1)  # the frame's ICP pose (and a full frame, untimed)
    pose = rec1.pose
    ctx.checkpoint_volume(restore=True)
    log(f"setup {time.perf_counter() - t0:.1f}s: bootstrap fused {rec0.fusion.fused}, frame-1 ICP pose found")
    # frame-1 dense constraints against the bootstrap surface at that pose (pipeline.cpp:161-240)
    ctx.upload_frame(frames[1])
    ctx.backproject_depth(download=False)
    ctx.extract_mesh(pose)
    ctx.compute_normals()
    ctx.rasterize(K, download=False)
    n_cons = ctx.find_dense_correspondences(K, CorrespondParams.make(), drop_inactive=True)
    p = SolverParams.make()
    for _ in range(args.warmup):
        ctx.checkpoint_volume(restore=True)
        ctx.solve_coarse_to_fine(pose, p)
    ctx.profile_enable(True)
    launches0 = ctx.launch_count
    total_ms, pcg, times = 0.0, 0, []
    with ClockSampler(0) as clocks:
        for _ in range(args.steps):
            ctx.checkpoint_volume(restore=True)
            ctx.flush_l2()
            ctx.timer_mark(0)
            tr = ctx.solve_coarse_to_fine(pose, p)
            ctx.timer_mark(1)
            times.append(ctx.timer_elapsed_ms(0, 1))
            total_ms += times[-1]
            pcg += sum(e["pcg_iterations"] for e in tr)
    launches = ctx.launch_count - launches0
    prof = ctx.profile_read()
    ctx.profile_enable(False)
    dims, act = ctx.hierarchy_info(3)
    ms = total_ms / args.steps
    peak, peak_src = measured_peak()
    achieved = prof.flip_flop_bytes / (prof.flip_flop_ms * 1e-3) / 1e9 if prof.flip_flop_ms > 0 else 0.0
    achieved_impl = prof.flip_flop_bytes_impl / (prof.flip_flop_ms * 1e-3) / 1e9 if prof.flip_flop_ms > 0 else 0.0
    out = {
        "metric": METRIC, "value": ms, "unit": "ms/solve", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64+f32 (mixed)" if args.fast else "f64",
        "data": DATA + f", frames {frames_idx[0]}-{frames_idx[1]}",
        "config": {"workload": cfg_s["desc"] + (" [WFK_PRECISION_FAST]" if args.fast else ""),
                   "precision": "fast (fp32 Krylov vectors on CG levels)" if args.fast else "fp64",
                   "lattice": [n] * 3, "depth_resolution": list(cfg_s["K"][4:]),
                   "rows_per_level": [int(x) for x in act], "dense_constraints": int(n_cons),
                   "l2": "flushed (256 MB write) before every solve",
                   "parallelism": (f"single GPU; matrix-free levels of >= {os.environ.get('WFK_SLAB_MIN_ROWS', 100000)} "
                                   f"rows: CG slab-partitioned into {args.slabs} ranks (block groups of one "
                                   "cooperative launch); smaller levels unpartitioned (replicated across ranks)")
                                  if args.slabs else "single GPU"},
        "pcg_iters_per_s": pcg / (total_ms * 1e-3), "pcg_iterations_per_solve": pcg / args.steps,
        "solve_ms": [round(x, 3) for x in times], "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_flip_flop", "achieved": achieved, "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                     "bytes_model": "SURVEY.md 8(d): PCG 160 N + 32 C_d + 20 C_s per iteration, rhs/diag 52 N, "
                                    "rotation 28 N, energy 28 N + 44 C",
                     "achieved_fp64_layout": achieved_impl, "frac_fp64_layout": achieved_impl / peak,
                     "launches": prof.flip_flop_launches,
                     "avg_launch_ms": prof.flip_flop_ms / max(prof.flip_flop_launches, 1),
                     "share_of_solve": prof.flip_flop_ms / max(total_ms, 1e-9)},
        "clocks": clocks.summary(),
        "energy_final": tr[-1]["energy"]["total"] if tr else None,
        "energy_final_hex": float(tr[-1]["energy"]["total"]).hex() if tr else None,
    }
    print(json.dumps(out), flush=True)
    ctx.close()


def cpu_baseline_sample(frames, n_frames):
    """The oracle port on this host's cores, frames 1..n of the same sequence
    after the (untimed) bootstrap frame 0; reports the median ms/frame."""
    from oracle import pyoracle as O
    from paper_1603_08161_b200.abi import SolverParams
    dims, voxel, origin = lattice_geometry()
    rec = O.Reconstructor(dims, voxel, origin, solver=SolverParams.make(), reassociations=3)
    rec.process_frame(frames[0])
    times = []
    for f in range(1, 1 + n_frames):
        t0 = time.perf_counter()
        rec.process_frame(frames[f])
        times.append((time.perf_counter() - t0) * 1e3)
    cores = int(O.lib().wfo_num_threads())
    kind = "reference" if O.backend() == "ref" else "port"
    # also the 1-thread figure, on the next frame of the sequence
    serial = None
    if 1 + n_frames < len(frames):
        O.lib().wfo_set_num_threads(1)
        t0 = time.perf_counter()
        rec.process_frame(frames[1 + n_frames])
        serial = (time.perf_counter() - t0) * 1e3
        O.lib().wfo_set_num_threads(cores)
    return {"value": float(np.median(times)), "unit": "ms/frame", "cores": cores,
            "kind": kind,
            "sample": (f"{REF_DESC if kind == 'reference' else 'oracle port (oracle/wf_oracle.cpp)'}: "
                       f"Reconstructor::process_frame on frames 1..{n_frames} of the same sequence after the "
                       f"bootstrap frame (median of {n_frames}), OpenMP threads = {cores}"),
            "serial_1thread_ms_per_frame": serial}


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port) on this host
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import pyoracle as O
    from paper_1603_08161_b200.abi import Intrinsics, SolverParams
    K = Intrinsics.make(FX, FY, CX, CY, W_PX, H_PX)
    n_frames = 1 + args.warmup + args.steps
    frames = render_frames(K, range(n_frames))
    dims, voxel, origin = lattice_geometry()
    rec = O.Reconstructor(dims, voxel, origin, solver=SolverParams.make(), reassociations=3)
    rec.process_frame(frames[0])
    for f in range(1, 1 + args.warmup):
        rec.process_frame(frames[f])
    t0 = time.perf_counter()
    pcg = 0
    for f in range(1 + args.warmup, n_frames):
        r = rec.process_frame(frames[f])
        pcg += r.pcg_iterations
    dt = time.perf_counter() - t0
    ms = dt * 1e3 / args.steps
    cores = int(O.lib().wfo_num_threads())
    kind = "reference" if O.backend() == "ref" else "port"
    what = REF_DESC if kind == "reference" else "oracle port of the reference path (oracle/wf_oracle.cpp)"
    out = {
        "impl": "reference",
        "metric": METRIC,
        "value": ms,
        "unit": "ms/frame",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": DATA,
        "config": workload_config(1),
        "pcg_iters_per_s": pcg / dt,
        "cpu_baseline": {"value": ms, "unit": "ms/frame", "cores": cores, "kind": kind,
                         "sample": f"{what}, OpenMP {cores} threads, wf::Reconstructor::process_frame on "
                                   f"{args.steps} full frames after bootstrap + {args.warmup} warm-up"},
        "e2e": {"value": ms, "unit": "ms/frame", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    global N_LATTICE
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-frames", type=int, default=2)
    ap.add_argument("--lattice", type=int, default=N_LATTICE,
                    help="lattice side (default 128 = configs[2]; 256 = the configs[3] lattice on one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solve-config", type=int, choices=[3, 4], default=None,
                    help="BASELINE configs[3] (256^3) or configs[4] (512^3, 1280x720 room): the frame-1 solve x K")
    ap.add_argument("--fast", action="store_true",
                    help="with --solve-config: WFK_PRECISION_FAST (fp32 Krylov vectors on the large CG levels)")
    ap.add_argument("--slabs", type=int, default=0,
                    help="with --solve-config: run the matrix-free levels' CG slab-partitioned into this many ranks "
                         "inside the persistent kernel (WFK_SLABS)")
    ap.add_argument("--partitioned", action="store_true",
                    help="BASELINE configs[3]: the 256^3 frame-1 solve with the PCG slab-partitioned over the ranks")
    args = ap.parse_args()
    N_LATTICE = args.lattice
    if args.warmup < 3 and args.impl == "b200":
        print("warning: W >= 3 warm-up steps are required for a valid number", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.solve_config:
        run_solve(args)
    elif args.partitioned:
        if args.lattice == 128 and "--lattice" not in sys.argv:
            N_LATTICE = 256
        run_partitioned(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
