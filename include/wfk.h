/* libwfk — B200-native (sm_100a) non-rigid alignment solver, deformed-TSDF
 * fusion and projective association of VolumeDeform (arXiv 1603.08161).
 *
 * Drop-in boundary for the reference's hot path (warpfuse, namespace wf).
 * Each entry point below names the reference function it replaces; the C++
 * adapter a maintainer adds on the reference side wraps a
 * wf::DeformableVolume / std::vector<wf::Correspondence> around these calls and
 * re-throws the reference's exception types from the returned status.
 *
 * Conventions
 *   - Every function returns WFK_OK (0) or a negative WFK_E_* status;
 *     wfk_last_error(ctx) describes the last failure.  No exception crosses.
 *   - Calls are synchronous (results are ready on return, like the reference)
 *     and not re-entrant per context; use one context per thread / GPU.
 *   - The context owns a device-resident copy of ONE DeformableVolume; host
 *     arrays are only touched by wfk_volume_upload / wfk_volume_download and
 *     the explicit download helpers, so a caller that keeps the volume resident
 *     pays no host<->device traffic between calls.
 *   - Exec arguments are accepted for interface parity; the device path is
 *     deterministic (run-to-run identical) for both values.
 */
#pragma once

#include "wfk_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wfk_ctx wfk_ctx;

typedef struct wfk_config {
  int32_t device;     /* CUDA ordinal */
  int32_t precision;  /* WFK_PRECISION_FP64 (default: the reference's arithmetic) or WFK_PRECISION_FAST */
  int32_t reserved_[6];
} wfk_config;

/* Precision of the context ("fp64 parity / fp32 fast").
 * FAST stores the Krylov vectors of the Chronopoulos-Gear PCG -- the variant
 * that runs levels too large for shared memory (>= 500 K rows) -- in fp32
 * (arithmetic, dot products, the initial residual and the solution stay fp64;
 * the solution is carried as x0 + an fp32 increment).  Levels that fit keep
 * fp64 either way.  Parity then holds to tolerance, not bit for bit. */
enum { WFK_PRECISION_FP64 = 0, WFK_PRECISION_FAST = 1 };

/* ---- context ------------------------------------------------------------- */
int wfk_create(const wfk_config* cfg, wfk_ctx** out);
void wfk_destroy(wfk_ctx* ctx);
/* change the context's precision (WFK_PRECISION_*) for subsequent solves */
int wfk_set_precision(wfk_ctx* ctx, int32_t precision);
const char* wfk_last_error(const wfk_ctx* ctx);
int wfk_version(void);
/* kernel launches issued by this context so far (for bench accounting) */
int64_t wfk_launch_count(const wfk_ctx* ctx);
/* total PCG iterations run by this context so far */
int64_t wfk_pcg_iteration_count(const wfk_ctx* ctx);

/* ---- volume residency (DeformableVolume, volume.hpp:29-112) --------------- */
/* (Re)allocates the device lattice when dims change; copies the fields in
 * `fields` (WFK_VOL_* mask). */
int wfk_volume_upload(wfk_ctx* ctx, const wfk_volume_view* v, uint32_t fields);
int wfk_volume_download(wfk_ctx* ctx, wfk_volume_view* v, uint32_t fields);
/* a DeformableVolume in its constructor state (volume.cpp:8-25) created on the
 * device (truncation 4 x voxel) -- no host lattice needed for large volumes */
int wfk_volume_create(wfk_ctx* ctx, const int32_t dims[3], double voxel_size, const double origin[3]);
/* device-side checkpoint of the fields a solve or an expansion mutates
 * (deformed, euler, age, active): restore = 0 saves, 1 restores (e.g. to
 * repeat one frame's solve from identical state without host traffic) */
int wfk_volume_checkpoint(wfk_ctx* ctx, int32_t restore);

/* ---- solver (proj/include/wf/solver.hpp) ------------------------------------- */
/* compute_active_set (solver.hpp:40, solver.cpp:32-69): grow-only.  Writes the
 * ascending active list to out (may be NULL) and its length to n_out. */
int wfk_compute_active_set(wfk_ctx* ctx, int32_t* out, int64_t cap, int64_t* n_out);

/* Constraints for the next solve / energy call (the std::vector<Correspondence>
 * argument of solver.hpp:89-119).  Anchors must be the trilinear anchors of a
 * lattice cell (anchor k = anchor 0 + corner offset k), as
 * DeformableVolume::trilinear_anchors produces them; anything else is
 * WFK_E_INVALID_ARG, an index outside the lattice WFK_E_OUT_OF_RANGE. */
int wfk_constraints_upload(wfk_ctx* ctx, const wfk_correspondence* c, int64_t n);
/* download the constraints the context currently holds (e.g. after
 * wfk_find_dense_correspondences); n_out = count */
int wfk_constraints_download(wfk_ctx* ctx, wfk_correspondence* out, int64_t cap, int64_t* n_out);

/* evaluate_energy (solver.hpp:88-90, solver.cpp:345-383) */
int wfk_evaluate_energy(wfk_ctx* ctx, const wfk_pose* pose, const wfk_solver_params* p,
                        wfk_energy* out);
/* update_rotations (solver.hpp:94, solver.cpp:385-417) */
int wfk_update_rotations(wfk_ctx* ctx, int32_t exec);
/* flip_flop_solve (solver.hpp:97-101, solver.cpp:419-453) on the volume */
int wfk_flip_flop_solve(wfk_ctx* ctx, const wfk_pose* pose, const wfk_solver_params* p,
                        int32_t level, wfk_trace_entry* trace, int32_t cap, int32_t* n_out);
/* solve_coarse_to_fine (solver.hpp:117-119, solver.cpp:505-534) */
int wfk_solve_coarse_to_fine(wfk_ctx* ctx, const wfk_pose* pose, const wfk_solver_params* p,
                             wfk_trace_entry* trace, int32_t cap, int32_t* n_out);

/* build_normal_equations (solver.hpp:62-66, solver.cpp:108-280), materialised
 * on the host in the reference layout.  Two-call: pass NULL arrays to get
 * rows_out, then call again with arrays sized rows*27*9 (blocks, row-major
 * 3x3), rows*27 (cols), rows*3 (rhs), rows (rows, frozen), n (node_row). */
typedef struct wfk_ne_host {
  int32_t* rows;
  int32_t* node_row;
  double* blocks;
  int32_t* cols;
  double* rhs;
  uint8_t* frozen;
} wfk_ne_host;
int wfk_build_normal_equations(wfk_ctx* ctx, const wfk_pose* pose, const wfk_solver_params* p,
                               wfk_ne_host* out, int32_t* rows_out);

/* pcg_solve (solver.hpp:83-86, solver.cpp:282-343) on an explicit assembled
 * NormalEquations (host arrays as above, `rows` rows); x is in/out (rows*3). */
int wfk_pcg_solve(wfk_ctx* ctx, int32_t rows, const double* blocks, const int32_t* cols,
                  const double* rhs, double* x, double tol, int32_t max_iters, int32_t exec,
                  wfk_pcg_result* out);

/* ---- snapshot and frame formats -------------------------
 * DeformableVolume::save / load (volume.cpp:150-217; volume.hpp:99-100): the
 * "WFVOL01\n" snapshot (60-byte header, one interleaved 73-byte record per
 * point), packed from / unpacked into the context's lattice on the device.
 * Load replaces the lattice (dims, voxel, origin, truncation and every field).
 * pack / unpack: the same byte image in memory (size query: out = NULL). */
int wfk_volume_save(wfk_ctx* ctx, const char* path);
int wfk_volume_load(wfk_ctx* ctx, const char* path);
int wfk_volume_pack(wfk_ctx* ctx, uint8_t* out, int64_t cap, int64_t* n_out);
int wfk_volume_unpack(wfk_ctx* ctx, const uint8_t* in, int64_t n);
/* FeatureStore::save / load (features.cpp:306-352; features.hpp:90-91), "WFFEAT1\n" */
int wfk_feature_store_save(wfk_ctx* ctx, const char* path);
int wfk_feature_store_load(wfk_ctx* ctx, const char* path);
/* load_depth_pgm + load_color_ppm (image.cpp:71-121) decoded on the device into
 * the context's frame (color_ppm may be NULL; the images must be intr's size);
 * save_depth_pgm / save_color_ppm (image.cpp:55-104) of the context's frame
 * (either path may be NULL); wfk_frame_download reads the frame back. */
int wfk_frame_load_pnm(wfk_ctx* ctx, const char* depth_pgm, const char* color_ppm,
                       const wfk_intrinsics* intr);
int wfk_frame_save_pnm(wfk_ctx* ctx, const char* depth_pgm, const char* color_ppm);
int wfk_frame_download(wfk_ctx* ctx, float* depth, float* color);

/* ---- slab-partitioned PCG ------------------------------------
 * pcg_solve with the rows split into contiguous ranges, one per rank (rows are
 * in lattice order, so a range is a z-slab): per iteration each rank applies A
 * to its rows, exchanges the halo rows of p with their owners and all-gathers
 * its partial dots, summed in rank order on every rank.  Every rank passes the
 * full system and receives the full x.
 *   wfk_dist_unique_id: an NCCL unique id (rank 0; share it, e.g. through
 *     torch.distributed); wfk_dist_init: join the communicator (world 1 needs no id).
 *   wfk_pcg_solve_dist: the partitioned solve over NCCL (one process per GPU).
 *   wfk_pcg_solve_slabs: the same partition run by one process on its GPU as
 *     `slabs` slab states with device copies for the halos (single-GPU check).
 *   wfk_dist_plan: the partition (host only): ranges[2 * world] = {lo, hi} per
 *     rank, xfers[4 * n] = {src, dst, row_lo, row_hi} halo transfers. */
int wfk_dist_unique_id(uint8_t* id /* 128 bytes */);
int wfk_dist_init(wfk_ctx* ctx, int32_t rank, int32_t world, const uint8_t* id);
int wfk_pcg_solve_dist(wfk_ctx* ctx, int32_t rows, const double* blocks, const int32_t* cols,
                       const double* rhs, double* x, double tol, int32_t max_iters, wfk_pcg_result* out);
int wfk_pcg_solve_slabs(wfk_ctx* ctx, int32_t slabs, int32_t rows, const double* blocks,
                        const int32_t* cols, const double* rhs, double* x, double tol, int32_t max_iters,
                        wfk_pcg_result* out);
/* solve_coarse_to_fine (solver.cpp:505-534) with every level's PCG partitioned
 * as above: the replicated lattice, hierarchy, normal-equation assembly,
 * write-back, Procrustes fit and energy run identically on every rank; the
 * PCG runs on the rank's slab.  _dist: the context's communicator; _slabs:
 * `slabs` slab states on this GPU. */
int wfk_solve_coarse_to_fine_dist(wfk_ctx* ctx, const wfk_pose* pose, const wfk_solver_params* p,
                                  wfk_trace_entry* trace, int32_t cap, int32_t* n_out);
int wfk_solve_coarse_to_fine_slabs(wfk_ctx* ctx, int32_t slabs, const wfk_pose* pose,
                                   const wfk_solver_params* p, wfk_trace_entry* trace, int32_t cap,
                                   int32_t* n_out);
int wfk_dist_plan(int32_t rows, const int32_t* cols, int32_t world, int32_t* ranges, int32_t* xfers,
                  int32_t cap, int32_t* n_xfers);
/* The in-kernel slab partition of the matrix-free levels' CG (WFK_SLABS=S;
 * no reference counterpart -- SURVEY.md 8(e)): host part of its plan.  The
 * rows are cut into *n_tiles tiles (blocks x clamp(rows / (blocks x
 * block_threads), 1, 8)) of about equal summed row_work: tile t = rows
 * [tile_rows[t], tile_rows[t + 1]) (tile_rows: 8 blocks + 1 entries); rank s
 * owns tiles [rank_tiles[s], rank_tiles[s + 1]) (ranks + 1 entries, equal
 * tile counts).  ranks <= blocks. */
int wfk_slab_plan(int32_t rows, const int32_t* row_work, int32_t blocks, int32_t block_threads, int32_t ranks,
                  int32_t* n_tiles, int32_t* tile_rows, int32_t* rank_tiles);
/* NormalEquations::multiply (solver.cpp:71-89) on an explicit system */
int wfk_ne_multiply(wfk_ctx* ctx, int32_t rows, const double* blocks, const int32_t* cols,
                    const double* x, double* y);

/* hierarchy shape (build_hierarchy, solver.cpp:455-503): dims and active count
 * of each level for the current volume + constraints. */
int wfk_hierarchy_info(wfk_ctx* ctx, int32_t levels, int32_t* dims_out, int64_t* active_out);

/* ---- fusion (proj/include/wf/fusion.hpp) ---------------------------------- */
/* Uploads the frame used by integrate / backproject / association. */
int wfk_frame_upload(wfk_ctx* ctx, const wfk_frame_view* frame);
/* integrate_frame (fusion.hpp:26-28, fusion.cpp:7-83) with the uploaded frame */
int wfk_integrate_frame(wfk_ctx* ctx, const wfk_pose* pose, const wfk_fusion_params* p,
                        int32_t exec, wfk_fusion_stats* out);
/* expand_grid (fusion.hpp:37, fusion.cpp:85-122) */
int wfk_expand_grid(wfk_ctx* ctx, wfk_expansion_stats* out);
/* advance_ages (fusion.hpp:40, fusion.cpp:124-126) */
int wfk_advance_ages(wfk_ctx* ctx, const int32_t* idx, int64_t n);
/* advance_ages over exactly the active set (pipeline.cpp:249-252) */
int wfk_advance_active_ages(wfk_ctx* ctx);

/* ---- association / "raycast" (correspond.hpp, isosurface.hpp) ------------ */
/* backproject_depth (correspond.hpp:44, correspond.cpp:7-57) of the uploaded
 * frame; out may be NULL (maps stay on the device). */
int wfk_backproject_depth(wfk_ctx* ctx, int32_t exec, wfk_point_normal_map* out);
/* caller-computed PointNormalMap (correspond.hpp:34-42) as the context's frame
 * maps -- what a drop-in estimate_global_pose / find_dense_correspondences
 * receives from the reference's caller */
int wfk_maps_upload(wfk_ctx* ctx, const wfk_point_normal_map* maps);
/* extract_mesh (isosurface.hpp:49, isosurface.cpp:39-97); sizes returned */
int wfk_extract_mesh(wfk_ctx* ctx, const wfk_pose* pose, int64_t* nv, int64_t* nt);
/* re-warp the mesh's canonical vertices through the current field (the
 * `redeform` step of pipeline.cpp:167-169) */
int wfk_mesh_warp(wfk_ctx* ctx, const wfk_pose* pose);
/* compute_normals (isosurface.hpp:52, isosurface.cpp:99-112) */
int wfk_compute_normals(wfk_ctx* ctx);
/* replace / read the device mesh */
int wfk_mesh_upload(wfk_ctx* ctx, const wfk_mesh_view* m);
int wfk_mesh_download(wfk_ctx* ctx, wfk_mesh_view* m);
/* rasterize (isosurface.hpp:56-57, rasterize.cpp:29-137); out may be NULL */
int wfk_rasterize(wfk_ctx* ctx, const wfk_intrinsics* intr, int32_t exec,
                  wfk_geometry_buffer* out);
int wfk_gbuffer_upload(wfk_ctx* ctx, const wfk_geometry_buffer* b);
/* find_dense_correspondences (correspond.hpp:61-64, correspond.cpp:114-150) from
 * the device geometry buffer and maps; the result replaces the context's
 * constraints.  With drop_inactive != 0 constraints with an inactive anchor
 * are removed as pipeline.cpp:220-229 does.  n_out = count. */
int wfk_find_dense_correspondences(wfk_ctx* ctx, const wfk_intrinsics* intr,
                                   const wfk_correspond_params* p, int32_t drop_inactive,
                                   int64_t* n_out);
/* append caller-supplied constraints (e.g. sparse feature constraints) to the
 * context's constraints; with drop_inactive != 0 keeps only fully active ones */
int wfk_constraints_append(wfk_ctx* ctx, const wfk_correspondence* c, int64_t n,
                           int32_t drop_inactive, int64_t* kept);

/* ---- feature front-end (features.hpp, features.cpp:12-433) ------------------------
 * build_pyramid + detect_keypoints + extract_descriptors of the uploaded (or
 * staged) frame's color and depth, as Reconstructor::add_features / the sparse
 * term compute them (pipeline.cpp:97-101, 187-193): features with pixel, scale,
 * orientation and descriptor (positions and frame id are left 0 / -1).  A frame
 * without color or below 64x64 yields none.  n_keypoints = detect_keypoints'
 * count before descriptors drop flat / border patches. */
int wfk_detect_features(wfk_ctx* ctx, const wfk_feature_params* p, wfk_feature* out, int32_t cap,
                        int32_t* n_out, int32_t* n_keypoints);
/* one level of the last detection's pyramid (octave o, gaussian level l or DoG level l) */
int wfk_feature_pyramid_level(wfk_ctx* ctx, int32_t octave, int32_t level, int32_t dog, float* out,
                              int32_t* width, int32_t* height);
/* match_features (features.cpp:354-433; replaces features.hpp:107-110): the store
 * grouped by frame id (ascending), per group mutual-best matching of descriptors,
 * the max_candidates cap, the (distance, source id) sort, keep_best and the
 * descriptor / reprojection / 3-D prune.  predicted = 3 doubles per store entry
 * (z <= 0: no prediction).  Host arrays; computed on the device. */
int wfk_match_features(wfk_ctx* ctx, const wfk_feature* current, int32_t n_current, const wfk_feature* store,
                       int32_t n_store, const double* predicted, const wfk_intrinsics* intr,
                       const wfk_feature_params* p, wfk_feature_match* out, int32_t cap, int32_t* n_out);
/* the context's FeatureStore (features.hpp:79-95): filled by wfk_process_frame
 * when cfg->use_features; upload replaces it (FeatureStore::load / resume). */
int wfk_feature_store_upload(wfk_ctx* ctx, const wfk_feature* in, int64_t n);
int wfk_feature_store_download(wfk_ctx* ctx, wfk_feature* out, int64_t cap, int64_t* n_out);

/* ---- batched warp inversion ------------------------------------------------------
 * DeformableVolume::invert_warp (volume.hpp:89-94, volume.cpp:95-126) for n points
 * (host arrays, 3n doubles each): canonical x with warp_point(pose, x) == y from
 * seed, damped Gauss-Newton on the analytic trilinear Jacobian with Eigen's
 * PartialPivLU; ok[i] = 0 where the reference returns nullopt (x = 0). */
int wfk_invert_warp(wfk_ctx* ctx, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                    int32_t max_iters, double tol, double* x, uint8_t* ok);

/* ---- global pose ---------------------------------------------------------------
 * estimate_global_pose (solver.cpp:536-614; replaces solver.hpp:144-147): dense
 * projective point-to-plane ICP.  Sources are the valid samples of the context's
 * geometry buffer (the last wfk_rasterize) re-warped through the context's
 * volume; targets are looked up projectively in the context's frame maps (the
 * last wfk_backproject_depth).  Runs on the device without host round trips
 * (per iteration: one accumulation launch and one single-block update). */
int wfk_estimate_global_pose(wfk_ctx* ctx, const wfk_intrinsics* intr, const wfk_pose* initial,
                             const wfk_icp_params* params, wfk_icp_result* out);

/* ---- per-frame hot path (Reconstructor::process_frame, pipeline.cpp:143-262) --
 * With use_features the feature front-end runs on the device against the
 * context's FeatureStore (pipeline.cpp:95-141, 185-217); caller-supplied sparse
 * constraints are appended after the feature ones. */
typedef struct wfk_pipeline_config {
  wfk_solver_params solver;
  wfk_correspond_params correspond;
  wfk_fusion_params fusion;
  int32_t reassociations;
  int32_t estimate_pose;  /* global ICP before the solve (config.hpp:45, default on) */
  wfk_icp_params icp;     /* its corr is replaced by `correspond` (pipeline.cpp:176) */
  int32_t use_features;   /* sparse feature term + feature store (config.hpp:44, default on) */
  int32_t reserved_;
  wfk_feature_params features;
} wfk_pipeline_config;

typedef struct wfk_frame_record {
  wfk_energy energy;
  int32_t dense_count;
  int32_t sparse_count;
  int32_t anomalies;
  int32_t trace_len;
  int32_t pcg_iterations;
  int32_t bootstrap;
  wfk_fusion_stats fusion;
  wfk_expansion_stats expansion;
  wfk_pose pose;           /* the frame's global pose (after ICP) -- pass it to the next frame */
  int32_t icp_degraded;    /* FrameRecord::icp_degraded */
  int32_t icp_iterations;
  double icp_rms;          /* FrameRecord::icp_rms */
  int32_t match_count;     /* FrameRecord::match_count */
  int32_t features_added;  /* FrameRecord::features_added */
} wfk_frame_record;

/* frame_index 0 bootstraps (pipeline.cpp:150-159) and empties the feature store.  sparse may be NULL.  `pose`
 * is the pose entering the frame (the Reconstructor's pose_); the frame's pose,
 * refined by ICP when cfg->estimate_pose, is returned in rec->pose. */
int wfk_process_frame(wfk_ctx* ctx, const wfk_frame_view* frame, const wfk_pose* pose,
                      const wfk_pipeline_config* cfg, const wfk_correspondence* sparse,
                      int64_t nsparse, int32_t frame_index, wfk_frame_record* rec);

/* Stage a frame in device memory (slot >= 0), then run the per-frame path on it
 * with no host->device traffic (HBM-resident benchmark inputs). */
int wfk_frame_stage(wfk_ctx* ctx, int32_t slot, const wfk_frame_view* frame);
int wfk_process_staged_frame(wfk_ctx* ctx, int32_t slot, const wfk_pose* pose,
                             const wfk_pipeline_config* cfg, const wfk_correspondence* sparse,
                             int64_t nsparse, int32_t frame_index, wfk_frame_record* rec);

/* ---- measurement --------------------------------------------------------------
 * Device-event profiling of the context's stream: every flip-flop kernel
 * launch (the dominant kernel) with its algorithmic bytes, and the stages of
 * wfk_process_frame.  Enabling resets the counters. */
typedef struct wfk_profile {
  int64_t flip_flop_launches;
  int64_t pcg_iterations;
  double flip_flop_ms;          /* summed CUDA-event durations of the launches */
  double flip_flop_bytes;       /* algorithmic bytes, SURVEY.md 8(d) model */
  double flip_flop_bytes_impl;  /* algorithmic bytes of the fp64 layout */
  double stage_ms[8];           /* maps+mesh+raster, associate, solve, redeform, fuse, frame */
  int64_t launches;             /* kernel launches so far */
} wfk_profile;
int wfk_profile_enable(wfk_ctx* ctx, int32_t on);
int wfk_profile_read(wfk_ctx* ctx, wfk_profile* out);
/* CUDA events on the context's stream (16 slots) */
int wfk_timer_mark(wfk_ctx* ctx, int32_t slot);
int wfk_timer_elapsed_ms(wfk_ctx* ctx, int32_t a, int32_t b, double* ms);
/* write 256 MB on the context's stream so the next call starts with a cold L2 */
int wfk_flush_l2(wfk_ctx* ctx);
/* ---- checked mode -------------------------------------------------------------
 * With WFK_CHECK=1 in the environment when the library loads, every device
 * buffer is poisoned (0xff bytes) when allocated and carries a 256-byte canary
 * tail that every call verifies before it returns: a write past the end of any
 * device buffer fails that call with WFK_E_CUDA (the stand-in for
 * compute-sanitizer memcheck / initcheck, which the GPU pool does not offer).
 * wfk_check_enabled: 1 in checked mode.  wfk_debug_overrun: self-test of the
 * detector -- a kernel writes `past_end` bytes beyond the end of a context
 * scratch buffer (0: within it, and the buffer's canary is renewed). */
int wfk_check_enabled(void);
int wfk_debug_overrun(wfk_ctx* ctx, int32_t past_end);
/* page-locked host memory for frame buffers (cudaMallocHost) */
int wfk_host_alloc(size_t bytes, void** out);
void wfk_host_free(void* p);

#ifdef __cplusplus
}
#endif
