/* Plain-old-data types crossing the C ABI of the B200 non-rigid solver
 * (libwfk.so, include/wfk.h).  Every struct is the C image of one type of the
 * reference's wf:: interface.  Layout-compatible with the reference (storage
 * may cross without conversion; pinned by static_asserts in
 * integration/wf_b200_adapter.cpp): wfk_correspondence == wf::Correspondence,
 * and the volume / point-map / geometry-buffer / mesh arrays are the
 * reference's std::vector<Vec3/Vec3f/Vec3i/float/uint8_t> storage.  The other
 * structs (wfk_fusion_params, wfk_trace_entry, wfk_solver_params, ...) carry
 * the same fields in a C-friendly order and are converted field by field by
 * the adapter.
 *
 * No torch / CUDA / Eigen types appear here: plain pointers, sizes and
 * fixed-width integers only. */
#pragma once

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ adapter re-throws them as the exception types the
 * reference uses (SURVEY.md 8(b) "Errors"):
 *   INVALID_ARG  -> std::invalid_argument   (solver.cpp:458,466; volume.cpp:10-13)
 *   OUT_OF_RANGE -> std::out_of_range       (volume.cpp:37, trilinear_anchors)
 *   LOGIC        -> std::logic_error        (solver.cpp:352-353, inactive anchor)
 *   CUDA/OOM     -> std::runtime_error */
enum {
  WFK_OK = 0,
  WFK_E_INVALID_ARG = -1,
  WFK_E_OUT_OF_RANGE = -2,
  WFK_E_LOGIC = -3,
  WFK_E_CUDA = -4,
  WFK_E_NCCL = -5,
  WFK_E_OOM = -6,
  WFK_E_CAPACITY = -7 /* caller-provided output buffer too small */
};

/* wf::Exec (core.hpp:15-17).  The GPU path is deterministic for both. */
enum { WFK_EXEC_SERIAL = 0, WFK_EXEC_PARALLEL = 1 };

/* wf::Correspondence::Kind (correspond.hpp:15) */
enum { WFK_DENSE_PLANE = 0, WFK_SPARSE_POINT = 1 };

/* Borrowed view of a wf::DeformableVolume (volume.hpp:29-112).  Storage is the
 * reference's SoA-per-attribute layout, x-fastest linear index
 * (volume.hpp:40-42); 3-vectors are packed xyz triples exactly as
 * std::vector<Eigen::Vector3d/3f> lays them out. */
typedef struct wfk_volume_view {
  int32_t dims[3];
  int32_t reserved_;
  double voxel_size;
  double origin[3];
  double truncation; /* mu, 4 * voxel by default (volume.cpp:14) */
  float* tsdf;       /* n */
  float* weight;     /* n */
  float* color;      /* 3n */
  double* deformed;  /* 3n  t_i */
  double* euler;     /* 3n  (a, b, c), R = Rz(c) Ry(b) Rx(a) (core.hpp:33-35) */
  int32_t* age;      /* n */
  uint8_t* active;   /* n */
} wfk_volume_view;

/* Field masks for partial upload / download of a volume. */
enum {
  WFK_VOL_TSDF = 1u << 0,
  WFK_VOL_WEIGHT = 1u << 1,
  WFK_VOL_COLOR = 1u << 2,
  WFK_VOL_DEFORMED = 1u << 3,
  WFK_VOL_EULER = 1u << 4,
  WFK_VOL_AGE = 1u << 5,
  WFK_VOL_ACTIVE = 1u << 6,
  WFK_VOL_ALL = 0x7fu
};

/* wf::Correspondence (correspond.hpp:14-23); identical field order, 184 B. */
typedef struct wfk_correspondence {
  int32_t kind;
  int32_t reserved_;
  double canonical[3];
  int32_t anchor_index[8];
  double anchor_weight[8];
  double target[3];
  double target_normal[3];
  double confidence;
} wfk_correspondence;

/* wf::GlobalPose (core.hpp:20-31); rotation is ROW-major here. */
typedef struct wfk_pose {
  double rotation[9];
  double translation[3];
} wfk_pose;

/* wf::Intrinsics (core.hpp:41-58) */
typedef struct wfk_intrinsics {
  double fx, fy, cx, cy;
  int32_t width, height;
} wfk_intrinsics;

/* wf::SolverParams (solver.hpp:12-22) */
typedef struct wfk_solver_params {
  double w_d, w_s, w_r;
  int32_t flip_flop_iters;
  int32_t pcg_max_iters;
  double flip_flop_rel_tol;
  double pcg_tol;
  int32_t levels;
  int32_t exec;
} wfk_solver_params;

/* wf::EnergyBreakdown (solver.hpp:24-26) */
typedef struct wfk_energy {
  double total, sparse, dense, reg;
} wfk_energy;

/* wf::EnergyTraceEntry (solver.hpp:28-35) */
typedef struct wfk_trace_entry {
  int32_t level;
  int32_t iteration;
  wfk_energy energy;
  int32_t pcg_iterations;
  int32_t anomaly;
  double pcg_residual;
} wfk_trace_entry;

/* wf::PcgResult (solver.hpp:78-81) */
typedef struct wfk_pcg_result {
  int32_t iterations;
  int32_t reserved_;
  double relative_residual;
} wfk_pcg_result;

/* wf::FusionParams (fusion.hpp:10-15) */
typedef struct wfk_fusion_params {
  int32_t k_min;
  int32_t bootstrap;
  double w_max;
  double sample_weight;
} wfk_fusion_params;

/* wf::FusionStats (fusion.hpp:17-22) */
typedef struct wfk_fusion_stats {
  int32_t fused, skipped_gate, skipped_frustum, skipped_occluded;
} wfk_fusion_stats;

/* wf::ExpansionStats (fusion.hpp:30-33) */
typedef struct wfk_expansion_stats {
  int32_t activated, orphans;
} wfk_expansion_stats;

/* wf::CorrespondenceParams (correspond.hpp:25-29) */
typedef struct wfk_correspond_params {
  double eps_d, eps_n, eps_v;
} wfk_correspond_params;

/* wf::FeatureParams (features.hpp:29-45) */
typedef struct wfk_feature_params {
  int32_t octaves;          /* 4 */
  int32_t dog_levels;       /* 3 */
  double sigma0;            /* 1.6 */
  double contrast_threshold;/* 0.01 */
  double edge_ratio;        /* 10 */
  int32_t max_keypoints;    /* 150 */
  int32_t max_orientations; /* 2 */
  double orientation_peak_ratio; /* 0.8 */
  int32_t max_candidates;   /* 128 */
  int32_t keep_best;        /* 64 */
  double tau_descriptor;    /* 0.7 */
  double tau_pixels;        /* 48 */
  double tau_3d;            /* 0.10 */
} wfk_feature_params;

/* wf::Feature (features.hpp:13-22) */
typedef struct wfk_feature {
  double canonical_pos[3];
  double world_pos[3];
  double pixel[2];
  double scale;
  double orientation;
  float descriptor[128];
  int32_t frame_id;
  int32_t reserved_;
} wfk_feature;

/* wf::FeatureMatch (features.hpp) */
typedef struct wfk_feature_match {
  int32_t source_id;  /* store index */
  int32_t target_id;  /* current-frame feature index */
  double distance;
} wfk_feature_match;

/* wf::IcpParams (solver.hpp:121-131) */
typedef struct wfk_icp_params {
  wfk_correspond_params corr;   /* the pipeline copies its CorrespondenceParams in (pipeline.cpp:176) */
  int32_t max_iters;            /* 20 */
  int32_t min_correspondences;  /* 6 */
  double rel_tol;               /* 1e-6 */
  double min_improvement;       /* 0 */
} wfk_icp_params;

/* wf::IcpResult (solver.hpp:133-139) */
typedef struct wfk_icp_result {
  wfk_pose pose;
  int32_t converged;
  int32_t degraded;  /* too few correspondences, pose unchanged */
  double rms;
  int32_t iterations;
  int32_t reserved_;
} wfk_icp_result;

/* wf::Frame (image.hpp:31-35): depth in meters (0 = invalid), optional RGB. */
typedef struct wfk_frame_view {
  wfk_intrinsics intrinsics;
  const float* depth; /* width*height */
  const float* color; /* 3*width*height, or NULL when the frame has no color */
} wfk_frame_view;

/* wf::PointNormalMap (correspond.hpp:34-42) */
typedef struct wfk_point_normal_map {
  int32_t width, height;
  double* point;  /* 3*W*H */
  double* normal; /* 3*W*H */
  uint8_t* point_valid;
  uint8_t* normal_valid;
} wfk_point_normal_map;

/* wf::GeometryBuffer (isosurface.hpp:26-44) */
typedef struct wfk_geometry_buffer {
  int32_t width, height;
  float* depth;      /* W*H, +inf where empty */
  double* point;     /* 3*W*H */
  double* normal;    /* 3*W*H */
  double* canonical; /* 3*W*H */
} wfk_geometry_buffer;

/* wf::SurfaceMesh (isosurface.hpp:13-22) */
typedef struct wfk_mesh_view {
  int64_t num_vertices;
  int64_t num_triangles;
  double* vertices_canonical; /* 3V */
  double* vertices_deformed;  /* 3V */
  double* normals_deformed;   /* 3V (may be NULL before compute_normals) */
  float* colors;              /* 3V */
  int32_t* triangles;         /* 3T */
} wfk_mesh_view;

#ifdef __cplusplus
}
#endif
