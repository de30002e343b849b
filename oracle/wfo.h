/* ORACLE — test infrastructure only.
 *
 * C ABI of the CPU restatement of the reference hot path (oracle/wf_oracle.cpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load liboracle; the product (libwfk.so) never links
 * or calls it.  All functions return WFK_OK or a negative WFK_E_* code;
 * wfo_last_error() gives the message of the last failure on this thread. */
#pragma once

#include "../include/wfk_types.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* wfo_last_error(void);
int wfo_num_threads(void);
void wfo_set_num_threads(int n);

/* core.cpp:7-29 */
void wfo_euler_to_matrix(const double abc[3], double r_rowmajor[9]);
void wfo_matrix_to_euler(const double r_rowmajor[9], double abc[3]);
/* Eigen::JacobiSVD<Matrix3d> restatement used by update_rotations */
void wfo_svd3(const double a_rowmajor[9], double u[9], double s[3], double v[9]);

/* volume.cpp:27-66 */
int wfo_contains(const wfk_volume_view* v, const double x[3]);
int wfo_trilinear_anchors(const wfk_volume_view* v, const double x[3], int32_t idx[8],
                          double w[8]);
int wfo_warp_point(const wfk_volume_view* v, const wfk_pose* pose, const double x[3],
                   double out[3]);
/* reset a view's attribute arrays to DeformableVolume's constructor state
 * (volume.cpp:8-25) */
void wfo_volume_init(wfk_volume_view* v);

/* solver.cpp */
int wfo_compute_active_set(wfk_volume_view* v, int32_t* out_active, int64_t cap,
                           int64_t* n_out);

typedef struct wfo_ne wfo_ne; /* NormalEquations (solver.hpp:46-60) */
int wfo_build_normal_equations(const wfk_volume_view* v, const wfk_pose* pose,
                               const wfk_correspondence* cons, int64_t ncons,
                               const wfk_solver_params* params, wfo_ne** out);
int32_t wfo_ne_num_rows(const wfo_ne* ne);
/* blocks: rows*27*9 row-major 3x3; cols: rows*27; rhs: rows*3 */
void wfo_ne_export(const wfo_ne* ne, int32_t* rows, int32_t* node_row, double* blocks,
                   int32_t* cols, double* rhs, uint8_t* frozen);
void wfo_ne_multiply(const wfo_ne* ne, const double* x, double* y, int32_t exec);
double wfo_ne_symmetry_error(const wfo_ne* ne);
int wfo_ne_pcg_solve(const wfo_ne* ne, double* x, double tol, int32_t max_iters,
                     int32_t exec, wfk_pcg_result* out);
void wfo_ne_free(wfo_ne* ne);

int wfo_evaluate_energy(const wfk_volume_view* v, const wfk_pose* pose,
                        const wfk_correspondence* cons, int64_t ncons,
                        const wfk_solver_params* params, wfk_energy* out);
int wfo_update_rotations(wfk_volume_view* v, int32_t exec);
int wfo_flip_flop_solve(wfk_volume_view* v, const wfk_pose* pose,
                        const wfk_correspondence* cons, int64_t ncons,
                        const wfk_solver_params* params, int32_t level,
                        wfk_trace_entry* trace, int32_t cap, int32_t* n_out);
/* build_hierarchy (solver.cpp:455-503): per level dims, voxel, active count,
 * and the re-anchored constraints of one level (level_out may be NULL). */
int wfo_hierarchy_info(const wfk_volume_view* v, const wfk_correspondence* cons,
                       int64_t ncons, int32_t levels, int32_t* dims_out /*3*levels*/,
                       int64_t* active_out /*levels*/, int32_t want_level,
                       wfk_correspondence* level_cons_out);
int wfo_solve_coarse_to_fine(wfk_volume_view* v, const wfk_pose* pose,
                             const wfk_correspondence* cons, int64_t ncons,
                             const wfk_solver_params* params, wfk_trace_entry* trace,
                             int32_t cap, int32_t* n_out);

/* fusion.cpp */
int wfo_integrate_frame(wfk_volume_view* v, const wfk_frame_view* frame,
                        const wfk_pose* pose, const wfk_fusion_params* params,
                        int32_t exec, wfk_fusion_stats* out);
int wfo_expand_grid(wfk_volume_view* v, wfk_expansion_stats* out);
int wfo_advance_ages(wfk_volume_view* v, const int32_t* idx, int64_t n);

/* correspond.cpp */
int wfo_backproject_depth(const wfk_frame_view* frame, int32_t exec,
                          wfk_point_normal_map* out);
double wfo_dense_confidence(double dist, double normal_dot, double view_dot,
                            const wfk_correspond_params* p);
int wfo_sample_point_normal(const wfk_point_normal_map* maps, const double uv[2],
                            double point[3], double normal[3]);
int wfo_find_dense_correspondences(const wfk_geometry_buffer* buf,
                                   const wfk_point_normal_map* maps,
                                   const wfk_intrinsics* intr,
                                   const wfk_correspond_params* params,
                                   const wfk_volume_view* v, wfk_correspondence* out,
                                   int64_t cap, int64_t* n_out);
/* solver.cpp:536-614 */
int wfo_estimate_global_pose(const wfk_geometry_buffer* buf, const wfk_point_normal_map* maps,
                             const wfk_intrinsics* intr, const wfk_volume_view* v, const wfk_pose* initial,
                             const wfk_icp_params* params, wfk_icp_result* out);
/* feature front-end (features.cpp, wf_features.cpp) */
int wfo_detect_features(const wfk_frame_view* frame, const wfk_feature_params* p, wfk_feature* out, int32_t cap,
                        int32_t* n_out, int32_t* n_keypoints);
int wfo_pyramid_level(const wfk_frame_view* frame, const wfk_feature_params* p, int32_t o, int32_t l,
                      int32_t dog, float* out, int32_t* w_out, int32_t* h_out);
double wfo_descriptor_distance(const float* a, const float* b);
int wfo_match_features(const wfk_feature* cur, int32_t nc, const wfk_feature* store, int32_t ns,
                       const double* predicted_world, const wfk_intrinsics* K, const wfk_feature_params* p,
                       wfk_feature_match* out, int32_t cap, int32_t* n_out);

/* DeformableVolume::invert_warp (volume.cpp:95-126) for n points; x = 0, ok = 0 on failure */
int wfo_invert_warp(const wfk_volume_view* v, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                    int32_t max_iters, double tol, double* x, uint8_t* ok);
/* Eigen LDLT<MatrixXd> (symmetric pivoting) restated, n <= 8: solves A x = b */
int wfo_ldlt_solve(int n, const double* a, const double* b, double* x);
int wfo_sparse_to_constraints(const double* canonical, const double* target, int64_t n,
                              const wfk_volume_view* v, wfk_correspondence* out,
                              int64_t* n_out);

/* isosurface.cpp / rasterize.cpp; the mesh is an oracle-owned handle */
typedef struct wfo_mesh wfo_mesh;
int wfo_extract_mesh(const wfk_volume_view* v, const wfk_pose* pose, wfo_mesh** out);
void wfo_mesh_sizes(const wfo_mesh* m, int64_t* nv, int64_t* nt);
void wfo_mesh_export(const wfo_mesh* m, wfk_mesh_view* out); /* copies into out's arrays */
int wfo_mesh_import(const wfk_mesh_view* in, wfo_mesh** out);
int wfo_mesh_warp(wfo_mesh* m, const wfk_volume_view* v, const wfk_pose* pose);
void wfo_compute_normals(wfo_mesh* m);
int wfo_rasterize(const wfo_mesh* m, const wfk_intrinsics* intr, int32_t exec,
                  wfk_geometry_buffer* out);
void wfo_mesh_free(wfo_mesh* m);

/* Reconstructor::process_frame (pipeline.cpp:143-262): global ICP when
 * estimate_pose, the feature front-end and FeatureStore when use_features
 * (pipeline.cpp:95-141, 185-217); caller-supplied sparse constraints are
 * appended after the feature ones. */
typedef struct wfo_recon_config {
  int32_t dims[3];
  int32_t reassociations;
  double voxel_size;
  double origin[3];
  wfk_solver_params solver;
  wfk_correspond_params correspond;
  wfk_fusion_params fusion;
  int32_t estimate_pose;
  int32_t reserved_;
  wfk_icp_params icp;
  int32_t use_features;
  int32_t reserved2_;
  wfk_feature_params features;
} wfo_recon_config;

typedef struct wfo_frame_record {
  wfk_energy energy;
  int32_t dense_count;
  int32_t sparse_count;
  int32_t anomalies;
  int32_t trace_len;
  int32_t pcg_iterations; /* summed over the trace */
  int32_t reserved_;
  wfk_fusion_stats fusion;
  wfk_expansion_stats expansion;
  wfk_pose pose;
  int32_t icp_degraded;
  int32_t icp_iterations;
  double icp_rms;
  int32_t match_count;
  int32_t features_added;
} wfo_frame_record;

typedef struct wfo_recon wfo_recon;
int wfo_recon_create(const wfo_recon_config* cfg, wfo_recon** out);
void wfo_recon_free(wfo_recon* r);
/* volume arrays owned by the reconstructor, borrowed */
void wfo_recon_volume(wfo_recon* r, wfk_volume_view* out);
int wfo_recon_process_frame(wfo_recon* r, const wfk_frame_view* frame,
                            const wfk_correspondence* sparse, int64_t nsparse,
                            wfo_frame_record* rec);
/* the reconstructor's FeatureStore (copies n_out <= cap entries when out != NULL) */
int wfo_recon_feature_store(const wfo_recon* r, wfk_feature* out, int64_t cap, int64_t* n_out);

/* snapshot / frame formats (wf_formats.cpp): volume.cpp:150-217,
 * features.cpp:306-352, image.cpp:21-121 */
int wfo_volume_save_bytes(const wfk_volume_view* v, uint8_t* out, int64_t cap, int64_t* n_out);
int wfo_volume_load_bytes(const uint8_t* in, int64_t n, wfk_volume_view* v);
int wfo_feature_store_bytes(const wfk_feature* f, int32_t nf, uint8_t* out, int64_t cap, int64_t* n_out);
int wfo_pgm_encode(const float* depth, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out);
int wfo_ppm_encode(const float* color, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out);
int wfo_pnm_decode(const uint8_t* in, int64_t n, int32_t channels, int32_t* w, int32_t* h, float* out);

#ifdef __cplusplus
}
#endif
