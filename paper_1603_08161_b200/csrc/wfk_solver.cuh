// Host-side entry points of the device solver (solver.cu), used by api.cu.
#pragma once

#include <vector>

#include "wfk_context.cuh"

namespace wfk {

PoseD pose_dev(const wfk_pose* p);
void solver_flip_flop(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, int level_tag,
                      std::vector<wfk_trace_entry>& trace);
void solver_energy(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, wfk_energy* e);
void solver_rotations(wfk_ctx* c);
void solver_c2f(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, std::vector<wfk_trace_entry>& trace);
void solver_hierarchy_info(wfk_ctx* c, int levels, int32_t* dims, int64_t* active);
// slab plan of the in-kernel partitioned CG (host part, solver.cu): tile
// count, tile bounds from the inclusive row-work prefix, rank split
int slab_tile_count(int N, int G, int tpb);
int slab_tile_bound_host(int t, int ntiles, int N, const int32_t* incl);
void slab_split(int ntiles, int S, int32_t* rank_tile);
int solver_build_ne(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, wfk_ne_host* out);
void solver_pcg_assembled(wfk_ctx* c, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x,
                          double tol, int max_iters, int mode, wfk_pcg_result* res, double* y);

// fusion.cu
void fusion_compute_active_set(wfk_ctx* c, int32_t* out, int64_t cap, int64_t* n_out);
void fusion_integrate(wfk_ctx* c, const wfk_pose* pose, const wfk_fusion_params& p, wfk_fusion_stats* out);
void fusion_expand(wfk_ctx* c, wfk_expansion_stats* out);
void fusion_advance_ages(wfk_ctx* c, const int32_t* idx, int64_t n);
void fusion_advance_active_ages(wfk_ctx* c);

// assoc.cu
void assoc_backproject(wfk_ctx* c, wfk_point_normal_map* out);
void assoc_extract_mesh(wfk_ctx* c, const wfk_pose* pose, int64_t* nv, int64_t* nt);
void assoc_mesh_warp(wfk_ctx* c, const wfk_pose* pose);
void assoc_compute_normals(wfk_ctx* c);
void assoc_rasterize(wfk_ctx* c, const wfk_intrinsics& K, wfk_geometry_buffer* out);
void features_detect(wfk_ctx* c, const wfk_feature_params& p, wfk_feature* out, int32_t cap, int32_t* n_out,
                     int32_t* n_kp_out);
void features_level(wfk_ctx* c, int o, int l, int dog, float* out, int32_t* w, int32_t* h);
void features_match_dev(wfk_ctx* c, const wfk_feature* cur, int nc, const wfk_feature* st, int64_t ns,
                        const double* pred, const wfk_intrinsics& K, const wfk_feature_params& p,
                        int64_t max_group);
void features_match_host(wfk_ctx* c, const wfk_feature* cur, int32_t nc, const wfk_feature* st, int32_t ns,
                         const double* pred, const wfk_intrinsics& K, const wfk_feature_params& p,
                         wfk_feature_match* out, int32_t cap, int32_t* n_out);
void features_frame_sparse(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& pose, const wfk_feature_params& p,
                           int32_t* match_count);
int64_t features_append_sparse(wfk_ctx* c);
int32_t features_add(wfk_ctx* c, const wfk_pose& pose, int32_t frame_id, bool bootstrap);
int64_t volume_image_bytes(wfk_ctx* c);
void volume_pack(wfk_ctx* c, uint8_t* out, int64_t cap, int64_t* n_out);
void volume_unpack(wfk_ctx* c, const uint8_t* in, int64_t n);
void volume_save(wfk_ctx* c, const char* path);
void volume_load(wfk_ctx* c, const char* path);
void feature_store_save(wfk_ctx* c, const char* path);
void feature_store_load(wfk_ctx* c, const char* path);
void frame_load_pnm(wfk_ctx* c, const char* depth_path, const char* color_path, const wfk_intrinsics& K);
void frame_save_pnm(wfk_ctx* c, const char* depth_path, const char* color_path);
void frame_download(wfk_ctx* c, float* depth, float* color);
void dist_destroy(wfk_ctx* c);
void dist_forget(wfk_ctx* c);
void dist_pcg_device(wfk_ctx* c, int slabs, int N, const double* blocks, const int32_t* cols, const double* rhs,
                     double* x, double tol, int max_iters, const void* plan_key, bool fresh, wfk_pcg_result* res);
void solver_c2f_dist(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, int slabs,
                     std::vector<wfk_trace_entry>& trace);
void dist_unique_id(uint8_t* out);
void dist_init(wfk_ctx* c, int rank, int world, const uint8_t* id_bytes);
void dist_plan(int N, const int32_t* cols, int world, int32_t* ranges, int32_t* xfers, int32_t cap, int32_t* n_xfers);
void dist_pcg(wfk_ctx* c, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x, double tol,
              int max_iters, wfk_pcg_result* res);
void slabs_pcg(wfk_ctx* c, int slabs, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x,
               double tol, int max_iters, wfk_pcg_result* res);
void features_store_upload(wfk_ctx* c, const wfk_feature* in, int64_t n);
void features_store_download(wfk_ctx* c, wfk_feature* out, int64_t cap, int64_t* n_out);
void volume_invert_warp(wfk_ctx* c, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                        int32_t max_iters, double tol, double* x, uint8_t* ok);
void assoc_estimate_pose(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& initial, const wfk_icp_params& prm,
                         wfk_icp_result* out);
void assoc_estimate_pose_begin(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& initial,
                               const wfk_icp_params& prm);
void assoc_estimate_pose_end(wfk_ctx* c, wfk_icp_result* out);
void assoc_find_dense(wfk_ctx* c, const wfk_intrinsics& K, const wfk_correspond_params& p, bool drop_inactive,
                      int64_t* n_out);

}  // namespace wfk
