// ORACLE (test infrastructure): the wfo_* C ABI of oracle/wfo.h implemented
// over the REFERENCE ITSELF — the unmodified wf:: library compiled from
// /root/reference/proj/src (oracle/ref/Makefile).  tests/ load it as
// oracle/_ref/libwfref.so in place of the restatement (oracle/pyoracle.py,
// WF_ORACLE=ref), so every parity test can run against the reference's own
// code.  Conversions only: every computation is a call into wf::.
//
// Entry points the reference has no public function for return
// WFK_E_INVALID_ARG with "not available in the reference build"
// (wfo_svd3 is answered by the Eigen shim's JacobiSVD, which is what the
// reference's update_rotations calls).
#include <omp.h>

#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>  // ios_base::Init: libstdc++ is linked statically into the .so
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unistd.h>
#include <vector>

#include "../../tools/synthscene.h"
#include "../wfo.h"
#include "wf/correspond.hpp"
#include "wf/features.hpp"
#include "wf/fusion.hpp"
#include "wf/image.hpp"
#include "wf/isosurface.hpp"
#include "wf/pipeline.hpp"
#include "wf/solver.hpp"
#include "wf/synthcam.hpp"
#include "wf/volume.hpp"

using namespace wf;

namespace {
// libstdc++ is linked statically into this .so (this image's toolchain): make
// sure its stream / locale state is initialised before the reference's
// formatted file writers run inside a host process that has no libstdc++
const std::ios_base::Init g_ios_init;
thread_local std::string g_err;
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
Exec exec_of(int32_t e) { return e == WFK_EXEC_SERIAL ? Exec::Serial : Exec::Parallel; }

Vec3 v3(const double* p) { return Vec3(p[0], p[1], p[2]); }
void put(const Vec3& v, double* p) {
  p[0] = v.x();
  p[1] = v.y();
  p[2] = v.z();
}
Mat3 m3_rowmajor(const double* p) {
  Mat3 m;
  for (int i = 0; i < 9; ++i) m(i / 3, i % 3) = p[i];
  return m;
}
void put_rowmajor(const Mat3& m, double* p) {
  for (int i = 0; i < 9; ++i) p[i] = m(i / 3, i % 3);
}
GlobalPose pose_of(const wfk_pose* p) {
  GlobalPose g;
  if (p) {
    g.rotation = m3_rowmajor(p->rotation);
    g.translation = v3(p->translation);
  }
  return g;
}
void pose_to_c(const GlobalPose& g, wfk_pose* o) {
  put_rowmajor(g.rotation, o->rotation);
  put(g.translation, o->translation);
}
Intrinsics intr_of(const wfk_intrinsics& k) {
  Intrinsics i;
  i.fx = k.fx;
  i.fy = k.fy;
  i.cx = k.cx;
  i.cy = k.cy;
  i.width = k.width;
  i.height = k.height;
  return i;
}
SolverParams params_of(const wfk_solver_params* p) {
  SolverParams s;
  s.w_d = p->w_d;
  s.w_s = p->w_s;
  s.w_r = p->w_r;
  s.flip_flop_iters = p->flip_flop_iters;
  s.pcg_max_iters = p->pcg_max_iters;
  s.flip_flop_rel_tol = p->flip_flop_rel_tol;
  s.pcg_tol = p->pcg_tol;
  s.levels = p->levels;
  s.exec = exec_of(p->exec);
  return s;
}
CorrespondenceParams cparams_of(const wfk_correspond_params& c) {
  CorrespondenceParams p;
  p.eps_d = c.eps_d;
  p.eps_n = c.eps_n;
  p.eps_v = c.eps_v;
  return p;
}
FusionParams fparams_of(const wfk_fusion_params& f) {
  FusionParams p;
  p.k_min = f.k_min;
  p.bootstrap = f.bootstrap != 0;
  p.w_max = f.w_max;
  p.sample_weight = f.sample_weight;
  return p;
}
FeatureParams featparams_of(const wfk_feature_params& q) {
  FeatureParams p;
  p.octaves = q.octaves;
  p.dog_levels = q.dog_levels;
  p.sigma0 = q.sigma0;
  p.contrast_threshold = q.contrast_threshold;
  p.edge_ratio = q.edge_ratio;
  p.max_keypoints = q.max_keypoints;
  p.max_orientations = q.max_orientations;
  p.orientation_peak_ratio = q.orientation_peak_ratio;
  p.max_candidates = q.max_candidates;
  p.keep_best = q.keep_best;
  p.tau_descriptor = q.tau_descriptor;
  p.tau_pixels = q.tau_pixels;
  p.tau_3d = q.tau_3d;
  return p;
}
IcpParams icpparams_of(const wfk_icp_params& q) {
  IcpParams p;
  p.corr = cparams_of(q.corr);
  p.max_iters = q.max_iters;
  p.min_correspondences = q.min_correspondences;
  p.rel_tol = q.rel_tol;
  p.min_improvement = q.min_improvement;
  return p;
}

// ---- DeformableVolume <-> borrowed SoA view ----
DeformableVolume vol_of(const wfk_volume_view* v) {
  DeformableVolume d(Vec3i(v->dims[0], v->dims[1], v->dims[2]), v->voxel_size, v3(v->origin));
  d.set_truncation(v->truncation);
  const int n = d.num_points();
  for (int i = 0; i < n; ++i) {
    d.tsdf(i) = v->tsdf[i];
    d.weight(i) = v->weight[i];
    d.color(i) = Vec3f(v->color[3 * i], v->color[3 * i + 1], v->color[3 * i + 2]);
    d.deformed(i) = v3(v->deformed + 3 * size_t(i));
    d.euler(i) = v3(v->euler + 3 * size_t(i));
    d.age(i) = v->age[i];
    d.set_active(i, v->active[i] != 0);
  }
  return d;
}
void vol_to(const DeformableVolume& d, wfk_volume_view* v) {
  const int n = d.num_points();
  v->truncation = d.truncation();
  for (int i = 0; i < n; ++i) {
    v->tsdf[i] = d.tsdf(i);
    v->weight[i] = d.weight(i);
    for (int k = 0; k < 3; ++k) v->color[3 * i + k] = d.color(i)[k];
    put(d.deformed(i), v->deformed + 3 * size_t(i));
    put(d.euler(i), v->euler + 3 * size_t(i));
    v->age[i] = d.age(i);
    v->active[i] = d.active(i) ? 1 : 0;
  }
}

Correspondence con_of(const wfk_correspondence& c) {
  Correspondence o;
  o.kind = c.kind == WFK_SPARSE_POINT ? Correspondence::Kind::SparsePoint : Correspondence::Kind::DensePlane;
  o.canonical = v3(c.canonical);
  for (int k = 0; k < 8; ++k) {
    o.anchor_index[size_t(k)] = c.anchor_index[k];
    o.anchor_weight[size_t(k)] = c.anchor_weight[k];
  }
  o.target = v3(c.target);
  o.target_normal = v3(c.target_normal);
  o.confidence = c.confidence;
  return o;
}
void con_to(const Correspondence& c, wfk_correspondence& o) {
  std::memset(&o, 0, sizeof(o));
  o.kind = c.kind == Correspondence::Kind::SparsePoint ? WFK_SPARSE_POINT : WFK_DENSE_PLANE;
  put(c.canonical, o.canonical);
  for (int k = 0; k < 8; ++k) {
    o.anchor_index[k] = c.anchor_index[size_t(k)];
    o.anchor_weight[k] = c.anchor_weight[size_t(k)];
  }
  put(c.target, o.target);
  put(c.target_normal, o.target_normal);
  o.confidence = c.confidence;
}
std::vector<Correspondence> cons_of(const wfk_correspondence* c, int64_t n) {
  std::vector<Correspondence> v;
  v.reserve(size_t(n));
  for (int64_t i = 0; i < n; ++i) v.push_back(con_of(c[i]));
  return v;
}
void fill_energy(const EnergyBreakdown& e, wfk_energy* o) {
  o->total = e.total;
  o->sparse = e.sparse;
  o->dense = e.dense;
  o->reg = e.reg;
}
int export_trace(const std::vector<EnergyTraceEntry>& t, wfk_trace_entry* out, int32_t cap, int32_t* n_out) {
  if (n_out) *n_out = int32_t(t.size());
  if (int32_t(t.size()) > cap) return fail(WFK_E_CAPACITY, "trace buffer too small");
  for (size_t i = 0; i < t.size(); ++i) {
    wfk_trace_entry& o = out[i];
    std::memset(&o, 0, sizeof(o));
    o.level = t[i].level;
    o.iteration = t[i].iteration;
    fill_energy(t[i].energy, &o.energy);
    o.pcg_iterations = t[i].pcg_iterations;
    o.anomaly = t[i].anomaly ? 1 : 0;
    o.pcg_residual = t[i].pcg_residual;
  }
  return WFK_OK;
}
Frame frame_of(const wfk_frame_view* f) {
  Frame o;
  o.intrinsics = intr_of(f->intrinsics);
  const int w = f->intrinsics.width, h = f->intrinsics.height;
  o.depth = DepthImage(w, h);
  std::memcpy(o.depth.data.data(), f->depth, size_t(w) * size_t(h) * sizeof(float));
  if (f->color) {
    o.color = ColorImage(w, h);
    for (size_t i = 0; i < size_t(w) * size_t(h); ++i)
      o.color.data[i] = Vec3f(f->color[3 * i], f->color[3 * i + 1], f->color[3 * i + 2]);
  }
  return o;
}
PointNormalMap maps_of(const wfk_point_normal_map* m) {
  PointNormalMap p;
  p.width = m->width;
  p.height = m->height;
  const size_t n = size_t(m->width) * size_t(m->height);
  p.point.resize(n);
  p.normal.resize(n);
  p.point_valid.assign(m->point_valid, m->point_valid + n);
  p.normal_valid.assign(m->normal_valid, m->normal_valid + n);
  for (size_t i = 0; i < n; ++i) {
    p.point[i] = v3(m->point + 3 * i);
    p.normal[i] = v3(m->normal + 3 * i);
  }
  return p;
}
GeometryBuffer gbuf_of(const wfk_geometry_buffer* b) {
  GeometryBuffer g(b->width, b->height);
  const size_t n = size_t(b->width) * size_t(b->height);
  for (size_t i = 0; i < n; ++i) {
    g.depth[i] = b->depth[i];
    g.point[i] = v3(b->point + 3 * i);
    g.normal[i] = v3(b->normal + 3 * i);
    g.canonical[i] = v3(b->canonical + 3 * i);
  }
  return g;
}
void gbuf_to(const GeometryBuffer& g, wfk_geometry_buffer* b) {
  b->width = g.width;
  b->height = g.height;
  const size_t n = size_t(g.width) * size_t(g.height);
  for (size_t i = 0; i < n; ++i) {
    b->depth[i] = g.depth[i];
    put(g.point[i], b->point + 3 * i);
    put(g.normal[i], b->normal + 3 * i);
    put(g.canonical[i], b->canonical + 3 * i);
  }
}
wfk_feature feature_to(const Feature& f) {
  wfk_feature o;
  std::memset(&o, 0, sizeof(o));
  put(f.canonical_pos, o.canonical_pos);
  put(f.world_pos, o.world_pos);
  o.pixel[0] = f.pixel.x();
  o.pixel[1] = f.pixel.y();
  o.scale = f.scale;
  o.orientation = f.orientation;
  std::memcpy(o.descriptor, f.descriptor.data(), sizeof(o.descriptor));
  o.frame_id = f.frame_id;
  return o;
}
Feature feature_of(const wfk_feature& f) {
  Feature o;
  o.canonical_pos = v3(f.canonical_pos);
  o.world_pos = v3(f.world_pos);
  o.pixel = Vec2(f.pixel[0], f.pixel[1]);
  o.scale = f.scale;
  o.orientation = f.orientation;
  std::memcpy(o.descriptor.data(), f.descriptor, sizeof(f.descriptor));
  o.frame_id = f.frame_id;
  return o;
}

// map every reference exception onto the ABI's status codes
template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    return fail(WFK_E_INVALID_ARG, e.what());
  } catch (const std::out_of_range& e) {
    return fail(WFK_E_OUT_OF_RANGE, e.what());
  } catch (const std::logic_error& e) {
    return fail(WFK_E_LOGIC, e.what());
  } catch (const std::exception& e) {
    return fail(WFK_E_INVALID_ARG, e.what());
  }
}

std::string temp_path(const char* tag) {
  static int counter = 0;
  char buf[256];
  std::snprintf(buf, sizeof(buf), "/tmp/wfref_%d_%d_%s", int(getpid()), counter++, tag);
  return buf;
}
std::vector<uint8_t> read_file(const std::string& p) {
  std::ifstream is(p, std::ios::binary);
  return std::vector<uint8_t>((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
}
void write_file(const std::string& p, const uint8_t* d, int64_t n) {
  std::ofstream os(p, std::ios::binary);
  os.write(reinterpret_cast<const char*>(d), n);
}
int copy_out(const std::vector<uint8_t>& bytes, uint8_t* out, int64_t cap, int64_t* n_out) {
  *n_out = int64_t(bytes.size());
  if (!out) return WFK_OK;
  if (int64_t(bytes.size()) > cap) return fail(WFK_E_CAPACITY, "byte buffer too small");
  std::memcpy(out, bytes.data(), bytes.size());
  return WFK_OK;
}
}  // namespace

struct wfo_ne {
  NormalEquations ne;
};
struct wfo_mesh {
  SurfaceMesh m;
};
struct wfo_recon {
  explicit wfo_recon(const ReconstructionConfig& c) : r(c) {}
  Reconstructor r;
};

extern "C" {

const char* wfo_last_error(void) { return g_err.c_str(); }
int wfo_num_threads(void) { return omp_get_max_threads(); }
void wfo_set_num_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}
int wfo_is_reference(void) { return 1; }

void wfo_euler_to_matrix(const double abc[3], double r[9]) { put_rowmajor(euler_to_matrix(v3(abc)), r); }
void wfo_matrix_to_euler(const double r[9], double abc[3]) { put(matrix_to_euler(m3_rowmajor(r)), abc); }
void wfo_svd3(const double a[9], double u[9], double s[3], double v[9]) {
  Eigen::JacobiSVD<Mat3> svd(m3_rowmajor(a), Eigen::ComputeFullU | Eigen::ComputeFullV);
  put_rowmajor(svd.matrixU(), u);
  put_rowmajor(svd.matrixV(), v);
  put(svd.singularValues(), s);
}

void wfo_volume_init(wfk_volume_view* view) {
  const DeformableVolume d(Vec3i(view->dims[0], view->dims[1], view->dims[2]), view->voxel_size, v3(view->origin));
  vol_to(d, view);
}
int wfo_contains(const wfk_volume_view* view, const double x[3]) {
  // geometry only: an attribute-free volume of the same lattice
  const DeformableVolume d(Vec3i(view->dims[0], view->dims[1], view->dims[2]), view->voxel_size, v3(view->origin));
  return d.contains(v3(x)) ? 1 : 0;
}
int wfo_trilinear_anchors(const wfk_volume_view* view, const double x[3], int32_t idx[8], double w[8]) {
  return guarded([&]() -> int {
    const DeformableVolume d(Vec3i(view->dims[0], view->dims[1], view->dims[2]), view->voxel_size,
                             v3(view->origin));
    const TrilinearAnchors a = d.trilinear_anchors(v3(x));
    for (int k = 0; k < 8; ++k) {
      idx[k] = a.index[size_t(k)];
      w[k] = a.weight[size_t(k)];
    }
    return WFK_OK;
  });
}
int wfo_warp_point(const wfk_volume_view* view, const wfk_pose* pose, const double x[3], double out[3]) {
  return guarded([&]() -> int {
    const DeformableVolume d = vol_of(view);
    put(d.warp_point(pose_of(pose), v3(x)), out);
    return WFK_OK;
  });
}

int wfo_compute_active_set(wfk_volume_view* view, int32_t* out, int64_t cap, int64_t* n_out) {
  DeformableVolume d = vol_of(view);
  const std::vector<int> a = compute_active_set(d);
  vol_to(d, view);
  if (n_out) *n_out = int64_t(a.size());
  if (out) {
    if (int64_t(a.size()) > cap) return fail(WFK_E_CAPACITY, "active list buffer too small");
    std::copy(a.begin(), a.end(), out);
  }
  return WFK_OK;
}

int wfo_build_normal_equations(const wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons,
                               int64_t ncons, const wfk_solver_params* params, wfo_ne** out) {
  return guarded([&]() -> int {
    const DeformableVolume d = vol_of(view);
    auto* ne = new wfo_ne;
    ne->ne = build_normal_equations(d, pose_of(pose), cons_of(cons, ncons), params_of(params), nullptr);
    *out = ne;
    return WFK_OK;
  });
}
int32_t wfo_ne_num_rows(const wfo_ne* ne) { return ne->ne.num_rows(); }
void wfo_ne_export(const wfo_ne* p, int32_t* rows, int32_t* node_row, double* blocks, int32_t* cols, double* rhs,
                   uint8_t* frozen) {
  const NormalEquations& ne = p->ne;
  const int n = ne.num_rows();
  if (rows) std::copy(ne.rows.begin(), ne.rows.end(), rows);
  if (node_row) std::copy(ne.node_row.begin(), ne.node_row.end(), node_row);
  for (int r = 0; r < n; ++r) {
    for (int s = 0; s < 27; ++s) {
      if (blocks) put_rowmajor(ne.blocks[size_t(r)][size_t(s)], blocks + (size_t(r) * 27 + size_t(s)) * 9);
      if (cols) cols[size_t(r) * 27 + size_t(s)] = ne.cols[size_t(r)][size_t(s)];
    }
    if (rhs) put(ne.rhs[size_t(r)], rhs + 3 * size_t(r));
    if (frozen) frozen[r] = ne.frozen[size_t(r)];
  }
}
void wfo_ne_multiply(const wfo_ne* p, const double* x, double* y, int32_t exec) {
  const int n = p->ne.num_rows();
  std::vector<Vec3> xv(static_cast<size_t>(n)), yv;
  for (int i = 0; i < n; ++i) xv[size_t(i)] = v3(x + 3 * i);
  p->ne.multiply(xv, yv, exec_of(exec));
  for (int i = 0; i < n; ++i) put(yv[size_t(i)], y + 3 * i);
}
double wfo_ne_symmetry_error(const wfo_ne* p) { return p->ne.symmetry_error(); }
int wfo_ne_pcg_solve(const wfo_ne* p, double* x, double tol, int32_t max_iters, int32_t exec, wfk_pcg_result* out) {
  const int n = p->ne.num_rows();
  std::vector<Vec3> xv(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) xv[size_t(i)] = v3(x + 3 * i);
  const PcgResult r = pcg_solve(p->ne, xv, tol, max_iters, exec_of(exec));
  for (int i = 0; i < n; ++i) put(xv[size_t(i)], x + 3 * i);
  if (out) {
    out->iterations = r.iterations;
    out->relative_residual = r.relative_residual;
  }
  return WFK_OK;
}
void wfo_ne_free(wfo_ne* ne) { delete ne; }

int wfo_evaluate_energy(const wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons,
                        int64_t ncons, const wfk_solver_params* params, wfk_energy* out) {
  return guarded([&]() -> int {
    const DeformableVolume d = vol_of(view);
    fill_energy(evaluate_energy(d, pose_of(pose), cons_of(cons, ncons), params_of(params)), out);
    return WFK_OK;
  });
}
int wfo_update_rotations(wfk_volume_view* view, int32_t exec) {
  DeformableVolume d = vol_of(view);
  update_rotations(d, exec_of(exec));
  vol_to(d, view);
  return WFK_OK;
}
int wfo_flip_flop_solve(wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons, int64_t ncons,
                        const wfk_solver_params* params, int32_t level, wfk_trace_entry* trace, int32_t cap,
                        int32_t* n_out) {
  return guarded([&]() -> int {
    DeformableVolume d = vol_of(view);
    const auto t = flip_flop_solve(d, pose_of(pose), cons_of(cons, ncons), params_of(params), level);
    vol_to(d, view);
    return export_trace(t, trace, cap, n_out);
  });
}
int wfo_hierarchy_info(const wfk_volume_view* view, const wfk_correspondence* cons, int64_t ncons, int32_t levels,
                       int32_t* dims_out, int64_t* active_out, int32_t want_level,
                       wfk_correspondence* level_cons_out) {
  return guarded([&]() -> int {
    const DeformableVolume d = vol_of(view);
    const auto h = build_hierarchy(d, cons_of(cons, ncons), levels);
    for (size_t l = 0; l < h.size(); ++l) {
      if (dims_out)
        for (int k = 0; k < 3; ++k) dims_out[3 * l + size_t(k)] = h[l].grid.dims()[k];
      if (active_out) {
        int64_t a = 0;
        for (int i = 0; i < h[l].grid.num_points(); ++i) a += h[l].grid.active(i) ? 1 : 0;
        active_out[l] = a;
      }
    }
    if (level_cons_out && want_level >= 0 && want_level < int(h.size()))
      for (size_t i = 0; i < h[size_t(want_level)].constraints.size(); ++i)
        con_to(h[size_t(want_level)].constraints[i], level_cons_out[i]);
    return WFK_OK;
  });
}
int wfo_solve_coarse_to_fine(wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons,
                             int64_t ncons, const wfk_solver_params* params, wfk_trace_entry* trace, int32_t cap,
                             int32_t* n_out) {
  return guarded([&]() -> int {
    DeformableVolume d = vol_of(view);
    const auto t = solve_coarse_to_fine(d, pose_of(pose), cons_of(cons, ncons), params_of(params));
    vol_to(d, view);
    return export_trace(t, trace, cap, n_out);
  });
}

int wfo_integrate_frame(wfk_volume_view* view, const wfk_frame_view* frame, const wfk_pose* pose,
                        const wfk_fusion_params* params, int32_t exec, wfk_fusion_stats* out) {
  return guarded([&]() -> int {
    DeformableVolume d = vol_of(view);
    const FusionStats s = integrate_frame(d, frame_of(frame), pose_of(pose), fparams_of(*params), exec_of(exec));
    vol_to(d, view);
    if (out) *out = {s.fused, s.skipped_gate, s.skipped_frustum, s.skipped_occluded};
    return WFK_OK;
  });
}
int wfo_expand_grid(wfk_volume_view* view, wfk_expansion_stats* out) {
  DeformableVolume d = vol_of(view);
  const ExpansionStats s = expand_grid(d);
  vol_to(d, view);
  if (out) *out = {s.activated, s.orphans};
  return WFK_OK;
}
int wfo_advance_ages(wfk_volume_view* view, const int32_t* idx, int64_t n) {
  DeformableVolume d = vol_of(view);
  advance_ages(d, std::vector<int>(idx, idx + n));
  vol_to(d, view);
  return WFK_OK;
}

int wfo_backproject_depth(const wfk_frame_view* frame, int32_t exec, wfk_point_normal_map* out) {
  return guarded([&]() -> int {
    const PointNormalMap m = backproject_depth(frame_of(frame), exec_of(exec));
    out->width = m.width;
    out->height = m.height;
    const size_t n = size_t(m.width) * size_t(m.height);
    for (size_t i = 0; i < n; ++i) {
      put(m.point[i], out->point + 3 * i);
      put(m.normal[i], out->normal + 3 * i);
      out->point_valid[i] = m.point_valid[i];
      out->normal_valid[i] = m.normal_valid[i];
    }
    return WFK_OK;
  });
}
double wfo_dense_confidence(double d, double nd, double vd, const wfk_correspond_params* p) {
  return dense_confidence(d, nd, vd, cparams_of(*p));
}
int wfo_sample_point_normal(const wfk_point_normal_map* maps, const double uv[2], double point[3],
                            double normal[3]) {
  Vec3 p, n;
  const bool ok = sample_point_normal(maps_of(maps), Vec2(uv[0], uv[1]), p, n);
  if (ok) {
    put(p, point);
    put(n, normal);
  }
  return ok ? 1 : 0;
}
int wfo_find_dense_correspondences(const wfk_geometry_buffer* buf, const wfk_point_normal_map* maps,
                                   const wfk_intrinsics* intr, const wfk_correspond_params* params,
                                   const wfk_volume_view* view, wfk_correspondence* out, int64_t cap,
                                   int64_t* n_out) {
  return guarded([&]() -> int {
    const auto c = find_dense_correspondences(gbuf_of(buf), maps_of(maps), intr_of(*intr), cparams_of(*params),
                                              vol_of(view));
    if (n_out) *n_out = int64_t(c.size());
    if (int64_t(c.size()) > cap) return fail(WFK_E_CAPACITY, "correspondence buffer too small");
    for (size_t i = 0; i < c.size(); ++i) con_to(c[i], out[i]);
    return WFK_OK;
  });
}
int wfo_estimate_global_pose(const wfk_geometry_buffer* buf, const wfk_point_normal_map* maps,
                             const wfk_intrinsics* intr, const wfk_volume_view* view, const wfk_pose* initial,
                             const wfk_icp_params* params, wfk_icp_result* out) {
  return guarded([&]() -> int {
    const IcpResult r = estimate_global_pose(gbuf_of(buf), maps_of(maps), intr_of(*intr), vol_of(view),
                                             pose_of(initial), icpparams_of(*params));
    std::memset(out, 0, sizeof(*out));
    pose_to_c(r.pose, &out->pose);
    out->converged = r.converged;
    out->degraded = r.degraded;
    out->rms = r.rms;
    out->iterations = r.iterations;
    return WFK_OK;
  });
}

int wfo_detect_features(const wfk_frame_view* frame, const wfk_feature_params* p, wfk_feature* out, int32_t cap,
                        int32_t* n_out, int32_t* n_keypoints) {
  // the pipeline's detection sequence (pipeline.cpp:97-101)
  *n_out = 0;
  if (!frame->color) return WFK_OK;
  const Frame f = frame_of(frame);
  const FeatureParams fp = featparams_of(*p);
  const DogPyramid pyr = build_pyramid(to_gray(f.color), fp);
  const auto kps = detect_keypoints(pyr, f.depth, fp);
  if (n_keypoints) *n_keypoints = int32_t(kps.size());
  const auto fs = extract_descriptors(kps, pyr, fp);
  *n_out = int32_t(fs.size());
  if (int32_t(fs.size()) > cap) return fail(WFK_E_CAPACITY, "feature buffer too small");
  for (size_t i = 0; i < fs.size(); ++i) out[i] = feature_to(fs[i]);
  return WFK_OK;
}
int wfo_pyramid_level(const wfk_frame_view* frame, const wfk_feature_params* p, int32_t o, int32_t l, int32_t dog,
                      float* out, int32_t* w_out, int32_t* h_out) {
  const Frame f = frame_of(frame);
  const DogPyramid pyr = build_pyramid(to_gray(f.color), featparams_of(*p));
  const GrayImage& im = dog ? pyr.dog[size_t(o)][size_t(l)] : pyr.gauss[size_t(o)][size_t(l)];
  *w_out = im.width;
  *h_out = im.height;
  if (out) std::memcpy(out, im.data.data(), im.data.size() * sizeof(float));
  return WFK_OK;
}
double wfo_descriptor_distance(const float* a, const float* b) {
  std::array<float, 128> x, y;
  std::memcpy(x.data(), a, sizeof(float) * 128);
  std::memcpy(y.data(), b, sizeof(float) * 128);
  return descriptor_distance(x, y);
}
int wfo_match_features(const wfk_feature* cur, int32_t nc, const wfk_feature* store, int32_t ns,
                       const double* predicted_world, const wfk_intrinsics* K, const wfk_feature_params* p,
                       wfk_feature_match* out, int32_t cap, int32_t* n_out) {
  std::vector<Feature> c;
  for (int i = 0; i < nc; ++i) c.push_back(feature_of(cur[i]));
  FeatureStore st;
  std::vector<Vec3> pw;
  for (int i = 0; i < ns; ++i) {
    st.add(feature_of(store[i]));
    pw.push_back(v3(predicted_world + 3 * i));
  }
  const auto m = match_features(c, st, pw, intr_of(*K), featparams_of(*p));
  *n_out = int32_t(m.size());
  if (int32_t(m.size()) > cap) return fail(WFK_E_CAPACITY, "match buffer too small");
  for (size_t i = 0; i < m.size(); ++i) out[i] = {m[i].source_id, m[i].target_id, m[i].distance};
  return WFK_OK;
}

int wfo_invert_warp(const wfk_volume_view* view, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                    int32_t max_iters, double tol, double* x, uint8_t* ok) {
  const DeformableVolume d = vol_of(view);
  const GlobalPose g = pose_of(pose);
  for (int64_t i = 0; i < n; ++i) {
    const auto r = d.invert_warp(g, v3(y + 3 * i), v3(seed + 3 * i), max_iters, tol);
    ok[i] = r ? 1 : 0;
    put(r ? *r : Vec3::Zero(), x + 3 * i);
  }
  return WFK_OK;
}
int wfo_ldlt_solve(int n, const double* a, const double* b, double* x) {
  if (n < 1 || n > 8) return fail(WFK_E_INVALID_ARG, "ldlt: n out of range");
  Eigen::MatrixXd m(n, n);
  Eigen::VectorXd v(n);
  for (int i = 0; i < n; ++i) {
    v(i) = b[i];
    for (int k = 0; k < n; ++k) m(i, k) = a[i * n + k];
  }
  const Eigen::VectorXd s = m.ldlt().solve(v);
  for (int i = 0; i < n; ++i) x[i] = s(i);
  return WFK_OK;
}
int wfo_sparse_to_constraints(const double* canonical, const double* target, int64_t n,
                              const wfk_volume_view* view, wfk_correspondence* out, int64_t* n_out) {
  std::vector<FeatureConstraintInput> in;
  for (int64_t i = 0; i < n; ++i) in.push_back({v3(canonical + 3 * i), v3(target + 3 * i)});
  const auto c = sparse_to_constraints(in, vol_of(view));
  for (size_t i = 0; i < c.size(); ++i) con_to(c[i], out[i]);
  *n_out = int64_t(c.size());
  return WFK_OK;
}

int wfo_extract_mesh(const wfk_volume_view* view, const wfk_pose* pose, wfo_mesh** out) {
  return guarded([&]() -> int {
    auto* m = new wfo_mesh;
    m->m = extract_mesh(vol_of(view), pose_of(pose));
    *out = m;
    return WFK_OK;
  });
}
void wfo_mesh_sizes(const wfo_mesh* m, int64_t* nv, int64_t* nt) {
  *nv = int64_t(m->m.vertices_canonical.size());
  *nt = int64_t(m->m.triangles.size());
}
void wfo_mesh_export(const wfo_mesh* mm, wfk_mesh_view* o) {
  const SurfaceMesh& m = mm->m;
  o->num_vertices = int64_t(m.vertices_canonical.size());
  o->num_triangles = int64_t(m.triangles.size());
  for (size_t i = 0; i < m.vertices_canonical.size(); ++i) {
    if (o->vertices_canonical) put(m.vertices_canonical[i], o->vertices_canonical + 3 * i);
    if (o->vertices_deformed) put(m.vertices_deformed[i], o->vertices_deformed + 3 * i);
    if (o->normals_deformed && m.normals_deformed.size() == m.vertices_canonical.size())
      put(m.normals_deformed[i], o->normals_deformed + 3 * i);
    if (o->colors)
      for (int k = 0; k < 3; ++k) o->colors[3 * i + size_t(k)] = m.colors[i][k];
  }
  if (o->triangles)
    for (size_t t = 0; t < m.triangles.size(); ++t)
      for (int k = 0; k < 3; ++k) o->triangles[3 * t + size_t(k)] = m.triangles[t][k];
}
int wfo_mesh_import(const wfk_mesh_view* in, wfo_mesh** out) {
  auto* mm = new wfo_mesh;
  SurfaceMesh& m = mm->m;
  const size_t nv = size_t(in->num_vertices), nt = size_t(in->num_triangles);
  m.vertices_canonical.resize(nv);
  m.vertices_deformed.resize(nv);
  m.colors.resize(nv);
  for (size_t i = 0; i < nv; ++i) {
    m.vertices_canonical[i] = v3(in->vertices_canonical + 3 * i);
    m.vertices_deformed[i] = v3(in->vertices_deformed + 3 * i);
    if (in->colors) m.colors[i] = Vec3f(in->colors[3 * i], in->colors[3 * i + 1], in->colors[3 * i + 2]);
  }
  if (in->normals_deformed) {
    m.normals_deformed.resize(nv);
    for (size_t i = 0; i < nv; ++i) m.normals_deformed[i] = v3(in->normals_deformed + 3 * i);
  }
  m.triangles.resize(nt);
  for (size_t t = 0; t < nt; ++t)
    m.triangles[t] = Vec3i(in->triangles[3 * t], in->triangles[3 * t + 1], in->triangles[3 * t + 2]);
  *out = mm;
  return WFK_OK;
}
int wfo_mesh_warp(wfo_mesh* mm, const wfk_volume_view* view, const wfk_pose* pose) {
  // the redeform step of process_frame (pipeline.cpp:167-169)
  const DeformableVolume d = vol_of(view);
  const GlobalPose g = pose_of(pose);
  for (size_t i = 0; i < mm->m.vertices_canonical.size(); ++i)
    mm->m.vertices_deformed[i] = d.warp_point(g, mm->m.vertices_canonical[i]);
  return WFK_OK;
}
void wfo_compute_normals(wfo_mesh* m) { compute_normals(m->m); }
int wfo_rasterize(const wfo_mesh* m, const wfk_intrinsics* intr, int32_t exec, wfk_geometry_buffer* out) {
  return guarded([&]() -> int {
    gbuf_to(rasterize(m->m, intr_of(*intr), exec_of(exec)), out);
    return WFK_OK;
  });
}
void wfo_mesh_free(wfo_mesh* m) { delete m; }

// ---- Reconstructor (pipeline.cpp:143-262) ----
int wfo_recon_create(const wfo_recon_config* c, wfo_recon** out) {
  return guarded([&]() -> int {
    ReconstructionConfig cfg;
    cfg.volume_dims = Vec3i(c->dims[0], c->dims[1], c->dims[2]);
    cfg.voxel_size = c->voxel_size;
    cfg.volume_origin = v3(c->origin);
    cfg.solver = params_of(&c->solver);
    cfg.correspond = cparams_of(c->correspond);
    cfg.fusion = fparams_of(c->fusion);
    cfg.estimate_pose = c->estimate_pose != 0;
    cfg.icp = icpparams_of(c->icp);
    cfg.use_features = c->use_features != 0;
    cfg.features = featparams_of(c->features);
    cfg.reassociations = c->reassociations;
    *out = new wfo_recon(cfg);
    return WFK_OK;
  });
}
void wfo_recon_free(wfo_recon* r) { delete r; }
// The reference keeps its volume as private std::vectors behind accessors;
// expose a snapshot (refreshed by this call) in the borrowed-view layout.
struct RefVolumeSnapshot {
  std::vector<float> tsdf, weight, color;
  std::vector<double> deformed, euler;
  std::vector<int32_t> age;
  std::vector<uint8_t> active;
};
static std::map<const wfo_recon*, RefVolumeSnapshot> g_snap;
void wfo_recon_volume(wfo_recon* r, wfk_volume_view* o) {
  const DeformableVolume& d = r->r.volume();
  RefVolumeSnapshot& s = g_snap[r];
  const size_t n = size_t(d.num_points());
  s.tsdf.resize(n);
  s.weight.resize(n);
  s.color.resize(3 * n);
  s.deformed.resize(3 * n);
  s.euler.resize(3 * n);
  s.age.resize(n);
  s.active.resize(n);
  for (int k = 0; k < 3; ++k) o->dims[k] = d.dims()[k];
  o->voxel_size = d.voxel_size();
  put(d.origin(), o->origin);
  o->tsdf = s.tsdf.data();
  o->weight = s.weight.data();
  o->color = s.color.data();
  o->deformed = s.deformed.data();
  o->euler = s.euler.data();
  o->age = s.age.data();
  o->active = s.active.data();
  vol_to(d, o);
}
int wfo_recon_process_frame(wfo_recon* r, const wfk_frame_view* frame, const wfk_correspondence* sparse,
                            int64_t nsparse, wfo_frame_record* rec) {
  std::memset(rec, 0, sizeof(*rec));
  if (nsparse > 0) return fail(WFK_E_INVALID_ARG, "caller sparse constraints: not available in the reference build");
  return guarded([&]() -> int {
    const FrameRecord fr = r->r.process_frame(frame_of(frame), r->r.frames_processed());
    fill_energy(fr.energy, &rec->energy);
    rec->dense_count = fr.dense_count;
    rec->sparse_count = fr.sparse_count;
    rec->anomalies = fr.anomalies;
    rec->trace_len = int32_t(fr.trace.size());
    for (const auto& e : fr.trace) rec->pcg_iterations += e.pcg_iterations;
    rec->fusion = {fr.fusion.fused, fr.fusion.skipped_gate, fr.fusion.skipped_frustum, fr.fusion.skipped_occluded};
    rec->expansion = {fr.expansion.activated, fr.expansion.orphans};
    pose_to_c(fr.pose, &rec->pose);
    rec->icp_degraded = fr.icp_degraded ? 1 : 0;
    rec->icp_iterations = -1;  // not part of the reference's FrameRecord
    rec->icp_rms = fr.icp_rms;
    rec->match_count = fr.match_count;
    rec->features_added = fr.features_added;
    return WFK_OK;
  });
}
int wfo_recon_feature_store(const wfo_recon* r, wfk_feature* out, int64_t cap, int64_t* n_out) {
  const auto& all = r->r.feature_store().all();
  const int64_t n = int64_t(all.size());
  if (n_out) *n_out = n;
  if (!out) return WFK_OK;
  if (n > cap) return fail(WFK_E_CAPACITY, "feature buffer too small");
  for (int64_t i = 0; i < n; ++i) out[i] = feature_to(all[size_t(i)]);
  return WFK_OK;
}

// ---- snapshot / frame formats through the reference's own file writers ----
int wfo_volume_save_bytes(const wfk_volume_view* v, uint8_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    const std::string p = temp_path("vol.bin");
    vol_of(v).save(p);
    const auto bytes = read_file(p);
    std::filesystem::remove(p);
    return copy_out(bytes, out, cap, n_out);
  });
}
int wfo_volume_load_bytes(const uint8_t* in, int64_t n, wfk_volume_view* v) {
  return guarded([&]() -> int {
    const std::string p = temp_path("vol_in.bin");
    write_file(p, in, n);
    const DeformableVolume d = DeformableVolume::load(p);
    std::filesystem::remove(p);
    for (int k = 0; k < 3; ++k) v->dims[k] = d.dims()[k];
    v->voxel_size = d.voxel_size();
    put(d.origin(), v->origin);
    if (v->tsdf) vol_to(d, v);
    return WFK_OK;
  });
}
int wfo_feature_store_bytes(const wfk_feature* f, int32_t nf, uint8_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    FeatureStore st;
    for (int i = 0; i < nf; ++i) st.add(feature_of(f[i]));
    const std::string p = temp_path("feat.bin");
    st.save(p);
    const auto bytes = read_file(p);
    std::filesystem::remove(p);
    return copy_out(bytes, out, cap, n_out);
  });
}
int wfo_pgm_encode(const float* depth, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    DepthImage img(w, h);
    std::memcpy(img.data.data(), depth, size_t(w) * size_t(h) * sizeof(float));
    const std::string p = temp_path("d.pgm");
    save_depth_pgm(img, p);
    const auto bytes = read_file(p);
    std::filesystem::remove(p);
    return copy_out(bytes, out, cap, n_out);
  });
}
int wfo_ppm_encode(const float* color, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out) {
  return guarded([&]() -> int {
    ColorImage img(w, h);
    for (size_t i = 0; i < size_t(w) * size_t(h); ++i)
      img.data[i] = Vec3f(color[3 * i], color[3 * i + 1], color[3 * i + 2]);
    const std::string p = temp_path("c.ppm");
    save_color_ppm(img, p);
    const auto bytes = read_file(p);
    std::filesystem::remove(p);
    return copy_out(bytes, out, cap, n_out);
  });
}
int wfo_pnm_decode(const uint8_t* in, int64_t n, int32_t channels, int32_t* w, int32_t* h, float* out) {
  return guarded([&]() -> int {
    const std::string p = temp_path(channels == 1 ? "in.pgm" : "in.ppm");
    write_file(p, in, n);
    if (channels == 1) {
      const DepthImage d = load_depth_pgm(p);
      *w = d.width;
      *h = d.height;
      if (out) std::memcpy(out, d.data.data(), d.data.size() * sizeof(float));
    } else {
      const ColorImage c = load_color_ppm(p);
      *w = c.width;
      *h = c.height;
      if (out)
        for (size_t i = 0; i < c.data.size(); ++i)
          for (int k = 0; k < 3; ++k) out[3 * i + size_t(k)] = c.data[i][k];
    }
    std::filesystem::remove(p);
    return WFK_OK;
  });
}

// ---- synthetic camera: the reference's own SyntheticScene::render_frame ----
int wfo_synth_render(const double center[3], double radius, const double pivot[3], double amplitude, int driver_axis,
                     int rot_axis, uint32_t tex_seed, double tex_scale, double dot_radius, const wfk_intrinsics* K,
                     float* depth, float* color) {
  return guarded([&]() -> int {
    // one sphere under a static bend of `amplitude` rad/m (frequency 0, frame
    // 1 of a 2-frame linear ramp => phase 1) with the Dots texture
    SceneSpec s;
    s.frames = 2;
    s.intrinsics = intr_of(*K);
    ShapeSpec sh;
    sh.type = ShapeType::Sphere;
    sh.center = v3(center);
    sh.radius = radius;
    s.shapes = {sh};
    s.texture.type = TextureType::Dots;
    s.texture.seed = tex_seed;
    s.texture.scale = tex_scale;
    s.texture.dot_radius = dot_radius;
    s.warp.type = amplitude == 0 ? WarpType::None : WarpType::Bend;
    s.warp.driver_axis = driver_axis;
    s.warp.rot_axis = rot_axis;
    s.warp.amplitude = amplitude;
    s.warp.frequency = 0;
    s.warp.pivot = v3(pivot);
    const SyntheticScene scene(s);
    const Frame f = scene.render_frame(1);
    const size_t n = size_t(K->width) * size_t(K->height);
    std::memcpy(depth, f.depth.data.data(), n * sizeof(float));
    for (size_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) color[3 * i + size_t(k)] = f.color.data[i][k];
    return WFK_OK;
  });
}

// the reference's SyntheticScene for a tools/synthscene.h scene description
// (checks tools/synthscene.cpp bit for bit, tests/test_synthscene.py)
static Vec3 sv(const double* p) { return Vec3(p[0], p[1], p[2]); }
int wfo_ref_render_scene(const ss_scene* q, int32_t frame, float* depth, float* color) {
  return guarded([&]() -> int {
    SceneSpec s;
    s.frames = q->frames;
    s.intrinsics = Intrinsics{q->fx, q->fy, q->cx, q->cy, q->width, q->height};
    s.shapes.clear();
    for (int i = 0; i < q->num_shapes; ++i) {
      const ss_shape& a = q->shapes[i];
      ShapeSpec b;
      b.type = ShapeType(a.type);
      b.center = sv(a.center);
      b.radius = a.radius;
      b.half_extents = sv(a.half_extents);
      b.normal = sv(a.normal);
      b.offset = a.offset;
      b.axis = sv(a.axis);
      b.half_height = a.half_height;
      s.shapes.push_back(b);
    }
    s.texture.type = TextureType(q->tex_type);
    s.texture.seed = q->tex_seed;
    s.texture.scale = q->tex_scale;
    s.texture.dot_radius = q->dot_radius;
    s.warp.type = WarpType(q->warp_type);
    s.warp.driver_axis = q->driver_axis;
    s.warp.rot_axis = q->rot_axis;
    s.warp.amplitude = q->amplitude;
    s.warp.frequency = q->frequency;
    s.warp.pivot = sv(q->pivot);
    s.warp.rotation_axis = sv(q->rotation_axis);
    s.warp.deg_per_frame = q->deg_per_frame;
    s.warp.trans_per_frame = sv(q->trans_per_frame);
    s.camera.rot_axis = sv(q->cam_rot_axis);
    s.camera.deg_per_frame = q->cam_deg_per_frame;
    s.camera.trans_per_frame = sv(q->cam_trans_per_frame);
    s.t_min = q->t_min;
    s.t_max = q->t_max;
    s.noise_sigma = q->noise_sigma;
    s.noise_seed = q->noise_seed;
    const SyntheticScene scene(s);
    const Frame f = scene.render_frame(frame);
    const size_t n = size_t(q->width) * size_t(q->height);
    std::memcpy(depth, f.depth.data.data(), n * sizeof(float));
    for (size_t i = 0; i < n; ++i)
      for (int k = 0; k < 3; ++k) color[3 * i + size_t(k)] = f.color.data[i][k];
    return WFK_OK;
  });
}

}  // extern "C"
