// ORACLE — test infrastructure, not product code.
//
// A CPU restatement of the reference hot path (warpfuse / VolumeDeform,
// /root/reference/proj/src/{core,volume,solver,fusion,correspond,isosurface,
// rasterize}.cpp), written without Eigen (absent from this image, so the
// reference itself is unbuildable here).  Every
// function follows the reference loop order and arithmetic order and cites the
// file:line it restates.  Built with -O2 -fopenmp -ffp-contract=off so that no
// multiply-add is fused, like the reference build the survey prescribes.
//
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
// this library; the product path (libwfk.so) never does.
//
// Eigen dependence: JacobiSVD<Matrix3d> (solver.cpp:401, core.cpp:32) is
// restated from Eigen 3.4's published two-sided Jacobi algorithm
// (Eigen/src/SVD/JacobiSVD.h, real_2x2_jacobi_svd + makeJacobi); Eigen is
// unpinned in the reference (proj/CMakeLists.txt:13).

#include "wfo.h"

#include <algorithm>
#include <array>
#include <stdexcept>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include "../include/wfk_mc_cases.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

// ---------------------------------------------------------------------------
// minimal fixed-size linear algebra (stands in for Eigen's Vector3d/Matrix3d)
// ---------------------------------------------------------------------------
struct V3 {
  double x = 0, y = 0, z = 0;
  V3() = default;
  V3(double a, double b, double c) : x(a), y(b), z(c) {}
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator-(const V3& a) { return {-a.x, -a.y, -a.z}; }
inline V3 operator*(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator*(const V3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 operator/(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline V3& operator+=(V3& a, const V3& b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
inline V3& operator-=(V3& a, const V3& b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double sqnorm(const V3& a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 normalized(const V3& a) {
  const double z = sqnorm(a);
  return z > 0 ? a / std::sqrt(z) : a;
}

struct F3 {
  float x = 0, y = 0, z = 0;
};

struct M3 {
  double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  static M3 identity() {
    M3 m;
    m.a[0][0] = m.a[1][1] = m.a[2][2] = 1;
    return m;
  }
  double& operator()(int i, int j) { return a[i][j]; }
  double operator()(int i, int j) const { return a[i][j]; }
};
inline M3 operator*(const M3& p, const M3& q) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.a[i][j] = p.a[i][0] * q.a[0][j] + p.a[i][1] * q.a[1][j] + p.a[i][2] * q.a[2][j];
  return r;
}
inline V3 operator*(const M3& m, const V3& v) {
  return {m.a[0][0] * v.x + m.a[0][1] * v.y + m.a[0][2] * v.z,
          m.a[1][0] * v.x + m.a[1][1] * v.y + m.a[1][2] * v.z,
          m.a[2][0] * v.x + m.a[2][1] * v.y + m.a[2][2] * v.z};
}
inline M3 operator+(const M3& p, const M3& q) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = p.a[i][j] + q.a[i][j];
  return r;
}
inline M3 transpose(const M3& m) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = m.a[j][i];
  return r;
}
// Eigen determinant_impl<3>
inline double det(const M3& m) {
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}

M3 from_rowmajor(const double* p) {
  M3 m;
  for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = p[i];
  return m;
}
void to_rowmajor(const M3& m, double* p) {
  for (int i = 0; i < 9; ++i) p[i] = m.a[i / 3][i % 3];
}

struct Pose {
  M3 r = M3::identity();
  V3 t;
  V3 apply(const V3& x) const { return r * x + t; }  // core.hpp:24
};
Pose pose_of(const wfk_pose* p) {
  Pose q;
  if (p) {
    q.r = from_rowmajor(p->rotation);
    q.t = {p->translation[0], p->translation[1], p->translation[2]};
  }
  return q;
}

// core.cpp:7-14  R = Rz(c) * Ry(b) * Rx(a)
M3 euler_to_matrix(const V3& abc) {
  const double a = abc.x, b = abc.y, c = abc.z;
  M3 rx, ry, rz;
  rx.a[0][0] = 1; rx.a[0][1] = 0; rx.a[0][2] = 0;
  rx.a[1][0] = 0; rx.a[1][1] = std::cos(a); rx.a[1][2] = -std::sin(a);
  rx.a[2][0] = 0; rx.a[2][1] = std::sin(a); rx.a[2][2] = std::cos(a);
  ry.a[0][0] = std::cos(b); ry.a[0][1] = 0; ry.a[0][2] = std::sin(b);
  ry.a[1][0] = 0; ry.a[1][1] = 1; ry.a[1][2] = 0;
  ry.a[2][0] = -std::sin(b); ry.a[2][1] = 0; ry.a[2][2] = std::cos(b);
  rz.a[0][0] = std::cos(c); rz.a[0][1] = -std::sin(c); rz.a[0][2] = 0;
  rz.a[1][0] = std::sin(c); rz.a[1][1] = std::cos(c); rz.a[1][2] = 0;
  rz.a[2][0] = 0; rz.a[2][1] = 0; rz.a[2][2] = 1;
  return (rz * ry) * rx;
}

// core.cpp:16-29
V3 matrix_to_euler(const M3& r) {
  const double b = std::asin(std::clamp(-r(2, 0), -1.0, 1.0));
  double a, c;
  if (std::abs(r(2, 0)) < 1.0 - 1e-12) {
    a = std::atan2(r(2, 1), r(2, 2));
    c = std::atan2(r(1, 0), r(0, 0));
  } else {
    a = std::atan2(-r(1, 2), r(1, 1));
    c = 0.0;
  }
  return {a, b, c};
}

// ---- Eigen 3.4 JacobiSVD<Matrix3d>, ComputeFullU | ComputeFullV -----------
struct Rot {  // JacobiRotation<double>: J = [c s; -s c]
  double c = 1, s = 0;
  Rot transpose() const { return {c, -s}; }
};
inline Rot operator*(const Rot& a, const Rot& b) {
  return {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c};
}
// apply_rotation_in_the_plane(x, y, j): x' = c x + s y ; y' = -s x + c y
inline void rot_rows(M3& m, int p, int q, const Rot& j) {
  for (int i = 0; i < 3; ++i) {
    const double xi = m.a[p][i], yi = m.a[q][i];
    m.a[p][i] = j.c * xi + j.s * yi;
    m.a[q][i] = -j.s * xi + j.c * yi;
  }
}
inline void rot_cols(M3& m, int p, int q, const Rot& j) {  // applyOnTheRight(p,q,j)
  const Rot t = j.transpose();
  for (int i = 0; i < 3; ++i) {
    const double xi = m.a[i][p], yi = m.a[i][q];
    m.a[i][p] = t.c * xi + t.s * yi;
    m.a[i][q] = -t.s * xi + t.c * yi;
  }
}
Rot make_jacobi(double x, double y, double z) {
  Rot r;
  const double deno = 2.0 * std::abs(y);
  if (deno < DBL_MIN) return r;
  const double tau = (x - z) / deno;
  const double w = std::sqrt(tau * tau + 1.0);
  const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0 ? 1.0 : -1.0;
  const double n = 1.0 / std::sqrt(t * t + 1.0);
  r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
  r.c = n;
  return r;
}
void real_2x2_jacobi_svd(const M3& w, int p, int q, Rot& jl, Rot& jr) {
  double m00 = w.a[p][p], m01 = w.a[p][q], m10 = w.a[q][p], m11 = w.a[q][q];
  Rot rot1;
  const double t = m00 + m11;
  const double d = m10 - m01;
  if (std::abs(d) < DBL_MIN) {
    rot1.s = 0;
    rot1.c = 1;
  } else {
    const double u = t / d;
    const double tmp = std::sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  // m.applyOnTheLeft(0, 1, rot1)
  const double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
  const double n10 = -rot1.s * m00 + rot1.c * m10, n11 = -rot1.s * m01 + rot1.c * m11;
  (void)n10;
  jr = make_jacobi(n00, n01, n11);
  jl = rot1 * jr.transpose();
}
void svd3(const M3& a, M3& u, double sv[3], M3& v) {
  double scale = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) scale = std::max(scale, std::abs(a.a[i][j]));
  if (!std::isfinite(scale)) {
    u = M3::identity();
    v = M3::identity();
    sv[0] = sv[1] = sv[2] = 0;
    return;
  }
  if (scale == 0) scale = 1;
  M3 w;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) w.a[i][j] = a.a[i][j] / scale;
  u = M3::identity();
  v = M3::identity();
  const double considerAsZero = DBL_MIN;
  const double precision = 2.0 * DBL_EPSILON;
  double maxDiag = std::max(std::abs(w.a[0][0]), std::max(std::abs(w.a[1][1]), std::abs(w.a[2][2])));
  bool finished = false;
  while (!finished) {
    finished = true;
    for (int p = 1; p < 3; ++p)
      for (int q = 0; q < p; ++q) {
        const double threshold = std::max(considerAsZero, precision * maxDiag);
        if (std::abs(w.a[p][q]) > threshold || std::abs(w.a[q][p]) > threshold) {
          finished = false;
          Rot jl, jr;
          real_2x2_jacobi_svd(w, p, q, jl, jr);
          rot_rows(w, p, q, jl);
          rot_cols(u, p, q, jl.transpose());
          rot_cols(w, p, q, jr);
          rot_cols(v, p, q, jr);
          maxDiag = std::max(maxDiag, std::max(std::abs(w.a[p][p]), std::abs(w.a[q][q])));
        }
      }
  }
  for (int i = 0; i < 3; ++i) {
    const double d = w.a[i][i];
    sv[i] = std::abs(d);
    if (d < 0)
      for (int k = 0; k < 3; ++k) u.a[k][i] = -u.a[k][i];
  }
  for (int i = 0; i < 3; ++i) sv[i] *= scale;
  for (int i = 0; i < 3; ++i) {
    int pos = i;
    double best = sv[i];
    for (int k = i + 1; k < 3; ++k)
      if (sv[k] > best) {
        best = sv[k];
        pos = k;
      }
    if (best == 0) break;
    if (pos != i) {
      std::swap(sv[i], sv[pos]);
      for (int k = 0; k < 3; ++k) {
        std::swap(u.a[k][i], u.a[k][pos]);
        std::swap(v.a[k][i], v.a[k][pos]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// DeformableVolume (volume.hpp:29-112, volume.cpp) over a borrowed or owned SoA
// ---------------------------------------------------------------------------
struct Vol {
  int nx = 0, ny = 0, nz = 0;
  double voxel = 0;
  V3 origin;
  double mu = 0;
  float* tsdf_ = nullptr;
  float* weight_ = nullptr;
  float* color_ = nullptr;
  double* deformed_ = nullptr;
  double* euler_ = nullptr;
  int32_t* age_ = nullptr;
  uint8_t* active_ = nullptr;
  // owned storage (hierarchy levels)
  std::vector<float> o_tsdf, o_weight, o_color;
  std::vector<double> o_def, o_eul;
  std::vector<int32_t> o_age;
  std::vector<uint8_t> o_act;

  static Vol borrow(const wfk_volume_view* v) {
    Vol r;
    r.nx = v->dims[0];
    r.ny = v->dims[1];
    r.nz = v->dims[2];
    r.voxel = v->voxel_size;
    r.origin = {v->origin[0], v->origin[1], v->origin[2]};
    r.mu = v->truncation;
    r.tsdf_ = v->tsdf;
    r.weight_ = v->weight;
    r.color_ = v->color;
    r.deformed_ = v->deformed;
    r.euler_ = v->euler;
    r.age_ = v->age;
    r.active_ = v->active;
    return r;
  }
  // DeformableVolume ctor (volume.cpp:8-25), geometry-only fields owned
  void make_owned(int x, int y, int z, double vox, const V3& o, bool with_tsdf) {
    nx = x; ny = y; nz = z; voxel = vox; origin = o; mu = 4.0 * vox;
    const size_t n = size_t(x) * y * z;
    if (with_tsdf) {
      o_tsdf.assign(n, 0.f); o_weight.assign(n, 0.f); o_color.assign(3 * n, 0.f);
      tsdf_ = o_tsdf.data(); weight_ = o_weight.data(); color_ = o_color.data();
    }
    o_def.resize(3 * n); o_eul.assign(3 * n, 0.0); o_age.assign(n, 0); o_act.assign(n, 0);
    deformed_ = o_def.data(); euler_ = o_eul.data(); age_ = o_age.data(); active_ = o_act.data();
    for (size_t i = 0; i < n; ++i) set_deformed(int(i), canonical(int(i)));
  }
  // move-safe pointer refresh after the owning Vol is moved into a vector
  void rebind() {
    if (!o_def.empty()) { deformed_ = o_def.data(); euler_ = o_eul.data(); age_ = o_age.data(); active_ = o_act.data(); }
    if (!o_tsdf.empty()) { tsdf_ = o_tsdf.data(); weight_ = o_weight.data(); color_ = o_color.data(); }
  }

  int num_points() const { return nx * ny * nz; }
  int lin(int x, int y, int z) const { return x + nx * (y + ny * z); }  // volume.hpp:40-42
  void idx3(int i, int& x, int& y, int& z) const {                      // volume.hpp:43-45
    x = i % nx;
    y = (i / nx) % ny;
    z = i / (nx * ny);
  }
  bool in_grid(int x, int y, int z) const {
    return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz;
  }
  V3 canonical(int i) const {  // volume.hpp:50-52
    int x, y, z;
    idx3(i, x, y, z);
    return {origin.x + voxel * double(x), origin.y + voxel * double(y), origin.z + voxel * double(z)};
  }
  V3 canonical3(int x, int y, int z) const {
    return {origin.x + voxel * double(x), origin.y + voxel * double(y), origin.z + voxel * double(z)};
  }
  V3 deformed(int i) const { return {deformed_[3 * i], deformed_[3 * i + 1], deformed_[3 * i + 2]}; }
  void set_deformed(int i, const V3& v) {
    deformed_[3 * i] = v.x; deformed_[3 * i + 1] = v.y; deformed_[3 * i + 2] = v.z;
  }
  V3 euler(int i) const { return {euler_[3 * i], euler_[3 * i + 1], euler_[3 * i + 2]}; }
  void set_euler(int i, const V3& v) {
    euler_[3 * i] = v.x; euler_[3 * i + 1] = v.y; euler_[3 * i + 2] = v.z;
  }
  M3 rotation(int i) const { return euler_to_matrix(euler(i)); }              // volume.hpp:70
  void set_rotation(int i, const M3& r) { set_euler(i, matrix_to_euler(r)); }  // volume.hpp:71
  bool active(int i) const { return active_[i] != 0; }
  void set_active(int i, bool a) { active_[i] = a ? 1 : 0; }

  // volume.cpp:27-33
  bool contains(const V3& x) const {
    const double eps = 1e-9;
    const V3 rel = (x - origin) / voxel;
    const int d[3] = {nx, ny, nz};
    for (int k = 0; k < 3; ++k)
      if (!(rel[k] >= -eps)) return false;
    for (int k = 0; k < 3; ++k)
      if (!(rel[k] <= (double(d[k]) - 1.0) + eps)) return false;
    return true;
  }
  // volume.cpp:35-59 (caller checks contains; throws out_of_range otherwise)
  void anchors(const V3& x, int idx[8], double w[8]) const {
    const V3 rel = (x - origin) / voxel;
    const int d[3] = {nx, ny, nz};
    int cell[3];
    double frac[3];
    for (int k = 0; k < 3; ++k) {
      int c = static_cast<int>(std::floor(rel[k]));
      c = std::clamp(c, 0, d[k] - 2);
      cell[k] = c;
      frac[k] = std::clamp(rel[k] - c, 0.0, 1.0);
    }
    int n = 0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          idx[n] = lin(cell[0] + dx, cell[1] + dy, cell[2] + dz);
          w[n] = (dx ? frac[0] : 1 - frac[0]) * (dy ? frac[1] : 1 - frac[1]) *
                 (dz ? frac[2] : 1 - frac[2]);
          ++n;
        }
  }
  // volume.cpp:61-66
  V3 interpolate_deformed(const V3& x) const {
    int idx[8];
    double w[8];
    anchors(x, idx, w);
    V3 p;
    for (int k = 0; k < 8; ++k) p += w[k] * deformed(idx[k]);
    return p;
  }
  V3 warp_point(const Pose& pose, const V3& x) const { return pose.apply(interpolate_deformed(x)); }
  // volume.cpp:128-137, color part
  F3 sample_color(const V3& x) const {
    int idx[8];
    double w[8];
    anchors(x, idx, w);
    F3 c;
    for (int k = 0; k < 8; ++k) {
      const float fw = static_cast<float>(w[k]);
      c.x += fw * color_[3 * idx[k]];
      c.y += fw * color_[3 * idx[k] + 1];
      c.z += fw * color_[3 * idx[k] + 2];
    }
    return c;
  }
};

const int kFace[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
constexpr int kCenter = 13;
inline int stencil_slot(int dx, int dy, int dz) { return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1); }

struct Params {
  double w_d = 1, w_s = 0.5, w_r = 5;
  int ff_iters = 4;
  double ff_rel_tol = 1e-6, pcg_tol = 1e-4;
  int pcg_max = 50, levels = 3;
  bool parallel = true;
};
Params params_of(const wfk_solver_params* p) {
  Params q;
  if (!p) return q;
  q.w_d = p->w_d; q.w_s = p->w_s; q.w_r = p->w_r;
  q.ff_iters = p->flip_flop_iters; q.ff_rel_tol = p->flip_flop_rel_tol;
  q.pcg_tol = p->pcg_tol; q.pcg_max = p->pcg_max_iters; q.levels = p->levels;
  q.parallel = p->exec != WFK_EXEC_SERIAL;
  return q;
}

struct Con {  // wf::Correspondence
  bool dense = true;
  V3 canonical;
  int idx[8];
  double w[8];
  V3 target, normal;
  double conf = 0;
};
std::vector<Con> cons_of(const wfk_correspondence* c, int64_t n) {
  std::vector<Con> out(size_t(std::max<int64_t>(n, 0)));
  for (int64_t i = 0; i < n; ++i) {
    Con& o = out[size_t(i)];
    o.dense = c[i].kind == WFK_DENSE_PLANE;
    o.canonical = {c[i].canonical[0], c[i].canonical[1], c[i].canonical[2]};
    for (int k = 0; k < 8; ++k) {
      o.idx[k] = c[i].anchor_index[k];
      o.w[k] = c[i].anchor_weight[k];
    }
    o.target = {c[i].target[0], c[i].target[1], c[i].target[2]};
    o.normal = {c[i].target_normal[0], c[i].target_normal[1], c[i].target_normal[2]};
    o.conf = c[i].confidence;
  }
  return out;
}
void con_to_c(const Con& o, wfk_correspondence& c) {
  std::memset(&c, 0, sizeof(c));
  c.kind = o.dense ? WFK_DENSE_PLANE : WFK_SPARSE_POINT;
  c.canonical[0] = o.canonical.x; c.canonical[1] = o.canonical.y; c.canonical[2] = o.canonical.z;
  for (int k = 0; k < 8; ++k) {
    c.anchor_index[k] = o.idx[k];
    c.anchor_weight[k] = o.w[k];
  }
  c.target[0] = o.target.x; c.target[1] = o.target.y; c.target[2] = o.target.z;
  c.target_normal[0] = o.normal.x; c.target_normal[1] = o.normal.y; c.target_normal[2] = o.normal.z;
  c.confidence = o.conf;
}

// ---------------------------------------------------------------------------
// solver.cpp
// ---------------------------------------------------------------------------
struct UnionFind {  // solver.cpp:20-28
  std::vector<int> parent;
  explicit UnionFind(int n) : parent(size_t(n)) { std::iota(parent.begin(), parent.end(), 0); }
  int find(int a) {
    while (parent[size_t(a)] != a) a = parent[size_t(a)] = parent[size_t(parent[size_t(a)])];
    return a;
  }
  void unite(int a, int b) { parent[size_t(find(a))] = find(b); }
};

// solver.cpp:32-69
std::vector<int> compute_active_set(Vol& v) {
  std::vector<uint8_t> on_surface(size_t(v.num_points()), 0);
  for (int cz = 0; cz < v.nz - 1; ++cz)
    for (int cy = 0; cy < v.ny - 1; ++cy)
      for (int cx = 0; cx < v.nx - 1; ++cx) {
        bool observed = true, pos = false, neg = false;
        int corners[8];
        int n = 0;
        for (int dz = 0; dz < 2 && observed; ++dz)
          for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              const int i = v.lin(cx + dx, cy + dy, cz + dz);
              if (v.weight_[i] <= 0.f) {
                observed = false;
                break;
              }
              corners[n++] = i;
              (v.tsdf_[i] < 0 ? neg : pos) = true;
            }
        if (!observed || !pos || !neg) continue;
        for (int k = 0; k < 8; ++k) on_surface[size_t(corners[k])] = 1;
      }
  for (int i = 0; i < v.num_points(); ++i) {
    if (!on_surface[size_t(i)]) continue;
    v.set_active(i, true);
    int x, y, z;
    v.idx3(i, x, y, z);
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], c = z + d[2];
      if (v.in_grid(a, b, c)) v.set_active(v.lin(a, b, c), true);
    }
  }
  std::vector<int> active;
  for (int i = 0; i < v.num_points(); ++i)
    if (v.active(i)) active.push_back(i);
  return active;
}

using Blocks = std::array<M3, 27>;

struct NE {  // NormalEquations (solver.hpp:46-60)
  std::vector<int> rows, node_row;
  std::vector<Blocks> blocks;
  std::vector<std::array<int, 27>> cols;
  std::vector<V3> rhs;
  std::vector<uint8_t> frozen;
  int num_rows() const { return int(rows.size()); }

  // solver.cpp:71-89
  void multiply(const std::vector<V3>& x, std::vector<V3>& out, bool parallel) const {
    out.resize(x.size());
    const int n = num_rows();
    auto row_op = [&](int r) {
      V3 acc;
      for (int s = 0; s < 27; ++s) {
        const int c = cols[size_t(r)][size_t(s)];
        if (c >= 0) acc += blocks[size_t(r)][size_t(s)] * x[size_t(c)];
      }
      out[size_t(r)] = acc;
    };
    if (parallel) {
#pragma omp parallel for schedule(static)
      for (int r = 0; r < n; ++r) row_op(r);
    } else {
      for (int r = 0; r < n; ++r) row_op(r);
    }
  }
  // solver.cpp:91-106
  double symmetry_error() const {
    double err = 0;
    for (int r = 0; r < num_rows(); ++r)
      for (int s = 0; s < 27; ++s) {
        const int c = cols[size_t(r)][size_t(s)];
        if (c < 0 || c < r) continue;
        const int mirror = 26 - s;
        const M3& a = blocks[size_t(r)][size_t(s)];
        M3 bt;
        if (cols[size_t(c)][size_t(mirror)] == r) bt = transpose(blocks[size_t(c)][size_t(mirror)]);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) err = std::max(err, std::abs(a.a[i][j] - bt.a[i][j]));
      }
    return err;
  }
};

struct Cache {  // ConstraintCache (solver.hpp:66-70)
  bool valid = false;
  std::vector<Blocks> blocks;
  std::vector<V3> rhs;
};

M3 scaled(const M3& m, double s) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = s * m.a[i][j];
  return r;
}
void add_to(M3& a, const M3& b) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a.a[i][j] += b.a[i][j];
}

// solver.cpp:108-280
NE build_normal_equations(const Vol& v, const Pose& pose, const std::vector<Con>& cons,
                          const Params& params, Cache* cache) {
  NE sys;
  sys.node_row.assign(size_t(v.num_points()), -1);
  for (int i = 0; i < v.num_points(); ++i)
    if (v.active(i)) {
      sys.node_row[size_t(i)] = int(sys.rows.size());
      sys.rows.push_back(i);
    }
  const int n = sys.num_rows();

  UnionFind uf(n);  // solver.cpp:124-135
  for (int r = 0; r < n; ++r) {
    int x, y, z;
    v.idx3(sys.rows[size_t(r)], x, y, z);
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], c = z + d[2];
      if (!v.in_grid(a, b, c)) continue;
      const int rr = sys.node_row[size_t(v.lin(a, b, c))];
      if (rr >= 0) uf.unite(r, rr);
    }
  }
  std::vector<uint8_t> constrained(size_t(n), 0);  // solver.cpp:136-144
  for (const Con& c : cons)
    for (int k = 0; k < 8; ++k) {
      const int r = sys.node_row[size_t(c.idx[k])];
      if (r >= 0 && c.w[k] > 0) constrained[size_t(uf.find(r))] = 1;
    }
  sys.frozen.assign(size_t(n), 0);
  for (int r = 0; r < n; ++r)
    if (!constrained[size_t(uf.find(r))]) sys.frozen[size_t(r)] = 1;

  sys.blocks.assign(size_t(n), Blocks{});  // solver.cpp:146-161
  sys.cols.assign(size_t(n), {});
  sys.rhs.assign(size_t(n), V3());
  for (int r = 0; r < n; ++r) {
    sys.cols[size_t(r)].fill(-1);
    int x, y, z;
    v.idx3(sys.rows[size_t(r)], x, y, z);
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          if (!v.in_grid(x + dx, y + dy, z + dz)) continue;
          const int rr = sys.node_row[size_t(v.lin(x + dx, y + dy, z + dz))];
          if (rr >= 0) sys.cols[size_t(r)][size_t(stencil_slot(dx, dy, dz))] = rr;
        }
  }

  const bool rebuild = !cache || !cache->valid;  // solver.cpp:163-237
  std::vector<Blocks> local_blocks;
  std::vector<V3> local_rhs;
  std::vector<Blocks>& cb = cache ? cache->blocks : local_blocks;
  std::vector<V3>& crhs = cache ? cache->rhs : local_rhs;
  if (rebuild) {
    cb.assign(size_t(n), Blocks{});
    crhs.assign(size_t(n), V3());
    std::unordered_map<int, std::vector<int>> by_cell;
    for (size_t ci = 0; ci < cons.size(); ++ci) by_cell[cons[ci].idx[0]].push_back(int(ci));
    const M3 rot_t = transpose(pose.r);
    auto assemble_row = [&](int r) {
      const int node = sys.rows[size_t(r)];
      int nx_, ny_, nz_;
      v.idx3(node, nx_, ny_, nz_);
      for (int oz = -1; oz <= 0; ++oz)
        for (int oy = -1; oy <= 0; ++oy)
          for (int ox = -1; ox <= 0; ++ox) {
            const int cx = nx_ + ox, cy = ny_ + oy, cz = nz_ + oz;
            if (cx < 0 || cy < 0 || cz < 0 || cx >= v.nx - 1 || cy >= v.ny - 1 || cz >= v.nz - 1)
              continue;
            auto it = by_cell.find(v.lin(cx, cy, cz));
            if (it == by_cell.end()) continue;
            for (int ci : it->second) {
              const Con& con = cons[size_t(ci)];
              double alpha_i = 0;
              for (int k = 0; k < 8; ++k)
                if (con.idx[k] == node) alpha_i = con.w[k];
              if (alpha_i == 0) continue;
              if (con.dense) {
                const V3 g = rot_t * con.normal;
                const double coef = params.w_d * con.conf;
                const double cst = dot(con.normal, pose.t - con.target);
                M3 ggt;
                for (int i = 0; i < 3; ++i)
                  for (int j = 0; j < 3; ++j) ggt.a[i][j] = g[i] * g[j];
                for (int k = 0; k < 8; ++k) {
                  int a, b, c;
                  v.idx3(con.idx[k], a, b, c);
                  add_to(cb[size_t(r)][size_t(stencil_slot(a - nx_, b - ny_, c - nz_))],
                         scaled(ggt, coef * alpha_i * con.w[k]));
                }
                crhs[size_t(r)] -= (coef * alpha_i * cst) * g;
              } else {
                const double coef = params.w_s * con.conf;
                for (int k = 0; k < 8; ++k) {
                  int a, b, c;
                  v.idx3(con.idx[k], a, b, c);
                  add_to(cb[size_t(r)][size_t(stencil_slot(a - nx_, b - ny_, c - nz_))],
                         scaled(M3::identity(), coef * alpha_i * con.w[k]));
                }
                crhs[size_t(r)] += (coef * alpha_i) * (rot_t * (con.target - pose.t));
              }
            }
          }
    };
    if (params.parallel) {
#pragma omp parallel for schedule(static)
      for (int r = 0; r < n; ++r) assemble_row(r);
    } else {
      for (int r = 0; r < n; ++r) assemble_row(r);
    }
    if (cache) cache->valid = true;
  }

  auto finish_row = [&](int r) {  // solver.cpp:240-269
    if (sys.frozen[size_t(r)]) {
      for (M3& b : sys.blocks[size_t(r)]) b = M3();
      sys.blocks[size_t(r)][kCenter] = M3::identity();
      sys.rhs[size_t(r)] = v.deformed(sys.rows[size_t(r)]);
      return;
    }
    sys.blocks[size_t(r)] = cb[size_t(r)];
    sys.rhs[size_t(r)] = crhs[size_t(r)];
    const int node = sys.rows[size_t(r)];
    int x, y, z;
    v.idx3(node, x, y, z);
    const M3 ri = v.rotation(node);
    const V3 can_i = v.canonical(node);
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], c = z + d[2];
      if (!v.in_grid(a, b, c)) continue;
      const int jnode = v.lin(a, b, c);
      const int rr = sys.node_row[size_t(jnode)];
      if (rr < 0) continue;
      const V3 dij = can_i - v.canonical(jnode);
      add_to(sys.blocks[size_t(r)][kCenter], scaled(M3::identity(), 2.0 * params.w_r));
      sys.rhs[size_t(r)] += params.w_r * ((ri + v.rotation(jnode)) * dij);
      if (sys.frozen[size_t(rr)]) {
        sys.rhs[size_t(r)] += (2.0 * params.w_r) * v.deformed(jnode);
      } else {
        M3& blk = sys.blocks[size_t(r)][size_t(stencil_slot(d[0], d[1], d[2]))];
        const M3 s = scaled(M3::identity(), 2.0 * params.w_r);
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) blk.a[i][j] -= s.a[i][j];
      }
    }
  };
  if (params.parallel) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) finish_row(r);
  } else {
    for (int r = 0; r < n; ++r) finish_row(r);
  }
  return sys;
}

struct PcgRes {
  int iterations = 0;
  double relres = 0;
};

// solver.cpp:282-343
PcgRes pcg_solve(const NE& sys, std::vector<V3>& x, double tol, int max_iters, bool parallel) {
  const int n = sys.num_rows();
  PcgRes res;
  if (n == 0) return res;
  std::vector<V3> inv_diag(static_cast<size_t>(n));
  for (int r = 0; r < n; ++r) {
    const M3& d = sys.blocks[size_t(r)][kCenter];
    for (int k = 0; k < 3; ++k) inv_diag[size_t(r)][k] = d.a[k][k] > 1e-300 ? 1.0 / d.a[k][k] : 1.0;
  }
  double b_norm2 = 0;
  for (const V3& b : sys.rhs) b_norm2 += sqnorm(b);
  const double b_norm = std::sqrt(b_norm2);
  if (b_norm == 0) {
    std::fill(x.begin(), x.end(), V3());
    return res;
  }
  std::vector<V3> r(static_cast<size_t>(n)), z(static_cast<size_t>(n)), p(static_cast<size_t>(n)), ap(static_cast<size_t>(n));
  sys.multiply(x, ap, parallel);
  for (int i = 0; i < n; ++i) {
    r[size_t(i)] = sys.rhs[size_t(i)] - ap[size_t(i)];
    const V3 ri = r[size_t(i)], di = inv_diag[size_t(i)];
    z[size_t(i)] = {di.x * ri.x, di.y * ri.y, di.z * ri.z};
    p[size_t(i)] = z[size_t(i)];
  }
  auto dotv = [n](const std::vector<V3>& a, const std::vector<V3>& b) {
    double s = 0;
    for (int i = 0; i < n; ++i) s += dot(a[size_t(i)], b[size_t(i)]);
    return s;
  };
  double rz = dotv(r, z);
  double r_norm = std::sqrt(dotv(r, r));
  res.relres = r_norm / b_norm;
  const double stop = std::max(tol * r_norm, 1e-13 * b_norm);
  for (int it = 0; it < max_iters && r_norm > stop; ++it) {
    sys.multiply(p, ap, parallel);
    const double pap = dotv(p, ap);
    if (pap <= 0) break;
    const double alpha = rz / pap;
    for (int i = 0; i < n; ++i) {
      x[size_t(i)] += alpha * p[size_t(i)];
      r[size_t(i)] -= alpha * ap[size_t(i)];
      const V3 ri = r[size_t(i)], di = inv_diag[size_t(i)];
      z[size_t(i)] = {di.x * ri.x, di.y * ri.y, di.z * ri.z};
    }
    const double rz_new = dotv(r, z);
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int i = 0; i < n; ++i) p[size_t(i)] = z[size_t(i)] + beta * p[size_t(i)];
    r_norm = std::sqrt(dotv(r, r));
    res.relres = r_norm / b_norm;
    res.iterations = it + 1;
  }
  return res;
}

struct Energy {
  double total = 0, sparse = 0, dense = 0, reg = 0;
};

struct LogicError {};

// solver.cpp:345-383
Energy evaluate_energy(const Vol& v, const Pose& pose, const std::vector<Con>& cons,
                       const Params& params) {
  Energy e;
  for (const Con& c : cons) {
    V3 q;
    for (int k = 0; k < 8; ++k) {
      if (c.w[k] > 0 && !v.active(c.idx[k])) throw LogicError{};
      q += c.w[k] * v.deformed(c.idx[k]);
    }
    const V3 s = pose.apply(q);
    if (c.dense) {
      const double r = dot(s - c.target, c.normal);
      e.dense += c.conf * r * r;
    } else {
      e.sparse += c.conf * sqnorm(s - c.target);
    }
  }
  for (int i = 0; i < v.num_points(); ++i) {
    if (!v.active(i)) continue;
    const M3 ri = v.rotation(i);
    int x, y, z;
    v.idx3(i, x, y, z);
    const V3 can_i = v.canonical(i);
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], cz = z + d[2];
      if (!v.in_grid(a, b, cz)) continue;
      const int j = v.lin(a, b, cz);
      if (!v.active(j)) continue;
      const V3 resid = (v.deformed(i) - v.deformed(j)) - ri * (can_i - v.canonical(j));
      e.reg += sqnorm(resid);
    }
  }
  e.total = params.w_s * e.sparse + params.w_d * e.dense + params.w_r * e.reg;
  return e;
}

// solver.cpp:385-417
void update_rotations(Vol& v, bool parallel) {
  const int n = v.num_points();
  auto fit_one = [&](int i) {
    if (!v.active(i)) return;
    int x, y, z;
    v.idx3(i, x, y, z);
    const V3 can_i = v.canonical(i);
    M3 h;
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], c = z + d[2];
      if (!v.in_grid(a, b, c)) continue;
      const int j = v.lin(a, b, c);
      if (!v.active(j)) continue;
      const V3 rest = can_i - v.canonical(j);
      const V3 cur = v.deformed(i) - v.deformed(j);
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) h.a[p][q] += rest[p] * cur[q];
    }
    M3 u, vv;
    double sv[3];
    svd3(h, u, sv, vv);
    if (sv[1] < 1e-14) return;
    M3 r = vv * transpose(u);
    if (det(r) < 0) {
      M3 flip = M3::identity();
      flip.a[2][2] = -1;
      r = (vv * flip) * transpose(u);
    }
    v.set_rotation(i, r);
  };
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) fit_one(i);
  } else {
    for (int i = 0; i < n; ++i) fit_one(i);
  }
}

struct Trace {
  int level = 0, iteration = 0;
  Energy energy;
  int pcg_iterations = 0;
  double pcg_residual = 0;
  bool anomaly = false;
};

// solver.cpp:419-453
std::vector<Trace> flip_flop_solve(Vol& v, const Pose& pose, const std::vector<Con>& cons,
                                   const Params& params, int level) {
  std::vector<Trace> trace;
  Energy prev = evaluate_energy(v, pose, cons, params);
  if (prev.total == 0) return trace;
  Cache cache;
  std::vector<V3> x;
  for (int it = 0; it < params.ff_iters; ++it) {
    NE sys = build_normal_equations(v, pose, cons, params, &cache);
    x.resize(size_t(sys.num_rows()));
    for (int r = 0; r < sys.num_rows(); ++r) x[size_t(r)] = v.deformed(sys.rows[size_t(r)]);
    const PcgRes pcg = pcg_solve(sys, x, params.pcg_tol, params.pcg_max, params.parallel);
    for (int r = 0; r < sys.num_rows(); ++r)
      if (!sys.frozen[size_t(r)]) v.set_deformed(sys.rows[size_t(r)], x[size_t(r)]);
    update_rotations(v, params.parallel);
    Trace entry;
    entry.level = level;
    entry.iteration = it;
    entry.energy = evaluate_energy(v, pose, cons, params);
    entry.pcg_iterations = pcg.iterations;
    entry.pcg_residual = pcg.relres;
    entry.anomaly = entry.energy.total > prev.total + 1e-9 * prev.total;
    trace.push_back(entry);
    const double rel = (prev.total - entry.energy.total) / std::max(prev.total, 1e-300);
    prev = entry.energy;
    if (rel >= 0 && rel < params.ff_rel_tol) break;
  }
  return trace;
}

struct Level {
  Vol grid;
  std::vector<Con> cons;
};

struct InvalidArg {};

// solver.cpp:455-503 (level 0 keeps only the deformation/activity the coarse
// levels read; the solve itself runs on the caller's volume, solver.cpp:531)
std::vector<Level> build_hierarchy(const Vol& volume, const std::vector<Con>& cons, int levels) {
  if (levels < 1) throw InvalidArg{};
  std::vector<Level> h;
  h.reserve(size_t(levels));
  {
    Level l0;
    l0.grid.nx = volume.nx; l0.grid.ny = volume.ny; l0.grid.nz = volume.nz;
    l0.grid.voxel = volume.voxel; l0.grid.origin = volume.origin; l0.grid.mu = volume.mu;
    const size_t n = size_t(volume.num_points());
    l0.grid.o_def.assign(volume.deformed_, volume.deformed_ + 3 * n);
    l0.grid.o_eul.assign(volume.euler_, volume.euler_ + 3 * n);
    l0.grid.o_age.assign(volume.age_, volume.age_ + n);
    l0.grid.o_act.assign(volume.active_, volume.active_ + n);
    l0.cons = cons;
    h.push_back(std::move(l0));
    h.back().grid.rebind();
  }
  for (int l = 1; l < levels; ++l) {
    const Vol& fine = h.back().grid;
    const int fd[3] = {fine.nx, fine.ny, fine.nz};
    int cd[3];
    for (int k = 0; k < 3; ++k) cd[k] = (fd[k] - 1 + 1) / 2 + 1;
    if (cd[0] < 2 || cd[1] < 2 || cd[2] < 2) throw InvalidArg{};
    Level lv;
    lv.grid.make_owned(cd[0], cd[1], cd[2], fine.voxel * 2.0, fine.origin, false);
    Vol& coarse = lv.grid;
    for (int i = 0; i < coarse.num_points(); ++i) {  // solver.cpp:470-483
      const V3 xc = coarse.canonical(i);
      V3 xq = xc;
      for (int k = 0; k < 3; ++k)
        xq[k] = std::clamp(xq[k], fine.origin[k], fine.origin[k] + fine.voxel * (fd[k] - 1));
      coarse.set_deformed(i, fine.interpolate_deformed(xq) + (xc - xq));
      int nearest[3];
      for (int k = 0; k < 3; ++k)
        nearest[k] = std::clamp(int(std::lround((xq[k] - fine.origin[k]) / fine.voxel)), 0, fd[k] - 1);
      coarse.set_euler(i, fine.euler(fine.lin(nearest[0], nearest[1], nearest[2])));
    }
    for (int i = 0; i < fine.num_points(); ++i) {  // solver.cpp:485-490
      if (!fine.active(i)) continue;
      const V3 x = fine.canonical(i);
      if (!coarse.contains(x)) throw std::out_of_range("trilinear_anchors");
      int idx[8];
      double w[8];
      coarse.anchors(x, idx, w);
      for (int k = 0; k < 8; ++k) coarse.set_active(idx[k], true);
    }
    lv.cons = h.back().cons;  // solver.cpp:492-499
    for (Con& c : lv.cons) {
      if (!coarse.contains(c.canonical)) throw std::out_of_range("trilinear_anchors");
      coarse.anchors(c.canonical, c.idx, c.w);
      for (int k = 0; k < 8; ++k)
        if (c.w[k] > 0) coarse.set_active(c.idx[k], true);
    }
    h.push_back(std::move(lv));
    h.back().grid.rebind();
  }
  return h;
}

// solver.cpp:505-534
std::vector<Trace> solve_coarse_to_fine(Vol& volume, const Pose& pose,
                                        const std::vector<Con>& cons, const Params& params) {
  std::vector<Level> h = build_hierarchy(volume, cons, params.levels);
  std::vector<Trace> trace;
  for (int l = int(h.size()) - 1; l >= 1; --l) {
    auto t = flip_flop_solve(h[size_t(l)].grid, pose, h[size_t(l)].cons, params, l);
    trace.insert(trace.end(), t.begin(), t.end());
    Vol& fine = (l - 1 == 0) ? volume : h[size_t(l - 1)].grid;
    const Vol& coarse = h[size_t(l)].grid;
    const int cd[3] = {coarse.nx, coarse.ny, coarse.nz};
    for (int i = 0; i < fine.num_points(); ++i) {
      if (!fine.active(i)) continue;
      const V3 x = fine.canonical(i);
      fine.set_deformed(i, coarse.interpolate_deformed(x));
      int nearest[3];
      for (int k = 0; k < 3; ++k)
        nearest[k] = std::clamp(int(std::lround((x[k] - coarse.origin[k]) / coarse.voxel)), 0, cd[k] - 1);
      fine.set_euler(i, coarse.euler(coarse.lin(nearest[0], nearest[1], nearest[2])));
    }
  }
  auto t = flip_flop_solve(volume, pose, cons, params, 0);
  trace.insert(trace.end(), t.begin(), t.end());
  return trace;
}

// ---------------------------------------------------------------------------
// fusion.cpp
// ---------------------------------------------------------------------------
struct FrameV {
  int w = 0, h = 0;
  double fx = 0, fy = 0, cx = 0, cy = 0;
  const float* depth = nullptr;
  const float* color = nullptr;
  float d(int x, int y) const { return depth[size_t(y) * size_t(w) + size_t(x)]; }
};
FrameV frame_of(const wfk_frame_view* f) {
  FrameV r;
  r.w = f->intrinsics.width;
  r.h = f->intrinsics.height;
  r.fx = f->intrinsics.fx; r.fy = f->intrinsics.fy; r.cx = f->intrinsics.cx; r.cy = f->intrinsics.cy;
  r.depth = f->depth;
  r.color = f->color;
  return r;
}
bool intr_valid(const wfk_intrinsics& k) { return k.fx > 0 && k.fy > 0 && k.width > 0 && k.height > 0; }

struct FusionStats {
  int fused = 0, gate = 0, frustum = 0, occluded = 0;
};

// fusion.cpp:7-83
FusionStats integrate_frame(Vol& v, const FrameV& f, const Pose& pose, const wfk_fusion_params& p,
                            bool parallel) {
  FusionStats stats;
  const double mu = v.mu;
  const int n = v.num_points();
  std::vector<int> fused(size_t(n), 0), gate(size_t(n), 0), frustum(size_t(n), 0), occluded(size_t(n), 0);
  auto one = [&](int i) {
    if (!p.bootstrap && (!v.active(i) || v.age_[i] < p.k_min)) {
      gate[size_t(i)] = 1;
      return;
    }
    const V3 warped = v.warp_point(pose, v.canonical(i));
    if (warped.z <= 0) {
      frustum[size_t(i)] = 1;
      return;
    }
    const double ux = f.fx * warped.x / warped.z + f.cx;  // core.hpp:48-50
    const double uy = f.fy * warped.y / warped.z + f.cy;
    const int u = int(std::lround(ux));
    const int vv = int(std::lround(uy));
    if (u < 0 || vv < 0 || u >= f.w || vv >= f.h) {
      frustum[size_t(i)] = 1;
      return;
    }
    double depth = f.d(u, vv);
    {
      const int u0 = std::clamp(int(std::floor(ux)), 0, f.w - 2);
      const int v0 = std::clamp(int(std::floor(uy)), 0, f.h - 2);
      const float d00 = f.d(u0, v0), d10 = f.d(u0 + 1, v0);
      const float d01 = f.d(u0, v0 + 1), d11 = f.d(u0 + 1, v0 + 1);
      if (d00 > 0 && d10 > 0 && d01 > 0 && d11 > 0) {
        const double fu = std::clamp(ux - u0, 0.0, 1.0);
        const double fv = std::clamp(uy - v0, 0.0, 1.0);
        depth = (1 - fv) * ((1 - fu) * d00 + fu * d10) + fv * ((1 - fu) * d01 + fu * d11);
      }
    }
    if (depth <= 0) {
      frustum[size_t(i)] = 1;
      return;
    }
    const double sdf = double(depth) - warped.z;
    if (sdf < -mu) {
      occluded[size_t(i)] = 1;
      return;
    }
    const double d = std::min(sdf, mu);
    const double w = p.sample_weight;
    const double w_old = v.weight_[i];
    v.tsdf_[i] = float((w_old * v.tsdf_[i] + w * d) / (w_old + w));
    if (f.color) {
      const size_t pix = 3 * (size_t(vv) * size_t(f.w) + size_t(u));
      float* c = v.color_ + 3 * size_t(i);
      for (int k = 0; k < 3; ++k) {
        float ck = (float(w_old) * c[k] + float(w) * f.color[pix + size_t(k)]) / float(w_old + w);
        c[k] = std::clamp(ck, 0.f, 255.f);
      }
    }
    v.weight_[i] = float(std::min(w_old + w, p.w_max));
    fused[size_t(i)] = 1;
  };
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) one(i);
  } else {
    for (int i = 0; i < n; ++i) one(i);
  }
  for (int i = 0; i < n; ++i) {
    stats.fused += fused[size_t(i)];
    stats.gate += gate[size_t(i)];
    stats.frustum += frustum[size_t(i)];
    stats.occluded += occluded[size_t(i)];
  }
  return stats;
}

// fusion.cpp:85-122
wfk_expansion_stats expand_grid(Vol& v) {
  wfk_expansion_stats stats{0, 0};
  std::vector<uint8_t> was(size_t(v.num_points()));
  for (int i = 0; i < v.num_points(); ++i) was[size_t(i)] = v.active(i);
  compute_active_set(v);
  for (int i = 0; i < v.num_points(); ++i) {
    if (!v.active(i) || was[size_t(i)]) continue;
    ++stats.activated;
    int x, y, z;
    v.idx3(i, x, y, z);
    const V3 can = v.canonical(i);
    V3 sum;
    int found = 0, nearest = -1;
    for (const auto& d : kFace) {
      const int a = x + d[0], b = y + d[1], c = z + d[2];
      if (!v.in_grid(a, b, c)) continue;
      const int j = v.lin(a, b, c);
      if (!was[size_t(j)]) continue;
      sum += v.deformed(j) + v.rotation(j) * (can - v.canonical(j));
      if (nearest < 0) nearest = j;
      ++found;
    }
    v.age_[i] = 0;
    if (found > 0) {
      v.set_deformed(i, sum / double(found));
      v.set_euler(i, v.euler(nearest));
    } else {
      v.set_deformed(i, can);
      v.set_euler(i, V3());
      ++stats.orphans;
    }
  }
  return stats;
}

// ---------------------------------------------------------------------------
// correspond.cpp
// ---------------------------------------------------------------------------
struct Maps {
  int w = 0, h = 0;
  double* point = nullptr;
  double* normal = nullptr;
  uint8_t* pv = nullptr;
  uint8_t* nv = nullptr;
  size_t idx(int x, int y) const { return size_t(y) * size_t(w) + size_t(x); }
  V3 P(size_t i) const { return {point[3 * i], point[3 * i + 1], point[3 * i + 2]}; }
  V3 N(size_t i) const { return {normal[3 * i], normal[3 * i + 1], normal[3 * i + 2]}; }
};

// correspond.cpp:7-57
void backproject_depth(const FrameV& f, Maps& m, bool parallel) {
  const int w = f.w, h = f.h;
  const size_t n = size_t(w) * size_t(h);
  std::fill(m.point, m.point + 3 * n, 0.0);
  std::fill(m.normal, m.normal + 3 * n, 0.0);
  std::fill(m.pv, m.pv + n, 0);
  std::fill(m.nv, m.nv + n, 0);
  auto row_points = [&](int y) {
    for (int x = 0; x < w; ++x) {
      const float d = f.d(x, y);
      if (d <= 0.f) continue;
      const double dd = d;
      const size_t i = m.idx(x, y);
      m.point[3 * i] = (double(x) - f.cx) / f.fx * dd;  // core.hpp:52-54
      m.point[3 * i + 1] = (double(y) - f.cy) / f.fy * dd;
      m.point[3 * i + 2] = dd;
      m.pv[i] = 1;
    }
  };
  auto row_normals = [&](int y) {
    if (y == 0 || y == h - 1) return;
    for (int x = 1; x < w - 1; ++x) {
      const size_t p = m.idx(x, y);
      if (!m.pv[p] || !m.pv[m.idx(x - 1, y)] || !m.pv[m.idx(x + 1, y)] || !m.pv[m.idx(x, y - 1)] ||
          !m.pv[m.idx(x, y + 1)])
        continue;
      const V3 du = m.P(m.idx(x + 1, y)) - m.P(m.idx(x - 1, y));
      const V3 dv = m.P(m.idx(x, y + 1)) - m.P(m.idx(x, y - 1));
      V3 nn = cross(du, dv);
      const double len = norm(nn);
      if (len < 1e-20) continue;
      nn = nn / len;
      if (dot(nn, m.P(p)) > 0) nn = -nn;
      m.normal[3 * p] = nn.x; m.normal[3 * p + 1] = nn.y; m.normal[3 * p + 2] = nn.z;
      m.nv[p] = 1;
    }
  };
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) row_points(y);
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) row_normals(y);
  } else {
    for (int y = 0; y < h; ++y) row_points(y);
    for (int y = 0; y < h; ++y) row_normals(y);
  }
}

inline double kernel(double r, double eps) { return 1.0 - r / eps; }  // correspond.hpp:53
// correspond.cpp:59-67
double dense_confidence(double dist, double nd, double vd, const wfk_correspond_params& p) {
  const double kd = kernel(dist, p.eps_d);
  const double kn = kernel(1.0 - nd, p.eps_n);
  const double kv = kernel(1.0 - vd, p.eps_v);
  if (kd < 0 || kn < 0 || kv < 0) return 0.0;
  const double avg = (kd + kn + kv) / 3.0;
  return avg * avg;
}

// correspond.cpp:69-112
bool sample_point_normal(const Maps& maps, double ux, double uy, V3& point, V3& normal) {
  const int tu = int(std::lround(ux));
  const int tv = int(std::lround(uy));
  if (tu < 0 || tv < 0 || tu >= maps.w || tv >= maps.h) return false;
  const int u0 = std::clamp(int(std::floor(ux)), 0, maps.w - 2);
  const int v0 = std::clamp(int(std::floor(uy)), 0, maps.h - 2);
  bool smooth = true;
  double zmin = std::numeric_limits<double>::infinity(), zmax = -zmin;
  for (int dy = 0; dy < 2 && smooth; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const size_t p = maps.idx(u0 + dx, v0 + dy);
      if (!maps.pv[p] || !maps.nv[p]) {
        smooth = false;
        break;
      }
      zmin = std::min(zmin, maps.point[3 * p + 2]);
      zmax = std::max(zmax, maps.point[3 * p + 2]);
    }
  if (smooth && zmax - zmin < 0.05) {
    const double fu = std::clamp(ux - u0, 0.0, 1.0);
    const double fv = std::clamp(uy - v0, 0.0, 1.0);
    point = V3();
    normal = V3();
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double w = (dx ? fu : 1 - fu) * (dy ? fv : 1 - fv);
        const size_t p = maps.idx(u0 + dx, v0 + dy);
        point += w * maps.P(p);
        normal += w * maps.N(p);
      }
    const double len = norm(normal);
    if (len > 1e-12) {
      normal = normal / len;
      return true;
    }
  }
  const size_t tp = maps.idx(tu, tv);
  if (!maps.pv[tp] || !maps.nv[tp]) return false;
  point = maps.P(tp);
  normal = maps.N(tp);
  return true;
}

struct GBuf {
  int w = 0, h = 0;
  float* depth = nullptr;
  double *point = nullptr, *normal = nullptr, *canonical = nullptr;
  size_t idx(int x, int y) const { return size_t(y) * size_t(w) + size_t(x); }
  V3 get(const double* a, size_t i) const { return {a[3 * i], a[3 * i + 1], a[3 * i + 2]}; }
};

// correspond.cpp:114-150
std::vector<Con> find_dense(const GBuf& buf, const Maps& maps, const wfk_intrinsics& K,
                            const wfk_correspond_params& params, const Vol& v) {
  std::vector<Con> out;
  for (int y = 0; y < buf.h; ++y)
    for (int x = 0; x < buf.w; ++x) {
      const size_t bp = buf.idx(x, y);
      if (!std::isfinite(buf.depth[bp])) continue;
      const V3 pc = buf.get(buf.point, bp);
      const V3 nc = buf.get(buf.normal, bp);
      if (sqnorm(nc) < 0.5) continue;
      const double ux = K.fx * pc.x / pc.z + K.cx;
      const double uy = K.fy * pc.y / pc.z + K.cy;
      V3 pa, na;
      if (!sample_point_normal(maps, ux, uy, pa, na)) continue;
      const V3 vdir = -normalized(pc);
      const double w = dense_confidence(norm(pc - pa), dot(nc, na), dot(nc, vdir), params);
      if (w <= 0) continue;
      Con c;
      c.dense = true;
      c.canonical = buf.get(buf.canonical, bp);
      if (!v.contains(c.canonical)) continue;
      v.anchors(c.canonical, c.idx, c.w);
      c.target = pa;
      c.normal = na;
      c.conf = w;
      out.push_back(c);
    }
  return out;
}

// ---------------------------------------------------------------------------
// DeformableVolume::invert_warp (volume.cpp:68-126)
// ---------------------------------------------------------------------------
// deformed_jacobian (volume.cpp:68-93): analytic d interpolate_deformed / dx
M3 deformed_jacobian(const Vol& v, const V3& x) {
  const V3 rel = (x - v.origin) / v.voxel;
  const int d[3] = {v.nx, v.ny, v.nz};
  int cell[3];
  double f[3];
  for (int k = 0; k < 3; ++k) {
    int c = static_cast<int>(std::floor(rel[k]));
    c = std::clamp(c, 0, d[k] - 2);
    cell[k] = c;
    f[k] = rel[k] - c;
  }
  M3 j;  // zero-initialised
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const V3 t = v.deformed(v.lin(cell[0] + dx, cell[1] + dy, cell[2] + dz));
        const double wx = dx ? f[0] : 1 - f[0];
        const double wy = dy ? f[1] : 1 - f[1];
        const double wz = dz ? f[2] : 1 - f[2];
        const double g[3] = {(dx ? 1.0 : -1.0) * wy * wz, (dy ? 1.0 : -1.0) * wx * wz, (dz ? 1.0 : -1.0) * wx * wy};
        for (int c = 0; c < 3; ++c) {
          j.a[0][c] += t.x * g[c];
          j.a[1][c] += t.y * g[c];
          j.a[2][c] += t.z * g[c];
        }
      }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) j.a[r][c] = j.a[r][c] / v.voxel;
  return j;
}

// Eigen PartialPivLU<Matrix3d>::solve restated: column k takes the row of the
// largest |entry| at or below the diagonal (first one on ties), the column
// below the pivot is divided by it and the trailing block takes the rank-1
// update; solve = row permutation, unit-lower forward, upper back substitution.
V3 lu3_solve(M3 a, const V3& b) {
  int perm[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int p = k;
    for (int i = k + 1; i < 3; ++i)
      if (std::abs(a.a[i][k]) > std::abs(a.a[p][k])) p = i;
    if (a.a[p][k] != 0) {
      if (p != k) {
        for (int c = 0; c < 3; ++c) std::swap(a.a[k][c], a.a[p][c]);
        std::swap(perm[k], perm[p]);
      }
      for (int i = k + 1; i < 3; ++i) a.a[i][k] /= a.a[k][k];
    }
    for (int i = k + 1; i < 3; ++i)
      for (int c = k + 1; c < 3; ++c) a.a[i][c] -= a.a[i][k] * a.a[k][c];
  }
  const double bb[3] = {b.x, b.y, b.z};
  double x[3] = {bb[perm[0]], bb[perm[1]], bb[perm[2]]};
  for (int i = 1; i < 3; ++i)
    for (int j = 0; j < i; ++j) x[i] -= a.a[i][j] * x[j];
  for (int i = 2; i >= 0; --i) {
    for (int j = 2; j > i; --j) x[i] -= a.a[i][j] * x[j];
    x[i] /= a.a[i][i];
  }
  return {x[0], x[1], x[2]};
}

bool invert_warp(const Vol& v, const Pose& pose, const V3& y, const V3& seed, int max_iters, double tol, V3& out) {
  const V3 target = transpose(pose.r) * (y - pose.t);  // GlobalPose::apply_inverse (core.hpp:25-27)
  V3 x = seed;
  if (!v.contains(x)) return false;
  const double hi[3] = {v.origin.x + v.voxel * (v.nx - 1), v.origin.y + v.voxel * (v.ny - 1),
                        v.origin.z + v.voxel * (v.nz - 1)};
  const double lo[3] = {v.origin.x, v.origin.y, v.origin.z};
  for (int it = 0; it < max_iters; ++it) {
    const V3 r = v.interpolate_deformed(x) - target;
    if (norm(r) <= tol) {
      out = x;
      return true;
    }
    const M3 j = deformed_jacobian(v, x);
    V3 step = std::abs(det(j)) > 1e-12 ? lu3_solve(j, r) : r;  // damped fixed-point fallback
    const double max_step = v.voxel;
    if (norm(step) > max_step) step = step * (max_step / norm(step));
    V3 xn = x - step;
    for (int k = 0; k < 3; ++k) xn[k] = std::clamp(xn[k], lo[k], hi[k]);  // keep the iterate inside the grid
    x = xn;
  }
  if (norm(v.interpolate_deformed(x) - target) <= tol) {
    out = x;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// global pose: estimate_global_pose (solver.cpp:536-614)
// ---------------------------------------------------------------------------
// Eigen 3.4 LDLT<MatrixXd> (ldlt_inplace<Lower>::unblocked and _solve_impl),
// restated: in-place on the lower triangle; at step k the remaining diagonal
// entry of largest magnitude is moved to k by a symmetric transposition; the
// k-th row of L is updated against the previous pivots, then column k below
// the diagonal is divided by the pivot (skipped for a zero pivot).  Solve:
// permute, unit-lower forward substitution, divide by D (pseudo-inverse: a
// |D_i| not above the smallest normal double gives 0), unit-upper back
// substitution with L^T, undo the permutation.
struct Ldlt {
  int n = 0;
  double a[8][8];
  int tr[8];
};
void ldlt_factor(Ldlt& f) {
  const int n = f.n;
  double temp[8];
  for (int k = 0; k < n; ++k) {
    int big = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(f.a[i][i]) > std::abs(f.a[big][big])) big = i;
    f.tr[k] = big;
    if (big != k) {
      for (int j = 0; j < k; ++j) std::swap(f.a[k][j], f.a[big][j]);
      for (int i = big + 1; i < n; ++i) std::swap(f.a[i][k], f.a[i][big]);
      std::swap(f.a[k][k], f.a[big][big]);
      for (int i = k + 1; i < big; ++i) {
        const double t = f.a[i][k];
        f.a[i][k] = f.a[big][i];
        f.a[big][i] = t;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = f.a[j][j] * f.a[k][j];
      double d = 0;
      for (int j = 0; j < k; ++j) d += f.a[k][j] * temp[j];
      f.a[k][k] -= d;
      for (int i = k + 1; i < n; ++i) {
        double s = 0;
        for (int j = 0; j < k; ++j) s += f.a[i][j] * temp[j];
        f.a[i][k] -= s;
      }
    }
    const double akk = f.a[k][k];
    if (std::abs(akk) > 0)
      for (int i = k + 1; i < n; ++i) f.a[i][k] /= akk;
  }
}
void ldlt_solve(const Ldlt& f, const double* b, double* x) {
  const int n = f.n;
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) std::swap(x[k], x[f.tr[k]]);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= f.a[i][j] * x[j];
  for (int i = 0; i < n; ++i) {
    const double d = f.a[i][i];
    x[i] = std::abs(d) > std::numeric_limits<double>::min() ? x[i] / d : 0.0;
  }
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) x[i] -= f.a[j][i] * x[j];
  for (int k = n - 1; k >= 0; --k) std::swap(x[k], x[f.tr[k]]);
}

// orthonormalize (core.cpp:30-40): nearest rotation through the Jacobi SVD
M3 orthonormalize(const M3& m) {
  M3 u, v;
  double sv[3];
  svd3(m, u, sv, v);
  M3 r = u * transpose(v);
  if (det(r) < 0) {
    M3 flip = M3::identity();
    flip.a[2][2] = -1;
    r = u * flip * transpose(v);
  }
  return r;
}

struct IcpOut {
  Pose pose;
  bool converged = false, degraded = false;
  double rms = 0;
  int iterations = 0;
};
IcpOut estimate_global_pose(const GBuf& buf, const Maps& maps, const wfk_intrinsics& K, const Vol& vol,
                            const Pose& initial, const wfk_icp_params& params) {
  IcpOut res;
  res.pose = initial;
  struct Source {
    V3 q, n0;
  };
  std::vector<Source> sources;
  const M3 r0t = transpose(initial.r);
  for (int y = 0; y < buf.h; ++y)  // solver.cpp:549-558
    for (int x = 0; x < buf.w; ++x) {
      const size_t p = buf.idx(x, y);
      if (!std::isfinite(buf.depth[p])) continue;
      const V3 nrm = buf.get(buf.normal, p);
      if (sqnorm(nrm) < 0.5) continue;
      const V3 can = buf.get(buf.canonical, p);
      if (!vol.contains(can)) continue;
      sources.push_back({vol.interpolate_deformed(can), r0t * nrm});
    }
  double prev_rms = std::numeric_limits<double>::infinity();
  Pose prev_pose = initial;
  for (int it = 0; it < params.max_iters; ++it) {
    double h[6][6] = {}, g[6] = {};
    double err = 0, wsum = 0;
    int count = 0;
    for (const Source& s : sources) {  // solver.cpp:567-589
      const V3 p = res.pose.apply(s.q);
      const double ux = K.fx * p.x / p.z + K.cx;
      const double uy = K.fy * p.y / p.z + K.cy;
      V3 pa, na;
      if (!sample_point_normal(maps, ux, uy, pa, na)) continue;
      const V3 nc = res.pose.r * s.n0;
      const V3 v = -normalized(p);
      const double w = dense_confidence(norm(p - pa), dot(nc, na), dot(nc, v), params.corr);
      if (w <= 0) continue;
      const V3 c = cross(p, na);
      const double j[6] = {c.x, c.y, c.z, na.x, na.y, na.z};
      const double r = dot(na, p - pa);
      for (int i = 0; i < 6; ++i) {
        const double wj = w * j[i];
        for (int k = 0; k < 6; ++k) h[i][k] += wj * j[k];
        g[i] += wj * r;
      }
      err += w * r * r;
      wsum += w;
      ++count;
    }
    if (count < params.min_correspondences) {  // :590-593
      res.degraded = true;
      return res;
    }
    res.rms = std::sqrt(err / std::max(wsum, 1e-300));
    res.iterations = it + 1;
    if (res.rms > prev_rms * (1.0 - std::max(params.rel_tol, params.min_improvement))) {  // :599-604
      res.pose = prev_pose;
      res.rms = prev_rms;
      res.converged = true;
      break;
    }
    prev_rms = res.rms;
    prev_pose = res.pose;
    double dmax = h[0][0];
    for (int i = 1; i < 6; ++i) dmax = std::max(dmax, h[i][i]);
    const double damp = 1e-3 * dmax;  // :608
    Ldlt f;
    f.n = 6;
    for (int i = 0; i < 6; ++i)
      for (int k = 0; k < 6; ++k) f.a[i][k] = h[i][k] + (i == k ? damp : 0.0);
    ldlt_factor(f);
    double mg[6], delta[6];
    for (int i = 0; i < 6; ++i) mg[i] = -g[i];
    ldlt_solve(f, mg, delta);
    M3 step = M3::identity();  // I + [omega]_x (:610-613)
    step.a[0][1] += -delta[2];
    step.a[0][2] += delta[1];
    step.a[1][0] += delta[2];
    step.a[1][2] += -delta[0];
    step.a[2][0] += -delta[1];
    step.a[2][1] += delta[0];
    res.pose.r = orthonormalize(step * res.pose.r);
    res.pose.t = step * res.pose.t + V3{delta[3], delta[4], delta[5]};
  }
  return res;
}

// ---------------------------------------------------------------------------
// isosurface.cpp / rasterize.cpp
// ---------------------------------------------------------------------------
struct Mesh {
  std::vector<V3> can, def, nrm;
  std::vector<F3> col;
  std::vector<std::array<int, 3>> tri;
};

struct CellEdge {
  int corner, axis;
};
// isosurface.cpp:25-35
CellEdge classify_edge(int e) {
  const int a = kWfMcEdgeCorners[e][0], b = kWfMcEdgeCorners[e][1];
  const int* oa = kWfMcCornerOffset[a];
  const int* ob = kWfMcCornerOffset[b];
  for (int axis = 0; axis < 3; ++axis)
    if (oa[axis] != ob[axis]) return {oa[axis] < ob[axis] ? a : b, axis};
  return {a, 0};
}
inline int hexval(char c) { return c <= '9' ? c - '0' : c - 'a' + 10; }

// isosurface.cpp:39-97
Mesh extract_mesh(const Vol& v, const Pose& pose) {
  Mesh mesh;
  std::unordered_map<int64_t, int> edge_vertices;
  CellEdge info[12];
  for (int e = 0; e < 12; ++e) info[e] = classify_edge(e);
  for (int cz = 0; cz < v.nz - 1; ++cz)
    for (int cy = 0; cy < v.ny - 1; ++cy)
      for (int cx = 0; cx < v.nx - 1; ++cx) {
        int ci[8];
        double cv[8];
        bool observed = true;
        int cube = 0;
        for (int c = 0; c < 8; ++c) {
          const int* o = kWfMcCornerOffset[c];
          ci[c] = v.lin(cx + o[0], cy + o[1], cz + o[2]);
          if (v.weight_[ci[c]] <= 0.f) {
            observed = false;
            break;
          }
          cv[c] = v.tsdf_[ci[c]];
          if (cv[c] < 0) cube |= 1 << c;
        }
        if (!observed || cube == 0 || cube == 255) continue;
        const char* tri = kWfMcCases[cube];
        for (int n = 0; tri[n]; n += 3) {
          int t[3];
          for (int k = 0; k < 3; ++k) {
            const int e = hexval(tri[n + k]);
            const CellEdge ce = info[e];
            const int64_t key = int64_t(ci[ce.corner]) * 3 + ce.axis;  // isosurface.cpp:15-17
            auto it = edge_vertices.find(key);
            if (it == edge_vertices.end()) {
              const int a = kWfMcEdgeCorners[e][0], b = kWfMcEdgeCorners[e][1];
              const double va = cv[a], vb = cv[b];
              const V3 pa = v.canonical(ci[a]);
              const V3 pb = v.canonical(ci[b]);
              const double s = va / (va - vb);
              const V3 p = pa + s * (pb - pa);
              it = edge_vertices.emplace(key, int(mesh.can.size())).first;
              mesh.can.push_back(p);
              mesh.def.push_back(v.warp_point(pose, p));
              mesh.col.push_back(v.sample_color(p));
            }
            t[k] = it->second;
          }
          std::swap(t[1], t[2]);
          if (t[0] != t[1] && t[1] != t[2] && t[0] != t[2]) mesh.tri.push_back({t[0], t[1], t[2]});
        }
      }
  return mesh;
}

// isosurface.cpp:99-112
void compute_normals(Mesh& mesh) {
  mesh.nrm.assign(mesh.can.size(), V3());
  for (const auto& t : mesh.tri) {
    const V3& a = mesh.def[size_t(t[0])];
    const V3& b = mesh.def[size_t(t[1])];
    const V3& c = mesh.def[size_t(t[2])];
    const V3 an = cross(b - a, c - a);
    for (int k = 0; k < 3; ++k) mesh.nrm[size_t(t[k])] += an;
  }
  for (V3& n : mesh.nrm) {
    const double len = norm(n);
    if (len > 1e-20) n = n / len;
  }
}

struct TriSetup {  // rasterize.cpp:11-22
  double sx[3], sy[3];
  double inv_z[3];
  V3 point_oz[3], normal_oz[3], canon_oz[3];
  double inv_area;
  int ymin, ymax, xmin, xmax;
  bool top_left[3];
};
inline double edge_fn(double ax, double ay, double bx, double by, double px, double py) {
  return (bx - ax) * (py - ay) - (by - ay) * (px - ax);  // rasterize.cpp:24-26
}

// rasterize.cpp:29-137
void rasterize(const Mesh& mesh, const wfk_intrinsics& K, bool parallel, GBuf& buf) {
  const size_t npx = size_t(K.width) * size_t(K.height);
  std::fill(buf.depth, buf.depth + npx, std::numeric_limits<float>::infinity());
  std::fill(buf.point, buf.point + 3 * npx, 0.0);
  std::fill(buf.normal, buf.normal + 3 * npx, 0.0);
  std::fill(buf.canonical, buf.canonical + 3 * npx, 0.0);
  if (mesh.tri.empty()) return;
  const bool have_normals = mesh.nrm.size() == mesh.can.size();
  constexpr double kNear = 1e-3;
  std::vector<TriSetup> setups;
  setups.reserve(mesh.tri.size());
  for (const auto& tri : mesh.tri) {
    const V3* v[3] = {&mesh.def[size_t(tri[0])], &mesh.def[size_t(tri[1])], &mesh.def[size_t(tri[2])]};
    if (v[0]->z < kNear || v[1]->z < kNear || v[2]->z < kNear) continue;
    TriSetup t;
    int order[3] = {0, 1, 2};
    for (int k = 0; k < 3; ++k) {
      t.sx[k] = K.fx * v[k]->x / v[k]->z + K.cx;
      t.sy[k] = K.fy * v[k]->y / v[k]->z + K.cy;
    }
    double area2 = edge_fn(t.sx[0], t.sy[0], t.sx[1], t.sy[1], t.sx[2], t.sy[2]);
    if (area2 == 0.0) continue;
    if (area2 < 0) {
      std::swap(t.sx[1], t.sx[2]);
      std::swap(t.sy[1], t.sy[2]);
      std::swap(order[1], order[2]);
      area2 = -area2;
    }
    for (int k = 0; k < 3; ++k) {
      const int vi = tri[size_t(order[k])];
      const double z = mesh.def[size_t(vi)].z;
      t.inv_z[k] = 1.0 / z;
      t.point_oz[k] = mesh.def[size_t(vi)] / z;
      t.normal_oz[k] = (have_normals ? mesh.nrm[size_t(vi)] : V3()) / z;
      t.canon_oz[k] = mesh.can[size_t(vi)] / z;
    }
    t.inv_area = 1.0 / area2;
    double uxmin = t.sx[0], uxmax = t.sx[0], uymin = t.sy[0], uymax = t.sy[0];
    for (int k = 1; k < 3; ++k) {
      uxmin = std::min(uxmin, t.sx[k]);
      uxmax = std::max(uxmax, t.sx[k]);
      uymin = std::min(uymin, t.sy[k]);
      uymax = std::max(uymax, t.sy[k]);
    }
    t.xmin = std::max(0, int(std::ceil(uxmin)));
    t.xmax = std::min(K.width - 1, int(std::floor(uxmax)));
    t.ymin = std::max(0, int(std::ceil(uymin)));
    t.ymax = std::min(K.height - 1, int(std::floor(uymax)));
    if (t.xmin > t.xmax || t.ymin > t.ymax) continue;
    for (int k = 0; k < 3; ++k) {
      const double ax = t.sx[k], ay = t.sy[k];
      const double bx = t.sx[(k + 1) % 3], by = t.sy[(k + 1) % 3];
      t.top_left[k] = (ay == by && bx > ax) || (by < ay);
    }
    setups.push_back(t);
  }
  auto process_row = [&](int y) {
    const double py = double(y);
    for (const TriSetup& t : setups) {
      if (y < t.ymin || y > t.ymax) continue;
      for (int x = t.xmin; x <= t.xmax; ++x) {
        const double px = double(x);
        bool inside = true;
        double w[3];
        for (int k = 0; k < 3; ++k) {
          const int a = (k + 1) % 3, b = (k + 2) % 3;
          w[k] = edge_fn(t.sx[a], t.sy[a], t.sx[b], t.sy[b], px, py);
          if (w[k] < 0 || (w[k] == 0 && !t.top_left[(k + 1) % 3])) {
            inside = false;
            break;
          }
        }
        if (!inside) continue;
        const double l0 = w[0] * t.inv_area;
        const double l1 = w[1] * t.inv_area;
        const double l2 = 1.0 - l0 - l1;
        const double inv_z = l0 * t.inv_z[0] + l1 * t.inv_z[1] + l2 * t.inv_z[2];
        const double z = 1.0 / inv_z;
        const size_t p = buf.idx(x, y);
        if (float(z) < buf.depth[p]) {
          buf.depth[p] = float(z);
          const V3 pt = (l0 * t.point_oz[0] + l1 * t.point_oz[1] + l2 * t.point_oz[2]) * z;
          const V3 nn = (l0 * t.normal_oz[0] + l1 * t.normal_oz[1] + l2 * t.normal_oz[2]) * z;
          const double nl = norm(nn);
          const V3 nrm = nl > 1e-20 ? nn / nl : V3();
          const V3 cn = (l0 * t.canon_oz[0] + l1 * t.canon_oz[1] + l2 * t.canon_oz[2]) * z;
          buf.point[3 * p] = pt.x; buf.point[3 * p + 1] = pt.y; buf.point[3 * p + 2] = pt.z;
          buf.normal[3 * p] = nrm.x; buf.normal[3 * p + 1] = nrm.y; buf.normal[3 * p + 2] = nrm.z;
          buf.canonical[3 * p] = cn.x; buf.canonical[3 * p + 1] = cn.y; buf.canonical[3 * p + 2] = cn.z;
        }
      }
    }
  };
  if (parallel) {
#pragma omp parallel for schedule(static)
    for (int y = 0; y < K.height; ++y) process_row(y);
  } else {
    for (int y = 0; y < K.height; ++y) process_row(y);
  }
}

void fill_energy(const Energy& e, wfk_energy* o) {
  o->total = e.total;
  o->sparse = e.sparse;
  o->dense = e.dense;
  o->reg = e.reg;
}
int export_trace(const std::vector<Trace>& t, wfk_trace_entry* out, int32_t cap, int32_t* n_out) {
  if (n_out) *n_out = int32_t(t.size());
  if (int64_t(t.size()) > int64_t(cap) || (!out && !t.empty()))
    return fail(WFK_E_CAPACITY, "trace buffer too small");
  for (size_t i = 0; i < t.size(); ++i) {
    out[i].level = t[i].level;
    out[i].iteration = t[i].iteration;
    fill_energy(t[i].energy, &out[i].energy);
    out[i].pcg_iterations = t[i].pcg_iterations;
    out[i].anomaly = t[i].anomaly ? 1 : 0;
    out[i].pcg_residual = t[i].pcg_residual;
  }
  return WFK_OK;
}

bool anchors_in_range(const Vol& v, const std::vector<Con>& cons) {
  const int n = v.num_points();
  for (const Con& c : cons)
    for (int k = 0; k < 8; ++k)
      if (c.idx[k] < 0 || c.idx[k] >= n) return false;
  return true;
}

}  // namespace

struct wfo_ne {
  NE ne;
};
struct wfo_mesh {
  Mesh m;
};

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

const char* wfo_last_error(void) { return g_err.c_str(); }

int wfo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
void wfo_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

void wfo_euler_to_matrix(const double abc[3], double r[9]) {
  to_rowmajor(euler_to_matrix({abc[0], abc[1], abc[2]}), r);
}
void wfo_matrix_to_euler(const double r[9], double abc[3]) {
  const V3 e = matrix_to_euler(from_rowmajor(r));
  abc[0] = e.x;
  abc[1] = e.y;
  abc[2] = e.z;
}
void wfo_svd3(const double a[9], double u[9], double s[3], double v[9]) {
  M3 mu, mv;
  svd3(from_rowmajor(a), mu, s, mv);
  to_rowmajor(mu, u);
  to_rowmajor(mv, v);
}

void wfo_volume_init(wfk_volume_view* view) {
  Vol v = Vol::borrow(view);
  const int n = v.num_points();
  for (int i = 0; i < n; ++i) {
    v.tsdf_[i] = 0.f;
    v.weight_[i] = 0.f;
    v.color_[3 * i] = v.color_[3 * i + 1] = v.color_[3 * i + 2] = 0.f;
    v.set_deformed(i, v.canonical(i));
    v.set_euler(i, V3());
    v.age_[i] = 0;
    v.active_[i] = 0;
  }
}

int wfo_contains(const wfk_volume_view* view, const double x[3]) {
  return Vol::borrow(view).contains({x[0], x[1], x[2]}) ? 1 : 0;
}
int wfo_trilinear_anchors(const wfk_volume_view* view, const double x[3], int32_t idx[8], double w[8]) {
  const Vol v = Vol::borrow(view);
  const V3 p{x[0], x[1], x[2]};
  if (!v.contains(p)) return fail(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  int ii[8];
  v.anchors(p, ii, w);
  for (int k = 0; k < 8; ++k) idx[k] = ii[k];
  return WFK_OK;
}
int wfo_warp_point(const wfk_volume_view* view, const wfk_pose* pose, const double x[3], double out[3]) {
  const Vol v = Vol::borrow(view);
  const V3 p{x[0], x[1], x[2]};
  if (!v.contains(p)) return fail(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  const V3 r = v.warp_point(pose_of(pose), p);
  out[0] = r.x;
  out[1] = r.y;
  out[2] = r.z;
  return WFK_OK;
}

int wfo_compute_active_set(wfk_volume_view* view, int32_t* out, int64_t cap, int64_t* n_out) {
  Vol v = Vol::borrow(view);
  const std::vector<int> a = compute_active_set(v);
  if (n_out) *n_out = int64_t(a.size());
  if (out) {
    if (int64_t(a.size()) > cap) return fail(WFK_E_CAPACITY, "active list buffer too small");
    std::copy(a.begin(), a.end(), out);
  }
  return WFK_OK;
}

int wfo_build_normal_equations(const wfk_volume_view* view, const wfk_pose* pose,
                               const wfk_correspondence* cons, int64_t ncons,
                               const wfk_solver_params* params, wfo_ne** out) {
  const Vol v = Vol::borrow(view);
  const auto c = cons_of(cons, ncons);
  if (!anchors_in_range(v, c)) return fail(WFK_E_OUT_OF_RANGE, "constraint anchor outside grid");
  auto* ne = new wfo_ne;
  ne->ne = build_normal_equations(v, pose_of(pose), c, params_of(params), nullptr);
  *out = ne;
  return WFK_OK;
}
int32_t wfo_ne_num_rows(const wfo_ne* ne) { return ne->ne.num_rows(); }
void wfo_ne_export(const wfo_ne* p, int32_t* rows, int32_t* node_row, double* blocks, int32_t* cols,
                   double* rhs, uint8_t* frozen) {
  const NE& ne = p->ne;
  const int n = ne.num_rows();
  if (rows) std::copy(ne.rows.begin(), ne.rows.end(), rows);
  if (node_row) std::copy(ne.node_row.begin(), ne.node_row.end(), node_row);
  for (int r = 0; r < n; ++r) {
    for (int s = 0; s < 27; ++s) {
      if (blocks) to_rowmajor(ne.blocks[size_t(r)][size_t(s)], blocks + (size_t(r) * 27 + size_t(s)) * 9);
      if (cols) cols[size_t(r) * 27 + size_t(s)] = ne.cols[size_t(r)][size_t(s)];
    }
    if (rhs) {
      rhs[3 * size_t(r)] = ne.rhs[size_t(r)].x;
      rhs[3 * size_t(r) + 1] = ne.rhs[size_t(r)].y;
      rhs[3 * size_t(r) + 2] = ne.rhs[size_t(r)].z;
    }
    if (frozen) frozen[r] = ne.frozen[size_t(r)];
  }
}
void wfo_ne_multiply(const wfo_ne* p, const double* x, double* y, int32_t exec) {
  const int n = p->ne.num_rows();
  std::vector<V3> xv(static_cast<size_t>(n)), yv;
  for (int i = 0; i < n; ++i) xv[size_t(i)] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  p->ne.multiply(xv, yv, exec != WFK_EXEC_SERIAL);
  for (int i = 0; i < n; ++i) {
    y[3 * i] = yv[size_t(i)].x;
    y[3 * i + 1] = yv[size_t(i)].y;
    y[3 * i + 2] = yv[size_t(i)].z;
  }
}
double wfo_ne_symmetry_error(const wfo_ne* p) { return p->ne.symmetry_error(); }
int wfo_ne_pcg_solve(const wfo_ne* p, double* x, double tol, int32_t max_iters, int32_t exec,
                     wfk_pcg_result* out) {
  const int n = p->ne.num_rows();
  std::vector<V3> xv(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) xv[size_t(i)] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
  const PcgRes r = pcg_solve(p->ne, xv, tol, max_iters, exec != WFK_EXEC_SERIAL);
  for (int i = 0; i < n; ++i) {
    x[3 * i] = xv[size_t(i)].x;
    x[3 * i + 1] = xv[size_t(i)].y;
    x[3 * i + 2] = xv[size_t(i)].z;
  }
  if (out) {
    out->iterations = r.iterations;
    out->relative_residual = r.relres;
  }
  return WFK_OK;
}
void wfo_ne_free(wfo_ne* ne) { delete ne; }

int wfo_evaluate_energy(const wfk_volume_view* view, const wfk_pose* pose,
                        const wfk_correspondence* cons, int64_t ncons,
                        const wfk_solver_params* params, wfk_energy* out) {
  const Vol v = Vol::borrow(view);
  const auto c = cons_of(cons, ncons);
  if (!anchors_in_range(v, c)) return fail(WFK_E_OUT_OF_RANGE, "constraint anchor outside grid");
  try {
    fill_energy(evaluate_energy(v, pose_of(pose), c, params_of(params)), out);
  } catch (const LogicError&) {
    return fail(WFK_E_LOGIC, "evaluate_energy: constraint anchors an inactive point");
  }
  return WFK_OK;
}

int wfo_update_rotations(wfk_volume_view* view, int32_t exec) {
  Vol v = Vol::borrow(view);
  update_rotations(v, exec != WFK_EXEC_SERIAL);
  return WFK_OK;
}

int wfo_flip_flop_solve(wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons,
                        int64_t ncons, const wfk_solver_params* params, int32_t level,
                        wfk_trace_entry* trace, int32_t cap, int32_t* n_out) {
  Vol v = Vol::borrow(view);
  const auto c = cons_of(cons, ncons);
  if (!anchors_in_range(v, c)) return fail(WFK_E_OUT_OF_RANGE, "constraint anchor outside grid");
  try {
    return export_trace(flip_flop_solve(v, pose_of(pose), c, params_of(params), level), trace, cap, n_out);
  } catch (const LogicError&) {
    return fail(WFK_E_LOGIC, "evaluate_energy: constraint anchors an inactive point");
  }
}

int wfo_hierarchy_info(const wfk_volume_view* view, const wfk_correspondence* cons, int64_t ncons,
                       int32_t levels, int32_t* dims_out, int64_t* active_out, int32_t want_level,
                       wfk_correspondence* level_cons_out) {
  const Vol v = Vol::borrow(view);
  const auto c = cons_of(cons, ncons);
  try {
    const auto h = build_hierarchy(v, c, levels);
    for (size_t l = 0; l < h.size(); ++l) {
      if (dims_out) {
        dims_out[3 * l] = h[l].grid.nx;
        dims_out[3 * l + 1] = h[l].grid.ny;
        dims_out[3 * l + 2] = h[l].grid.nz;
      }
      if (active_out) {
        int64_t a = 0;
        for (int i = 0; i < h[l].grid.num_points(); ++i) a += h[l].grid.active(i) ? 1 : 0;
        active_out[l] = a;
      }
    }
    if (level_cons_out && want_level >= 0 && want_level < int(h.size()))
      for (size_t i = 0; i < h[size_t(want_level)].cons.size(); ++i)
        con_to_c(h[size_t(want_level)].cons[i], level_cons_out[i]);
  } catch (const InvalidArg&) {
    return fail(WFK_E_INVALID_ARG, "build_hierarchy: bad level count");
  } catch (const std::out_of_range&) {
    return fail(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  }
  return WFK_OK;
}

int wfo_solve_coarse_to_fine(wfk_volume_view* view, const wfk_pose* pose, const wfk_correspondence* cons,
                             int64_t ncons, const wfk_solver_params* params, wfk_trace_entry* trace,
                             int32_t cap, int32_t* n_out) {
  Vol v = Vol::borrow(view);
  const auto c = cons_of(cons, ncons);
  if (!anchors_in_range(v, c)) return fail(WFK_E_OUT_OF_RANGE, "constraint anchor outside grid");
  try {
    return export_trace(solve_coarse_to_fine(v, pose_of(pose), c, params_of(params)), trace, cap, n_out);
  } catch (const LogicError&) {
    return fail(WFK_E_LOGIC, "evaluate_energy: constraint anchors an inactive point");
  } catch (const InvalidArg&) {
    return fail(WFK_E_INVALID_ARG, "build_hierarchy: bad level count");
  } catch (const std::out_of_range&) {
    return fail(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  }
}

int wfo_integrate_frame(wfk_volume_view* view, const wfk_frame_view* frame, const wfk_pose* pose,
                        const wfk_fusion_params* params, int32_t exec, wfk_fusion_stats* out) {
  Vol v = Vol::borrow(view);
  const FusionStats s = integrate_frame(v, frame_of(frame), pose_of(pose), *params, exec != WFK_EXEC_SERIAL);
  if (out) {
    out->fused = s.fused;
    out->skipped_gate = s.gate;
    out->skipped_frustum = s.frustum;
    out->skipped_occluded = s.occluded;
  }
  return WFK_OK;
}
int wfo_expand_grid(wfk_volume_view* view, wfk_expansion_stats* out) {
  Vol v = Vol::borrow(view);
  const wfk_expansion_stats s = expand_grid(v);
  if (out) *out = s;
  return WFK_OK;
}
int wfo_advance_ages(wfk_volume_view* view, const int32_t* idx, int64_t n) {  // fusion.cpp:124-126
  for (int64_t k = 0; k < n; ++k) view->age[idx[k]] += 1;
  return WFK_OK;
}

int wfo_backproject_depth(const wfk_frame_view* frame, int32_t exec, wfk_point_normal_map* out) {
  if (!intr_valid(frame->intrinsics)) return fail(WFK_E_INVALID_ARG, "backproject_depth: invalid intrinsics");
  Maps m;
  m.w = frame->intrinsics.width;
  m.h = frame->intrinsics.height;
  m.point = out->point;
  m.normal = out->normal;
  m.pv = out->point_valid;
  m.nv = out->normal_valid;
  out->width = m.w;
  out->height = m.h;
  backproject_depth(frame_of(frame), m, exec != WFK_EXEC_SERIAL);
  return WFK_OK;
}
double wfo_dense_confidence(double d, double nd, double vd, const wfk_correspond_params* p) {
  return dense_confidence(d, nd, vd, *p);
}
static Maps maps_of(const wfk_point_normal_map* m) {
  Maps r;
  r.w = m->width;
  r.h = m->height;
  r.point = m->point;
  r.normal = m->normal;
  r.pv = m->point_valid;
  r.nv = m->normal_valid;
  return r;
}
int wfo_sample_point_normal(const wfk_point_normal_map* maps, const double uv[2], double point[3],
                            double normal[3]) {
  V3 p, n;
  const bool ok = sample_point_normal(maps_of(maps), uv[0], uv[1], p, n);
  if (ok) {
    point[0] = p.x; point[1] = p.y; point[2] = p.z;
    normal[0] = n.x; normal[1] = n.y; normal[2] = n.z;
  }
  return ok ? 1 : 0;
}
static GBuf gbuf_of(const wfk_geometry_buffer* b) {
  GBuf g;
  g.w = b->width;
  g.h = b->height;
  g.depth = b->depth;
  g.point = b->point;
  g.normal = b->normal;
  g.canonical = b->canonical;
  return g;
}
int wfo_find_dense_correspondences(const wfk_geometry_buffer* buf, const wfk_point_normal_map* maps,
                                   const wfk_intrinsics* intr, const wfk_correspond_params* params,
                                   const wfk_volume_view* view, wfk_correspondence* out, int64_t cap,
                                   int64_t* n_out) {
  if (buf->width != maps->width || buf->height != maps->height)
    return fail(WFK_E_INVALID_ARG, "find_dense_correspondences: size mismatch");
  const auto c = find_dense(gbuf_of(buf), maps_of(maps), *intr, *params, Vol::borrow(view));
  if (n_out) *n_out = int64_t(c.size());
  if (int64_t(c.size()) > cap) return fail(WFK_E_CAPACITY, "correspondence buffer too small");
  for (size_t i = 0; i < c.size(); ++i) con_to_c(c[i], out[i]);
  return WFK_OK;
}
void pose_to_c(const Pose& q, wfk_pose* o) {
  for (int i = 0; i < 9; ++i) o->rotation[i] = q.r.a[i / 3][i % 3];
  o->translation[0] = q.t.x;
  o->translation[1] = q.t.y;
  o->translation[2] = q.t.z;
}
int wfo_estimate_global_pose(const wfk_geometry_buffer* buf, const wfk_point_normal_map* maps,
                             const wfk_intrinsics* intr, const wfk_volume_view* view, const wfk_pose* initial,
                             const wfk_icp_params* params, wfk_icp_result* out) {
  if (buf->width != maps->width || buf->height != maps->height)
    return fail(WFK_E_INVALID_ARG, "estimate_global_pose: size mismatch");
  const IcpOut r = estimate_global_pose(gbuf_of(buf), maps_of(maps), *intr, Vol::borrow(view), pose_of(initial),
                                        *params);
  std::memset(out, 0, sizeof(*out));
  pose_to_c(r.pose, &out->pose);
  out->converged = r.converged;
  out->degraded = r.degraded;
  out->rms = r.rms;
  out->iterations = r.iterations;
  return WFK_OK;
}
int wfo_invert_warp(const wfk_volume_view* view, const wfk_pose* pose, int64_t n, const double* y,
                    const double* seed, int32_t max_iters, double tol, double* x, uint8_t* ok) {
  const Vol v = Vol::borrow(view);
  const Pose p = pose_of(pose);
  for (int64_t i = 0; i < n; ++i) {
    V3 o{0, 0, 0};
    const bool good = invert_warp(v, p, {y[3 * i], y[3 * i + 1], y[3 * i + 2]},
                                  {seed[3 * i], seed[3 * i + 1], seed[3 * i + 2]}, max_iters, tol, o);
    ok[i] = good ? 1 : 0;
    x[3 * i] = o.x;
    x[3 * i + 1] = o.y;
    x[3 * i + 2] = o.z;
  }
  return WFK_OK;
}
int wfo_ldlt_solve(int n, const double* a, const double* b, double* x) {
  if (n < 1 || n > 8) return fail(WFK_E_INVALID_ARG, "ldlt: n out of range");
  Ldlt f;
  f.n = n;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) f.a[i][k] = a[i * n + k];
  ldlt_factor(f);
  ldlt_solve(f, b, x);
  return WFK_OK;
}
int wfo_sparse_to_constraints(const double* canonical, const double* target, int64_t n,
                              const wfk_volume_view* view, wfk_correspondence* out, int64_t* n_out) {
  const Vol v = Vol::borrow(view);  // correspond.cpp:152-169
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    const V3 c{canonical[3 * i], canonical[3 * i + 1], canonical[3 * i + 2]};
    if (!v.contains(c)) continue;
    Con o;
    o.dense = false;
    o.canonical = c;
    v.anchors(c, o.idx, o.w);
    o.target = {target[3 * i], target[3 * i + 1], target[3 * i + 2]};
    o.conf = 1.0;
    con_to_c(o, out[k++]);
  }
  *n_out = k;
  return WFK_OK;
}

int wfo_extract_mesh(const wfk_volume_view* view, const wfk_pose* pose, wfo_mesh** out) {
  auto* m = new wfo_mesh;
  m->m = extract_mesh(Vol::borrow(view), pose_of(pose));
  *out = m;
  return WFK_OK;
}
void wfo_mesh_sizes(const wfo_mesh* m, int64_t* nv, int64_t* nt) {
  *nv = int64_t(m->m.can.size());
  *nt = int64_t(m->m.tri.size());
}
void wfo_mesh_export(const wfo_mesh* mm, wfk_mesh_view* o) {
  const Mesh& m = mm->m;
  o->num_vertices = int64_t(m.can.size());
  o->num_triangles = int64_t(m.tri.size());
  for (size_t i = 0; i < m.can.size(); ++i) {
    if (o->vertices_canonical) {
      o->vertices_canonical[3 * i] = m.can[i].x; o->vertices_canonical[3 * i + 1] = m.can[i].y; o->vertices_canonical[3 * i + 2] = m.can[i].z;
    }
    if (o->vertices_deformed) {
      o->vertices_deformed[3 * i] = m.def[i].x; o->vertices_deformed[3 * i + 1] = m.def[i].y; o->vertices_deformed[3 * i + 2] = m.def[i].z;
    }
    if (o->normals_deformed && m.nrm.size() == m.can.size()) {
      o->normals_deformed[3 * i] = m.nrm[i].x; o->normals_deformed[3 * i + 1] = m.nrm[i].y; o->normals_deformed[3 * i + 2] = m.nrm[i].z;
    }
    if (o->colors) {
      o->colors[3 * i] = m.col[i].x; o->colors[3 * i + 1] = m.col[i].y; o->colors[3 * i + 2] = m.col[i].z;
    }
  }
  if (o->triangles)
    for (size_t t = 0; t < m.tri.size(); ++t)
      for (int k = 0; k < 3; ++k) o->triangles[3 * t + size_t(k)] = m.tri[t][size_t(k)];
}
int wfo_mesh_import(const wfk_mesh_view* in, wfo_mesh** out) {
  auto* mm = new wfo_mesh;
  Mesh& m = mm->m;
  const size_t nv = size_t(in->num_vertices), nt = size_t(in->num_triangles);
  m.can.resize(nv);
  m.def.resize(nv);
  m.col.resize(nv);
  for (size_t i = 0; i < nv; ++i) {
    m.can[i] = {in->vertices_canonical[3 * i], in->vertices_canonical[3 * i + 1], in->vertices_canonical[3 * i + 2]};
    m.def[i] = {in->vertices_deformed[3 * i], in->vertices_deformed[3 * i + 1], in->vertices_deformed[3 * i + 2]};
    if (in->colors) m.col[i] = {in->colors[3 * i], in->colors[3 * i + 1], in->colors[3 * i + 2]};
  }
  if (in->normals_deformed) {
    m.nrm.resize(nv);
    for (size_t i = 0; i < nv; ++i)
      m.nrm[i] = {in->normals_deformed[3 * i], in->normals_deformed[3 * i + 1], in->normals_deformed[3 * i + 2]};
  }
  m.tri.resize(nt);
  for (size_t t = 0; t < nt; ++t)
    m.tri[t] = {in->triangles[3 * t], in->triangles[3 * t + 1], in->triangles[3 * t + 2]};
  *out = mm;
  return WFK_OK;
}
int wfo_mesh_warp(wfo_mesh* mm, const wfk_volume_view* view, const wfk_pose* pose) {
  const Vol v = Vol::borrow(view);  // pipeline.cpp:167-169 (redeform)
  const Pose p = pose_of(pose);
  for (size_t i = 0; i < mm->m.can.size(); ++i) mm->m.def[i] = v.warp_point(p, mm->m.can[i]);
  return WFK_OK;
}
void wfo_compute_normals(wfo_mesh* m) { compute_normals(m->m); }
int wfo_rasterize(const wfo_mesh* m, const wfk_intrinsics* intr, int32_t exec, wfk_geometry_buffer* out) {
  if (!intr_valid(*intr)) return fail(WFK_E_INVALID_ARG, "rasterize: invalid intrinsics");
  GBuf b = gbuf_of(out);
  b.w = intr->width;
  b.h = intr->height;
  out->width = b.w;
  out->height = b.h;
  rasterize(m->m, *intr, exec != WFK_EXEC_SERIAL, b);
  return WFK_OK;
}
void wfo_mesh_free(wfo_mesh* m) { delete m; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Reconstructor::process_frame (pipeline.cpp:143-262), hot-path subset
// ---------------------------------------------------------------------------
struct wfo_recon {
  wfo_recon_config cfg;
  Vol vol;
  Pose pose;
  int frames = 0;
  std::vector<double> pt, nr, bp, bn, bc;
  std::vector<uint8_t> pv, nv;
  std::vector<float> bd;
  std::vector<wfk_feature> store;  // FeatureStore (features.hpp:79-95)
};

namespace {
// build_pyramid + detect_keypoints + extract_descriptors of the frame (pipeline.cpp:97-101)
std::vector<wfk_feature> detect_frame(const wfk_frame_view* frame, const wfk_feature_params& p) {
  std::vector<wfk_feature> out(4096);
  int32_t n = 0;
  int rc = wfo_detect_features(frame, &p, out.data(), int32_t(out.size()), &n, nullptr);
  if (rc == WFK_E_CAPACITY) {
    out.resize(size_t(n));
    rc = wfo_detect_features(frame, &p, out.data(), int32_t(out.size()), &n, nullptr);
  }
  out.resize(size_t(n));
  return out;
}

// Reconstructor::add_features (pipeline.cpp:95-141)
int add_features(wfo_recon* r, const wfk_frame_view* frame, const Maps& maps, int frame_index, const GBuf* buffer) {
  if (!frame->color) return 0;
  const Vol& vol = r->vol;
  auto features = detect_frame(frame, r->cfg.features);
  int added = 0;
  for (wfk_feature& f : features) {
    const int px = int(std::lround(f.pixel[0])), py = int(std::lround(f.pixel[1]));
    if (px < 0 || py < 0 || px >= maps.w || py >= maps.h) continue;
    const size_t idx = maps.idx(px, py);
    if (!maps.pv[idx]) continue;
    const V3 w = maps.P(idx);
    V3 can = w;  // bootstrap frame: the warp is the identity
    if (buffer) {
      V3 seed;
      bool have = false;
      for (int rr = 0; rr <= 4 && !have; ++rr)
        for (int dy = -rr; dy <= rr && !have; ++dy)
          for (int dx = -rr; dx <= rr && !have; ++dx) {
            const int sx = px + dx, sy = py + dy;
            if (sx < 0 || sy < 0 || sx >= buffer->w || sy >= buffer->h) continue;
            if (!std::isfinite(buffer->depth[buffer->idx(sx, sy)])) continue;
            seed = buffer->get(buffer->canonical, buffer->idx(sx, sy));
            have = true;
          }
      if (!have) continue;
      if (!invert_warp(vol, r->pose, w, seed, 20, 1e-6, can) || !vol.contains(can)) continue;
    }
    if (!vol.contains(can)) continue;
    f.world_pos[0] = w.x; f.world_pos[1] = w.y; f.world_pos[2] = w.z;
    f.canonical_pos[0] = can.x; f.canonical_pos[1] = can.y; f.canonical_pos[2] = can.z;
    f.frame_id = frame_index;
    r->store.push_back(f);
    ++added;
  }
  return added;
}

// the sparse term against the full history (pipeline.cpp:185-217)
std::vector<Con> feature_constraints(wfo_recon* r, const wfk_frame_view* frame, const Maps& maps, int* match_count) {
  const Vol& vol = r->vol;
  auto current = detect_frame(frame, r->cfg.features);
  for (wfk_feature& f : current) {
    const int px = int(std::lround(f.pixel[0])), py = int(std::lround(f.pixel[1]));
    V3 w{0, 0, -1};  // invalid, pruned by matching
    if (px >= 0 && py >= 0 && px < maps.w && py < maps.h && maps.pv[maps.idx(px, py)]) w = maps.P(maps.idx(px, py));
    f.world_pos[0] = w.x; f.world_pos[1] = w.y; f.world_pos[2] = w.z;
  }
  const size_t ns = r->store.size();
  std::vector<double> pred(3 * ns);
  for (size_t i = 0; i < ns; ++i) {
    const V3 c{r->store[i].canonical_pos[0], r->store[i].canonical_pos[1], r->store[i].canonical_pos[2]};
    const V3 p = vol.contains(c) ? vol.warp_point(r->pose, c) : V3{0, 0, -1};
    pred[3 * i] = p.x; pred[3 * i + 1] = p.y; pred[3 * i + 2] = p.z;
  }
  std::vector<wfk_feature_match> m(ns * 64 + 64);
  int32_t nm = 0;
  int rc = wfo_match_features(current.data(), int32_t(current.size()), r->store.data(), int32_t(ns), pred.data(),
                              &frame->intrinsics, &r->cfg.features, m.data(), int32_t(m.size()), &nm);
  if (rc == WFK_E_CAPACITY) {
    m.resize(size_t(nm));
    wfo_match_features(current.data(), int32_t(current.size()), r->store.data(), int32_t(ns), pred.data(),
                       &frame->intrinsics, &r->cfg.features, m.data(), int32_t(m.size()), &nm);
  }
  *match_count = nm;
  std::vector<Con> out;  // sparse_to_constraints (correspond.cpp:152-169)
  for (int i = 0; i < nm; ++i) {
    const wfk_feature& cf = current[size_t(m[size_t(i)].target_id)];
    if (cf.world_pos[2] <= 0) continue;
    const wfk_feature& sf = r->store[size_t(m[size_t(i)].source_id)];
    const V3 x{sf.canonical_pos[0], sf.canonical_pos[1], sf.canonical_pos[2]};
    if (!vol.contains(x)) continue;
    Con c;
    c.dense = false;
    c.canonical = x;
    vol.anchors(x, c.idx, c.w);
    c.target = {cf.world_pos[0], cf.world_pos[1], cf.world_pos[2]};
    c.normal = {0, 0, 0};
    c.conf = 1.0;
    out.push_back(c);
  }
  return out;
}
}  // namespace

extern "C" {

int wfo_recon_create(const wfo_recon_config* cfg, wfo_recon** out) {
  if (cfg->dims[0] < 2 || cfg->dims[1] < 2 || cfg->dims[2] < 2 || cfg->voxel_size <= 0)
    return fail(WFK_E_INVALID_ARG, "DeformableVolume: bad dims or voxel size");
  auto* r = new wfo_recon;
  r->cfg = *cfg;
  r->vol.make_owned(cfg->dims[0], cfg->dims[1], cfg->dims[2], cfg->voxel_size,
                    {cfg->origin[0], cfg->origin[1], cfg->origin[2]}, true);
  *out = r;
  return WFK_OK;
}
void wfo_recon_free(wfo_recon* r) { delete r; }
void wfo_recon_volume(wfo_recon* r, wfk_volume_view* o) {
  Vol& v = r->vol;
  o->dims[0] = v.nx; o->dims[1] = v.ny; o->dims[2] = v.nz;
  o->voxel_size = v.voxel;
  o->origin[0] = v.origin.x; o->origin[1] = v.origin.y; o->origin[2] = v.origin.z;
  o->truncation = v.mu;
  o->tsdf = v.tsdf_; o->weight = v.weight_; o->color = v.color_;
  o->deformed = v.deformed_; o->euler = v.euler_; o->age = v.age_; o->active = v.active_;
}

int wfo_recon_process_frame(wfo_recon* r, const wfk_frame_view* frame, const wfk_correspondence* sparse,
                            int64_t nsparse, wfo_frame_record* rec) {
  std::memset(rec, 0, sizeof(*rec));
  if (!intr_valid(frame->intrinsics)) return fail(WFK_E_INVALID_ARG, "frame has invalid intrinsics");
  const wfo_recon_config& cfg = r->cfg;
  Params sp = params_of(&cfg.solver);
  const bool par = sp.parallel;
  const FrameV f = frame_of(frame);
  const int W = f.w, H = f.h;
  const size_t npx = size_t(W) * size_t(H);
  r->pt.resize(3 * npx); r->nr.resize(3 * npx); r->pv.resize(npx); r->nv.resize(npx);
  Maps maps;
  maps.w = W; maps.h = H; maps.point = r->pt.data(); maps.normal = r->nr.data(); maps.pv = r->pv.data(); maps.nv = r->nv.data();
  backproject_depth(f, maps, par);
  Vol& vol = r->vol;
  if (r->frames == 0) {  // pipeline.cpp:150-159
    wfk_fusion_params boot = cfg.fusion;
    boot.bootstrap = 1;
    const FusionStats s = integrate_frame(vol, f, r->pose, boot, par);
    rec->fusion = {s.fused, s.gate, s.frustum, s.occluded};
    compute_active_set(vol);
    if (cfg.use_features) rec->features_added = add_features(r, frame, maps, r->frames, nullptr);  // :155
    pose_to_c(r->pose, &rec->pose);
    ++r->frames;
    return WFK_OK;
  }
  Mesh mesh = extract_mesh(vol, r->pose);  // pipeline.cpp:161-165
  if (mesh.tri.empty()) return fail(WFK_E_LOGIC, "empty isosurface");
  compute_normals(mesh);
  r->bd.resize(npx); r->bp.resize(3 * npx); r->bn.resize(3 * npx); r->bc.resize(3 * npx);
  GBuf buf;
  buf.w = W; buf.h = H; buf.depth = r->bd.data(); buf.point = r->bp.data(); buf.normal = r->bn.data(); buf.canonical = r->bc.data();
  rasterize(mesh, frame->intrinsics, par, buf);
  auto redeform = [&]() {  // pipeline.cpp:167-172
    for (size_t i = 0; i < mesh.can.size(); ++i) mesh.def[i] = vol.warp_point(r->pose, mesh.can[i]);
    compute_normals(mesh);
    rasterize(mesh, frame->intrinsics, par, buf);
  };
  if (cfg.estimate_pose) {  // pipeline.cpp:174-183
    wfk_icp_params ip = cfg.icp;
    ip.corr = cfg.correspond;
    const IcpOut icp = estimate_global_pose(buf, maps, frame->intrinsics, vol, r->pose, ip);
    rec->icp_degraded = icp.degraded;
    rec->icp_rms = icp.rms;
    rec->icp_iterations = icp.iterations;
    r->pose = icp.pose;
    redeform();
  }
  std::vector<Con> sparse_c;
  if (cfg.use_features && frame->color) sparse_c = feature_constraints(r, frame, maps, &rec->match_count);
  for (const Con& c : cons_of(sparse, nsparse)) sparse_c.push_back(c);
  auto all_active = [&](const Con& c) {
    for (int a : c.idx)
      if (!vol.active(a)) return false;
    return true;
  };
  try {
    for (int outer = 0; outer < cfg.reassociations; ++outer) {  // pipeline.cpp:226-247
      auto cons = find_dense(buf, maps, frame->intrinsics, cfg.correspond, vol);
      std::erase_if(cons, [&](const Con& c) { return !all_active(c); });
      rec->dense_count = int(cons.size());
      int kept = 0;
      for (const Con& c : sparse_c)
        if (all_active(c)) {
          cons.push_back(c);
          ++kept;
        }
      rec->sparse_count = kept;
      if (cons.empty()) break;
      const auto trace = solve_coarse_to_fine(vol, r->pose, cons, sp);
      for (const Trace& e : trace) {
        if (e.anomaly) ++rec->anomalies;
        rec->pcg_iterations += e.pcg_iterations;
        ++rec->trace_len;
      }
      if (!trace.empty()) fill_energy(trace.back().energy, &rec->energy);
      redeform();
    }
  } catch (const LogicError&) {
    return fail(WFK_E_LOGIC, "evaluate_energy: constraint anchors an inactive point");
  } catch (const InvalidArg&) {
    return fail(WFK_E_INVALID_ARG, "build_hierarchy: bad level count");
  } catch (const std::out_of_range&) {
    return fail(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  }
  for (int i = 0; i < vol.num_points(); ++i)  // pipeline.cpp:249-252
    if (vol.active(i)) vol.age_[i] += 1;
  const FusionStats s = integrate_frame(vol, f, r->pose, cfg.fusion, par);  // :254
  rec->fusion = {s.fused, s.gate, s.frustum, s.occluded};
  rec->expansion = expand_grid(vol);  // :255
  if (cfg.use_features) rec->features_added = add_features(r, frame, maps, r->frames, &buf);  // :257
  pose_to_c(r->pose, &rec->pose);
  ++r->frames;
  return WFK_OK;
}

int wfo_recon_feature_store(const wfo_recon* r, wfk_feature* out, int64_t cap, int64_t* n_out) {
  const int64_t n = int64_t(r->store.size());
  if (n_out) *n_out = n;
  if (!out) return WFK_OK;
  if (n > cap) return fail(WFK_E_CAPACITY, "feature buffer too small");
  std::copy(r->store.begin(), r->store.end(), out);
  return WFK_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// synthetic test-bed: SyntheticScene::render_frame (synthcam.cpp:252-316) for
// one sphere under the bend warp (synthcam.cpp:141-147, 164-201) with the Dots
// texture (synthcam.cpp:98-112).  Used only to make benchmark inputs for the
// CPU reference arm.
// ---------------------------------------------------------------------------
namespace {
M3 axis_unit(int axis, double ang) {
  M3 r = M3::identity();
  const double c = std::cos(ang), s = std::sin(ang);
  if (axis == 0) { r.a[1][1] = c; r.a[1][2] = -s; r.a[2][1] = s; r.a[2][2] = c; }
  else if (axis == 1) { r.a[0][0] = c; r.a[0][2] = s; r.a[2][0] = -s; r.a[2][2] = c; }
  else { r.a[0][0] = c; r.a[0][1] = -s; r.a[1][0] = s; r.a[1][1] = c; }
  return r;
}
uint64_t smix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t hcell(int64_t x, int64_t y, int64_t z, uint32_t seed) {
  uint64_t h = seed;
  h = smix(h ^ uint64_t(x));
  h = smix(h ^ uint64_t(y));
  h = smix(h ^ uint64_t(z));
  return h;
}
double r01(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }
}  // namespace

extern "C" int wfo_synth_render(const double center[3], double radius, const double pivot[3], double amplitude,
                                int driver_axis, int rot_axis, uint32_t tex_seed, double tex_scale,
                                double dot_radius, const wfk_intrinsics* K, float* depth, float* color) {
  const V3 c0{center[0], center[1], center[2]}, pv{pivot[0], pivot[1], pivot[2]};
  auto inverse_warp = [&](const V3& world) {
    if (amplitude == 0) return world;
    const V3 p = world - pv;
    auto g = [&](double s) { return (transpose(axis_unit(rot_axis, amplitude * s)) * p)[driver_axis] - s; };
    double s = p[driver_axis];
    bool ok = false;
    for (int it = 0; it < 50; ++it) {
      const double gs = g(s);
      if (std::abs(gs) < 1e-12) { ok = true; break; }
      const double h = 1e-7;
      const double dg = (g(s + h) - g(s - h)) / (2 * h);
      if (std::abs(dg) < 1e-12) break;
      s -= gs / dg;
    }
    if (!ok && std::abs(g(s)) > 1e-10) {
      double lo = -(norm(p) + 1), hi = norm(p) + 1;
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (g(lo) * g(mid) <= 0) hi = mid; else lo = mid;
      }
      s = 0.5 * (lo + hi);
    }
    return pv + axis_unit(rot_axis, -amplitude * s) * p;
  };
  const int W = K->width, H = K->height;
#pragma omp parallel for schedule(dynamic, 4)
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      const size_t i = size_t(y) * size_t(W) + size_t(x);
      depth[i] = 0.f;
      color[3 * i] = color[3 * i + 1] = color[3 * i + 2] = 0.f;
      const V3 dir = normalized(V3{(double(x) - K->cx) / K->fx, (double(y) - K->cy) / K->fy, 1.0});
      auto field = [&](double t) { return norm(inverse_warp(t * dir) - c0) - radius; };
      double t = 0.05, f = field(t);
      if (f <= 0) continue;
      double hit = -1;
      for (int it = 0; it < 2000 && t < 6.0; ++it) {
        const double step = std::clamp(0.7 * f, 5e-5, 0.25);
        const double tn = t + step;
        const double fn = field(tn);
        if (fn <= 1e-7) {
          if (fn < 0) {
            double lo = t, hi = tn;
            for (int b = 0; b < 60; ++b) {
              const double mid = 0.5 * (lo + hi);
              if (field(mid) > 0) lo = mid; else hi = mid;
            }
            hit = 0.5 * (lo + hi);
          } else {
            hit = tn;
          }
          break;
        }
        t = tn;
        f = fn;
      }
      if (hit < 0) continue;
      const V3 pc = hit * dir;
      depth[i] = float(pc.z);
      const V3 can = inverse_warp(pc);
      const V3 cell = can / tex_scale;
      const V3 fl{std::floor(cell.x), std::floor(cell.y), std::floor(cell.z)};
      const uint64_t h = hcell(int64_t(fl.x), int64_t(fl.y), int64_t(fl.z), tex_seed);
      const double margin = dot_radius + 0.05;
      const V3 jit{margin + r01(h) * (1 - 2 * margin), margin + r01(smix(h)) * (1 - 2 * margin),
                   margin + r01(smix(smix(h))) * (1 - 2 * margin)};
      if (norm(cell - (fl + jit)) < dot_radius) {
        const uint64_t hc = smix(h ^ 0xd0d5u);
        color[3 * i] = 20 + 160 * float(r01(hc));
        color[3 * i + 1] = 20 + 160 * float(r01(smix(hc)));
        color[3 * i + 2] = 20 + 160 * float(r01(smix(smix(hc))));
      } else {
        color[3 * i] = color[3 * i + 1] = color[3 * i + 2] = 210.f;
      }
    }
  return WFK_OK;
}
