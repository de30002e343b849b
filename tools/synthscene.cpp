// Synthetic RGB-D input generator (bench / test infrastructure, not the
// product): restates SyntheticScene (proj/src/synthcam.cpp) with the same
// operation order the reference's Eigen expressions evaluate in (products
// and dots accumulated left to right, x / s as a division, AngleAxis /
// normalized as Eigen 3.4 computes them), so the frames are bit-identical to
// the reference's renderer (tests/test_synthscene.py).
#include "synthscene.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>

namespace {

struct V3 {
  double x = 0, y = 0, z = 0;
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(double s, const V3& a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator*(const V3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 operator/(const V3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double norm(const V3& a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(const V3& a) {  // Eigen: x / sqrt(squaredNorm), zero stays
  const double n = dot(a, a);
  return n == 0 ? a : a / std::sqrt(n);
}
V3 v3(const double* p) { return {p[0], p[1], p[2]}; }

struct M3 {
  double a[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
};
inline V3 mul(const M3& m, const V3& v) {  // rows accumulated left to right
  return {m.a[0][0] * v.x + m.a[0][1] * v.y + m.a[0][2] * v.z, m.a[1][0] * v.x + m.a[1][1] * v.y + m.a[1][2] * v.z,
          m.a[2][0] * v.x + m.a[2][1] * v.y + m.a[2][2] * v.z};
}
inline V3 mul_t(const M3& m, const V3& v) {  // m^T v
  return {m.a[0][0] * v.x + m.a[1][0] * v.y + m.a[2][0] * v.z, m.a[0][1] * v.x + m.a[1][1] * v.y + m.a[2][1] * v.z,
          m.a[0][2] * v.x + m.a[1][2] * v.y + m.a[2][2] * v.z};
}

// Eigen::AngleAxisd(rad, n).toRotationMatrix()
M3 angle_axis(double rad, const V3& n) {
  M3 r;
  const V3 sin_axis = std::sin(rad) * n;
  const double c = std::cos(rad);
  const V3 cos1_axis = (1.0 - c) * n;
  double tmp;
  tmp = cos1_axis.x * n.y;
  r.a[0][1] = tmp - sin_axis.z;
  r.a[1][0] = tmp + sin_axis.z;
  tmp = cos1_axis.x * n.z;
  r.a[0][2] = tmp + sin_axis.y;
  r.a[2][0] = tmp - sin_axis.y;
  tmp = cos1_axis.y * n.z;
  r.a[1][2] = tmp - sin_axis.x;
  r.a[2][1] = tmp + sin_axis.x;
  r.a[0][0] = cos1_axis.x * n.x + c;
  r.a[1][1] = cos1_axis.y * n.y + c;
  r.a[2][2] = cos1_axis.z * n.z + c;
  return r;
}
// synthcam.cpp:18-22
M3 axis_angle(const V3& axis, double rad) {
  const double n = norm(axis);
  if (n < 1e-12) return M3{};
  return angle_axis(rad, axis / n);
}
V3 unit_axis(int i) {
  V3 e;
  e[i] = 1;
  return e;
}
inline double deg2rad(double d) { return d * M_PI / 180.0; }

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t hash_cell(int64_t x, int64_t y, int64_t z, uint32_t seed) {
  uint64_t h = seed;
  h = splitmix64(h ^ uint64_t(x));
  h = splitmix64(h ^ uint64_t(y));
  h = splitmix64(h ^ uint64_t(z));
  return h;
}
double rand01(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }
double smoothstep(double t) { return t * t * (3 - 2 * t); }

// synthcam.cpp:49-65
double value_noise(const V3& p, uint32_t seed) {
  const V3 f{std::floor(p.x), std::floor(p.y), std::floor(p.z)};
  const int64_t ix = int64_t(f.x), iy = int64_t(f.y), iz = int64_t(f.z);
  const double tx = smoothstep(p.x - f.x), ty = smoothstep(p.y - f.y), tz = smoothstep(p.z - f.z);
  double acc = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double v = rand01(hash_cell(ix + dx, iy + dy, iz + dz, seed));
        acc += v * (dx ? tx : 1 - tx) * (dy ? ty : 1 - ty) * (dz ? tz : 1 - tz);
      }
  return acc;
}

// synthcam.cpp:69-90
double shape_sdf(const ss_shape& s, const V3& p) {
  switch (s.type) {
    case SS_SPHERE:
      return norm(p - v3(s.center)) - s.radius;
    case SS_BOX: {
      const V3 d = p - v3(s.center);
      const V3 q = V3{std::abs(d.x), std::abs(d.y), std::abs(d.z)} - v3(s.half_extents);
      const V3 qm{q.x < 0.0 ? 0.0 : q.x, q.y < 0.0 ? 0.0 : q.y, q.z < 0.0 ? 0.0 : q.z};  // cwiseMax(0)
      const double outside = norm(qm);
      double mx = q.x;  // maxCoeff
      if (q.y > mx) mx = q.y;
      if (q.z > mx) mx = q.z;
      const double inside = std::min(mx, 0.0);
      return outside + inside;
    }
    case SS_PLANE:
      return dot(normalized(v3(s.normal)), p) - s.offset;
    case SS_CYLINDER: {
      const V3 a = normalized(v3(s.axis));
      const V3 rel = p - v3(s.center);
      const double y = dot(rel, a);
      const double r = norm(rel - y * a);
      const double d0 = r - s.radius, d1 = std::abs(y) - s.half_height;
      const double mx = d1 > d0 ? d1 : d0;
      const double m0 = d0 < 0.0 ? 0.0 : d0, m1 = d1 < 0.0 ? 0.0 : d1;
      return std::min(mx, 0.0) + std::sqrt(m0 * m0 + m1 * m1);
    }
  }
  return 0;
}

// synthcam.cpp:92-123
void texture_color(const ss_scene& s, const V3& canonical, float out[3]) {
  const V3 cell = canonical / s.tex_scale;
  switch (s.tex_type) {
    case SS_CHECKER: {
      const int64_t k = int64_t(std::floor(cell.x)) + int64_t(std::floor(cell.y)) + int64_t(std::floor(cell.z));
      out[0] = out[1] = out[2] = (k & 1) ? 45.f : 235.f;
      return;
    }
    case SS_NOISE: {
      const float v = float(value_noise(cell, s.tex_seed));
      out[0] = out[1] = out[2] = 40 + 180 * v;
      return;
    }
    case SS_DOTS: {
      const V3 f{std::floor(cell.x), std::floor(cell.y), std::floor(cell.z)};
      const uint64_t h = hash_cell(int64_t(f.x), int64_t(f.y), int64_t(f.z), s.tex_seed);
      const double margin = s.dot_radius + 0.05;
      const V3 jitter{margin + rand01(h) * (1 - 2 * margin), margin + rand01(splitmix64(h)) * (1 - 2 * margin),
                      margin + rand01(splitmix64(splitmix64(h))) * (1 - 2 * margin)};
      const V3 center = f + jitter;
      if (norm(cell - center) < s.dot_radius) {
        const uint64_t hc = splitmix64(h ^ 0xd0d5u);
        out[0] = 20 + 160 * float(rand01(hc));
        out[1] = 20 + 160 * float(rand01(splitmix64(hc)));
        out[2] = 20 + 160 * float(rand01(splitmix64(splitmix64(hc))));
        return;
      }
      out[0] = out[1] = out[2] = 210.f;
      return;
    }
  }
  out[0] = out[1] = out[2] = 0.f;
}

double scene_sdf(const ss_scene& s, const V3& p) {  // synthcam.cpp:132-136
  double d = std::numeric_limits<double>::infinity();
  for (int i = 0; i < s.num_shapes; ++i) d = std::min(d, shape_sdf(s.shapes[i], p));
  return d;
}

double warp_phase(const ss_scene& s, int frame) {  // synthcam.cpp:138-143
  if (s.frequency > 0) return std::sin(2 * M_PI * s.frequency * frame / s.frames);
  return s.frames > 1 ? double(frame) / (s.frames - 1) : 0.0;
}

// synthcam.cpp:167-216
V3 inverse_warp(const ss_scene& s, int frame, const V3& world) {
  const V3 pv = v3(s.pivot);
  switch (s.warp_type) {
    case SS_WARP_NONE:
      return world;
    case SS_WARP_RIGID: {
      const M3 r = axis_angle(v3(s.rotation_axis), deg2rad(s.deg_per_frame) * frame);
      return pv + mul_t(r, world - v3(s.trans_per_frame) * double(frame) - pv);
    }
    case SS_WARP_TWIST: {
      const double rate = s.amplitude * warp_phase(s, frame);
      const V3 p = world - pv;
      const double theta = rate * p[s.driver_axis];
      return pv + mul(axis_angle(unit_axis(s.driver_axis), -theta), p);
    }
    case SS_WARP_BEND: {
      const double a = s.amplitude * warp_phase(s, frame);
      const V3 p = world - pv;
      const V3 e = unit_axis(s.rot_axis);
      auto g = [&](double t) { return mul_t(axis_angle(e, a * t), p)[s.driver_axis] - t; };
      double t = p[s.driver_axis];
      bool ok = false;
      for (int it = 0; it < 50; ++it) {
        const double gs = g(t);
        if (std::abs(gs) < 1e-12) {
          ok = true;
          break;
        }
        const double h = 1e-7;
        const double dg = (g(t + h) - g(t - h)) / (2 * h);
        if (std::abs(dg) < 1e-12) break;
        t -= gs / dg;
      }
      if (!ok && std::abs(g(t)) > 1e-10) {
        double lo = -(norm(p) + 1), hi = norm(p) + 1;
        for (int it = 0; it < 200; ++it) {
          const double mid = 0.5 * (lo + hi);
          if (g(lo) * g(mid) <= 0)
            hi = mid;
          else
            lo = mid;
        }
        t = 0.5 * (lo + hi);
      }
      return pv + mul(axis_angle(e, -a * t), p);
    }
  }
  return world;
}

}  // namespace

extern "C" {

double ss_warp_phase(const ss_scene* s, int32_t frame) { return warp_phase(*s, frame); }

void ss_inverse_warp(const ss_scene* s, int32_t frame, const double world[3], double canonical[3]) {
  const V3 c = inverse_warp(*s, frame, v3(world));
  canonical[0] = c.x;
  canonical[1] = c.y;
  canonical[2] = c.z;
}

// SyntheticScene::render_frame (synthcam.cpp:252-316)
int ss_render(const ss_scene* sp, int32_t frame, float* depth, float* color, int32_t threads) {
  const ss_scene& s = *sp;
  if (s.num_shapes < 1 || s.num_shapes > SS_MAX_SHAPES || s.frames < 1 || !(s.fx > 0 && s.fy > 0) || s.width <= 0 ||
      s.height <= 0)
    return -1;
  const int w = s.width, h = s.height;
  const M3 cam_r = axis_angle(v3(s.cam_rot_axis), deg2rad(s.cam_deg_per_frame) * frame);  // camera_pose
  const V3 cam_t = v3(s.cam_trans_per_frame) * double(frame);
  auto to_canonical = [&](const V3& p_cam) { return inverse_warp(s, frame, mul_t(cam_r, p_cam - cam_t)); };
  auto field = [&](const V3& p_cam) { return scene_sdf(s, to_canonical(p_cam)); };
  auto render_row = [&](int y) {
    for (int x = 0; x < w; ++x) {
      const size_t i = size_t(y) * size_t(w) + size_t(x);
      depth[i] = 0.f;
      color[3 * i] = color[3 * i + 1] = color[3 * i + 2] = 0.f;
      const V3 dir = normalized(V3{(x - s.cx) / s.fx * 1.0, (y - s.cy) / s.fy * 1.0, 1.0});  // backproject(x, y, 1)
      double t = s.t_min;
      double f = field(t * dir);
      if (f <= 0) continue;
      double hit = -1;
      for (int it = 0; it < 2000 && t < s.t_max; ++it) {
        const double step = std::clamp(0.7 * f, 5e-5, 0.25);
        const double tn = t + step;
        const double fn = field(tn * dir);
        if (fn <= 1e-7) {
          if (fn < 0) {
            double lo = t, hi = tn;
            for (int b = 0; b < 60; ++b) {
              const double mid = 0.5 * (lo + hi);
              if (field(mid * dir) > 0)
                lo = mid;
              else
                hi = mid;
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
      const V3 p_cam = hit * dir;
      depth[i] = float(p_cam.z);
      texture_color(s, to_canonical(p_cam), color + 3 * i);
    }
  };
  const int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4) num_threads(nt)
  for (int y = 0; y < h; ++y) render_row(y);
  if (s.noise_sigma > 0) {
    std::mt19937 rng(s.noise_seed ^ (uint32_t(frame) * 2654435761u));
    std::normal_distribution<double> gauss(0.0, s.noise_sigma);
    for (size_t i = 0; i < size_t(w) * size_t(h); ++i)
      if (depth[i] > 0) depth[i] = float(std::max(1e-3, double(depth[i]) + gauss(rng)));
  }
  return 0;
}

}  // extern "C"
