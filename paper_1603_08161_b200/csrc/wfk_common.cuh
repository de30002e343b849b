// Shared device helpers for libwfk (sm_100a).
//
// All kernels are compiled with -fmad=false: every fp64 multiply and add is
// rounded separately, in the reference's operation order, so integer decisions
// derived from floating-point geometry (cell indices, coverage, gates,
// selection) come out bit-identical to the CPU reference (SURVEY.md 7 "Hard
// parts" 1).  Only sin/cos/atan2/asin differ from glibc in the last ulp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>

#define WF_HD __host__ __device__ __forceinline__
#define WF_D __device__ __forceinline__

namespace wfk {

constexpr int kBlock = 256;
constexpr int kCoopBlock = 512;     // persistent cooperative kernels: 1 block / SM
constexpr int kCoopBlockShared = 384;  // the flip-flop kernel with its row state in shared memory
constexpr int kAssembleRatio = 32; // incidences per row above which B^T B is assembled
#ifndef WFK_ASM_LANES
#define WFK_ASM_LANES 8
#endif
constexpr int kAsmLanes = WFK_ASM_LANES;  // lanes per row on small assembled levels (27 stencil slots)
constexpr int kAsmThreadRows = 16384;  // rows from which assembled levels put one row per lane
#ifndef WFK_MF_LANES
#define WFK_MF_LANES 2
#endif
constexpr int kMfLanes = WFK_MF_LANES;  // lanes per row of the matrix-free row pass (pipelined PCG)
constexpr int kItemLen = 8;         // incidences per work item of the matrix-free row pass
constexpr int kCacheWarpRow = 32;   // incidences above which the constraint cache sums a row by warp
constexpr int kCenter = 13;

struct V3 {
  double x, y, z;
};
WF_HD V3 mk(double x, double y, double z) { return V3{x, y, z}; }
WF_HD V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
WF_HD V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
WF_HD V3 operator-(V3 a) { return {-a.x, -a.y, -a.z}; }
WF_HD V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
WF_HD V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
WF_HD V3 operator/(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
WF_HD V3& operator+=(V3& a, V3 b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
WF_HD V3& operator-=(V3& a, V3 b) { a.x -= b.x; a.y -= b.y; a.z -= b.z; return a; }
WF_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
WF_HD double sqnorm(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
WF_HD double norm3(V3 a) { return sqrt(sqnorm(a)); }
WF_HD V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
WF_HD V3 cmul(V3 a, V3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
WF_HD double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

WF_HD V3 ld3(const double* p, int64_t i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
WF_HD void st3(double* p, int64_t i, V3 v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}

struct M3 {
  double a[3][3];
};
WF_HD M3 m3_zero() {
  M3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m.a[i][j] = 0.0;
  return m;
}
WF_HD M3 m3_identity() {
  M3 m = m3_zero();
  m.a[0][0] = m.a[1][1] = m.a[2][2] = 1.0;
  return m;
}
WF_HD M3 mul(const M3& p, const M3& q) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      r.a[i][j] = p.a[i][0] * q.a[0][j] + p.a[i][1] * q.a[1][j] + p.a[i][2] * q.a[2][j];
  return r;
}
WF_HD V3 mul(const M3& m, V3 v) {
  return {m.a[0][0] * v.x + m.a[0][1] * v.y + m.a[0][2] * v.z,
          m.a[1][0] * v.x + m.a[1][1] * v.y + m.a[1][2] * v.z,
          m.a[2][0] * v.x + m.a[2][1] * v.y + m.a[2][2] * v.z};
}
WF_HD M3 add(const M3& p, const M3& q) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = p.a[i][j] + q.a[i][j];
  return r;
}
WF_HD M3 transpose(const M3& m) {
  M3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.a[i][j] = m.a[j][i];
  return r;
}
WF_HD double det(const M3& m) {  // Eigen determinant_impl<3>
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}
WF_HD M3 ld_m3(const double* p, int64_t i) {
  M3 m;
  for (int k = 0; k < 9; ++k) m.a[k / 3][k % 3] = p[9 * i + k];
  return m;
}
WF_HD void st_m3(double* p, int64_t i, const M3& m) {
  for (int k = 0; k < 9; ++k) p[9 * i + k] = m.a[k / 3][k % 3];
}

// core.cpp:7-14  R = Rz(c) * Ry(b) * Rx(a)
WF_HD M3 euler_to_matrix(V3 abc) {
  const double a = abc.x, b = abc.y, c = abc.z;
  M3 rx, ry, rz;
  rx.a[0][0] = 1; rx.a[0][1] = 0; rx.a[0][2] = 0;
  rx.a[1][0] = 0; rx.a[1][1] = cos(a); rx.a[1][2] = -sin(a);
  rx.a[2][0] = 0; rx.a[2][1] = sin(a); rx.a[2][2] = cos(a);
  ry.a[0][0] = cos(b); ry.a[0][1] = 0; ry.a[0][2] = sin(b);
  ry.a[1][0] = 0; ry.a[1][1] = 1; ry.a[1][2] = 0;
  ry.a[2][0] = -sin(b); ry.a[2][1] = 0; ry.a[2][2] = cos(b);
  rz.a[0][0] = cos(c); rz.a[0][1] = -sin(c); rz.a[0][2] = 0;
  rz.a[1][0] = sin(c); rz.a[1][1] = cos(c); rz.a[1][2] = 0;
  rz.a[2][0] = 0; rz.a[2][1] = 0; rz.a[2][2] = 1;
  return mul(mul(rz, ry), rx);
}

WF_HD double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
WF_HD int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
WF_HD float clampf(float v, float lo, float hi) { return v < lo ? lo : (v > hi ? hi : v); }

// core.cpp:16-29
WF_HD V3 matrix_to_euler(const M3& r) {
  const double b = asin(clampd(-r.a[2][0], -1.0, 1.0));
  double a, c;
  if (fabs(r.a[2][0]) < 1.0 - 1e-12) {
    a = atan2(r.a[2][1], r.a[2][2]);
    c = atan2(r.a[1][0], r.a[0][0]);
  } else {
    a = atan2(-r.a[1][2], r.a[1][1]);
    c = 0.0;
  }
  return {a, b, c};
}

// --- Eigen 3.4 JacobiSVD<Matrix3d> (ComputeFullU|ComputeFullV), restated ----
struct Rot {
  double c, s;
};
WF_HD Rot rot_t(Rot j) { return {j.c, -j.s}; }
WF_HD Rot rot_mul(Rot a, Rot b) { return {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c}; }
WF_HD void rot_rows(M3& m, int p, int q, Rot j) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double xi = m.a[p][i], yi = m.a[q][i];
    m.a[p][i] = j.c * xi + j.s * yi;
    m.a[q][i] = -j.s * xi + j.c * yi;
  }
}
WF_HD void rot_cols(M3& m, int p, int q, Rot j) {
  const Rot t = rot_t(j);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double xi = m.a[i][p], yi = m.a[i][q];
    m.a[i][p] = t.c * xi + t.s * yi;
    m.a[i][q] = -t.s * xi + t.c * yi;
  }
}
WF_HD Rot make_jacobi(double x, double y, double z) {
  Rot r{1.0, 0.0};
  const double deno = 2.0 * fabs(y);
  if (deno < DBL_MIN) return r;
  const double tau = (x - z) / deno;
  const double w = sqrt(tau * tau + 1.0);
  const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0 ? 1.0 : -1.0;
  const double n = 1.0 / sqrt(t * t + 1.0);
  r.s = -sign_t * (y / fabs(y)) * fabs(t) * n;
  r.c = n;
  return r;
}
WF_HD void svd3(const M3& a, M3& u, double sv[3], M3& v) {
  double scale = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) scale = fmax(scale, fabs(a.a[i][j]));
  u = m3_identity();
  v = m3_identity();
  if (!isfinite(scale)) {
    sv[0] = sv[1] = sv[2] = 0;
    return;
  }
  if (scale == 0) scale = 1;
  M3 w;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) w.a[i][j] = a.a[i][j] / scale;
  const double considerAsZero = DBL_MIN;
  const double precision = 2.0 * DBL_EPSILON;
  double maxDiag = fmax(fabs(w.a[0][0]), fmax(fabs(w.a[1][1]), fabs(w.a[2][2])));
  bool finished = false;
  int sweeps = 0;
  while (!finished && sweeps < 64) {
    finished = true;
    ++sweeps;
    // fully unrolled (p, q) pairs: the 3x3 matrices stay in registers
#pragma unroll
    for (int p = 1; p < 3; ++p)
#pragma unroll
      for (int q = 0; q < p; ++q) {
        const double threshold = fmax(considerAsZero, precision * maxDiag);
        if (fabs(w.a[p][q]) > threshold || fabs(w.a[q][p]) > threshold) {
          finished = false;
          const double m00 = w.a[p][p], m01 = w.a[p][q], m10 = w.a[q][p], m11 = w.a[q][q];
          Rot rot1;
          const double t = m00 + m11;
          const double d = m10 - m01;
          if (fabs(d) < DBL_MIN) {
            rot1.s = 0;
            rot1.c = 1;
          } else {
            const double uu = t / d;
            const double tmp = sqrt(1.0 + uu * uu);
            rot1.s = 1.0 / tmp;
            rot1.c = uu / tmp;
          }
          const double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
          const double n11 = -rot1.s * m01 + rot1.c * m11;
          const Rot jr = make_jacobi(n00, n01, n11);
          const Rot jl = rot_mul(rot1, rot_t(jr));
          rot_rows(w, p, q, jl);
          rot_cols(u, p, q, rot_t(jl));
          rot_cols(w, p, q, jr);
          rot_cols(v, p, q, jr);
          maxDiag = fmax(maxDiag, fmax(fabs(w.a[p][p]), fabs(w.a[q][q])));
        }
      }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double d = w.a[i][i];
    sv[i] = fabs(d);
    if (d < 0)
#pragma unroll
      for (int k = 0; k < 3; ++k) u.a[k][i] = -u.a[k][i];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) sv[i] *= scale;
  // selection sort by decreasing singular value; the swap with the chosen
  // column is spelled out per candidate so no index is dynamic
  bool stop = false;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (stop) continue;
    int pos = i;
    double best = sv[i];
#pragma unroll
    for (int k = i + 1; k < 3; ++k)
      if (sv[k] > best) {
        best = sv[k];
        pos = k;
      }
    if (best == 0) {
      stop = true;
      continue;
    }
#pragma unroll
    for (int k = i + 1; k < 3; ++k)
      if (pos == k) {
        double t = sv[i]; sv[i] = sv[k]; sv[k] = t;
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          t = u.a[m][i]; u.a[m][i] = u.a[m][k]; u.a[m][k] = t;
          t = v.a[m][i]; v.a[m][i] = v.a[m][k]; v.a[m][k] = t;
        }
      }
  }
}

// --- lattice geometry (volume.hpp:40-55, volume.cpp:27-66) -------------------
struct Grid {
  int nx, ny, nz;
  double voxel;
  double ox, oy, oz;
  WF_HD int64_t n() const { return int64_t(nx) * ny * nz; }
  WF_HD int lin(int x, int y, int z) const { return x + nx * (y + ny * z); }
  WF_HD void idx3(int i, int& x, int& y, int& z) const {
    x = i % nx;
    y = (i / nx) % ny;
    z = i / (nx * ny);
  }
  WF_HD bool in_grid(int x, int y, int z) const {
    return x >= 0 && y >= 0 && z >= 0 && x < nx && y < ny && z < nz;
  }
  WF_HD V3 canonical(int i) const {
    int x, y, z;
    idx3(i, x, y, z);
    return {ox + voxel * double(x), oy + voxel * double(y), oz + voxel * double(z)};
  }
  WF_HD V3 origin() const { return {ox, oy, oz}; }
  WF_HD int dim(int k) const { return k == 0 ? nx : (k == 1 ? ny : nz); }
  WF_HD double org(int k) const { return k == 0 ? ox : (k == 1 ? oy : oz); }
  // volume.cpp:27-33
  WF_HD bool contains(V3 x) const {
    const double eps = 1e-9;
    const V3 rel = (x - origin()) / voxel;
    if (!(rel.x >= -eps) || !(rel.y >= -eps) || !(rel.z >= -eps)) return false;
    if (!(rel.x <= (double(nx) - 1.0) + eps)) return false;
    if (!(rel.y <= (double(ny) - 1.0) + eps)) return false;
    if (!(rel.z <= (double(nz) - 1.0) + eps)) return false;
    return true;
  }
  // volume.cpp:35-59 (caller guarantees contains())
  WF_HD void anchors(V3 x, int idx[8], double w[8]) const {
    const V3 rel = (x - origin()) / voxel;
    int cell[3];
    double frac[3];
    for (int k = 0; k < 3; ++k) {
      const double rk = comp(rel, k);
      int c = static_cast<int>(floor(rk));
      c = clampi(c, 0, dim(k) - 2);
      cell[k] = c;
      frac[k] = clampd(rk - c, 0.0, 1.0);
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
  WF_HD V3 interpolate(const double* deformed, V3 x) const {
    int idx[8];
    double w[8];
    anchors(x, idx, w);
    V3 p{0, 0, 0};
    for (int k = 0; k < 8; ++k) p += w[k] * ld3(deformed, idx[k]);
    return p;
  }
};

__device__ __constant__ static const int kFace[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0},
                                                        {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};

WF_HD int stencil_slot(int dx, int dy, int dz) { return (dz + 1) * 9 + (dy + 1) * 3 + (dx + 1); }

struct PoseD {
  M3 r;
  V3 t;
  WF_HD V3 apply(V3 x) const { return mul(r, x) + t; }  // core.hpp:24
};

// --- deterministic reductions ------------------------------------------------
WF_D double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NV values; result valid in every thread.  Fixed tree
// order, so the result is reproducible run to run.
template <int NV>
WF_D void block_sum(double (&v)[NV], double* smem /* >= NV * 32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[k * 32 + warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = lane < nw ? smem[k * 32 + lane] : 0.0;
    v[k] = warp_sum(s);
  }
  __syncthreads();
}

// Sum of partials[b] over b < nblocks (<= 512), fixed order; every lane of the
// calling warp gets the result.  All loads are issued before the adds.
constexpr int kMaxCoopBlocks = 512;
WF_D double sum_partials(const double* partials, int nblocks) {
  const int lane = threadIdx.x & 31;
  double v[kMaxCoopBlocks / 32];
#pragma unroll
  for (int j = 0; j < kMaxCoopBlocks / 32; ++j) {
    const int b = lane + 32 * j;
    v[j] = b < nblocks ? __ldcg(partials + b) : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < kMaxCoopBlocks / 32; ++j) s += v[j];
  return warp_sum(s);
}

}  // namespace wfk
