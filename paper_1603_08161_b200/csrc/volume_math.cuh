// DeformableVolume::invert_warp (volume.cpp:68-126) as device functions,
// shared by the batched entry point (fusion.cu) and the feature lift
// (features.cu, pipeline.cpp:112-130).
#pragma once
#include "wfk_common.cuh"

namespace wfk {

// deformed_jacobian (volume.cpp:68-93)
WF_D M3 deformed_jacobian(const Grid& g, const double* deformed, V3 x) {
  const double rel[3] = {(x.x - g.ox) / g.voxel, (x.y - g.oy) / g.voxel, (x.z - g.oz) / g.voxel};
  const int d[3] = {g.nx, g.ny, g.nz};
  int cell[3];
  double f[3];
  for (int k = 0; k < 3; ++k) {
    int c = int(floor(rel[k]));
    c = min(max(c, 0), d[k] - 2);
    cell[k] = c;
    f[k] = rel[k] - c;
  }
  M3 j = m3_zero();
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const V3 t = ld3(deformed, g.lin(cell[0] + dx, cell[1] + dy, cell[2] + dz));
        const double wx = dx ? f[0] : 1 - f[0];
        const double wy = dy ? f[1] : 1 - f[1];
        const double wz = dz ? f[2] : 1 - f[2];
        const double gr[3] = {(dx ? 1.0 : -1.0) * wy * wz, (dy ? 1.0 : -1.0) * wx * wz,
                              (dz ? 1.0 : -1.0) * wx * wy};
        for (int c = 0; c < 3; ++c) {
          j.a[0][c] += t.x * gr[c];
          j.a[1][c] += t.y * gr[c];
          j.a[2][c] += t.z * gr[c];
        }
      }
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) j.a[r][c] = j.a[r][c] / g.voxel;
  return j;
}
// Eigen PartialPivLU<Matrix3d>::solve, restated as in the oracle
WF_D V3 lu3_solve(M3 a, V3 b) {
  int perm[3] = {0, 1, 2};
  for (int k = 0; k < 3; ++k) {
    int p = k;
    for (int i = k + 1; i < 3; ++i)
      if (fabs(a.a[i][k]) > fabs(a.a[p][k])) p = i;
    if (a.a[p][k] != 0) {
      if (p != k) {
        for (int c = 0; c < 3; ++c) {
          const double t = a.a[k][c];
          a.a[k][c] = a.a[p][c];
          a.a[p][c] = t;
        }
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
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
// invert_warp of one point: canonical x with warp_point(pose, x) == y from seed
WF_D bool invert_warp_point(const Grid& g, const double* deformed, const PoseD& pose, V3 y, V3 seed, int max_iters,
                            double tol, V3& out) {
  const V3 target = mul(transpose(pose.r), y - pose.t);  // apply_inverse (core.hpp:25-27)
  V3 x = seed;
  out = V3{0, 0, 0};
  if (!g.contains(x)) return false;
  const double lo[3] = {g.ox, g.oy, g.oz};
  const double hi[3] = {g.ox + g.voxel * (g.nx - 1), g.oy + g.voxel * (g.ny - 1), g.oz + g.voxel * (g.nz - 1)};
  for (int it = 0; it < max_iters; ++it) {
    const V3 r = g.interpolate(deformed, x) - target;
    if (norm3(r) <= tol) {
      out = x;
      return true;
    }
    const M3 j = deformed_jacobian(g, deformed, x);
    V3 step = fabs(det(j)) > 1e-12 ? lu3_solve(j, r) : r;  // damped fixed-point fallback
    const double max_step = g.voxel;
    if (norm3(step) > max_step) step = step * (max_step / norm3(step));
    const V3 xn = x - step;
    x = V3{fmin(fmax(xn.x, lo[0]), hi[0]), fmin(fmax(xn.y, lo[1]), hi[1]), fmin(fmax(xn.z, lo[2]), hi[2])};
  }
  if (norm3(g.interpolate(deformed, x) - target) <= tol) {
    out = x;
    return true;
  }
  return false;
}

}  // namespace wfk
