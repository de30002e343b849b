// Global-pose ICP arithmetic shared by the device update (assoc.cu) and a host
// check: the restated Eigen LDLT, orthonormalize and the per-iteration
// decisions of estimate_global_pose (solver.cpp:590-613).
#pragma once
#include "../../include/wfk_types.h"
#include "wfk_common.cuh"

namespace wfk {

struct IcpDev {
  double R[9], t[3];    // res.pose
  double pR[9], pt[3];  // prev_pose
  double prev_rms, rms;
  int32_t iterations, done, converged, degraded;
};
constexpr int kIcpVals = 30;  // 21 (lower triangle of H) + 6 (g) + err + wsum + count

// Eigen LDLT<MatrixXd> (symmetric pivoting) restated as in the oracle, 6x6
WF_HD void icp_ldlt_solve(double (*A)[6], const double* b, double* x) {
  constexpr int n = 6;
  int tr[n];
  double temp[n];
  for (int k = 0; k < n; ++k) {
    int big = k;
    for (int i = k + 1; i < n; ++i)
      if (fabs(A[i][i]) > fabs(A[big][big])) big = i;
    tr[k] = big;
    if (big != k) {
      for (int j = 0; j < k; ++j) {
        const double t = A[k][j];
        A[k][j] = A[big][j];
        A[big][j] = t;
      }
      for (int i = big + 1; i < n; ++i) {
        const double t = A[i][k];
        A[i][k] = A[i][big];
        A[i][big] = t;
      }
      const double t = A[k][k];
      A[k][k] = A[big][big];
      A[big][big] = t;
      for (int i = k + 1; i < big; ++i) {
        const double u = A[i][k];
        A[i][k] = A[big][i];
        A[big][i] = u;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = A[j][j] * A[k][j];
      double d = 0;
      for (int j = 0; j < k; ++j) d += A[k][j] * temp[j];
      A[k][k] -= d;
      for (int i = k + 1; i < n; ++i) {
        double s = 0;
        for (int j = 0; j < k; ++j) s += A[i][j] * temp[j];
        A[i][k] -= s;
      }
    }
    const double akk = A[k][k];
    if (fabs(akk) > 0)
      for (int i = k + 1; i < n; ++i) A[i][k] /= akk;
  }
  for (int i = 0; i < n; ++i) x[i] = b[i];
  for (int k = 0; k < n; ++k) {
    const double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) x[i] -= A[i][j] * x[j];
  for (int i = 0; i < n; ++i) {
    const double d = A[i][i];
    x[i] = fabs(d) > 2.2250738585072014e-308 ? x[i] / d : 0.0;
  }
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) x[i] -= A[j][i] * x[j];
  for (int k = n - 1; k >= 0; --k) {
    const double t = x[k];
    x[k] = x[tr[k]];
    x[tr[k]] = t;
  }
}

// orthonormalize (core.cpp:30-40)
WF_HD M3 icp_orthonormalize(const M3& m) {
  M3 u, v;
  double sv[3];
  svd3(m, u, sv, v);
  M3 r = mul(u, transpose(v));
  if (det(r) < 0) {
    M3 flip = m3_identity();
    flip.a[2][2] = -1;
    r = mul(mul(u, flip), transpose(v));
  }
  return r;
}

// one ICP iteration's decisions and step from the summed terms (solver.cpp:590-613).
// h / mg / delta are caller-provided scratch: the device update passes shared
// memory -- with thread-local arrays the inlined step returned wrong
// translations on sm_100a while each piece alone was bit-exact with the host
// (tools/icp_step_test.cu compares the two).
WF_HD void icp_step(const double* tot, IcpDev& st, const wfk_icp_params& prm, double (*h)[6], double* mg,
                    double* delta) {
  double R0[9], t0[3];
  for (int i = 0; i < 9; ++i) R0[i] = st.R[i];
  for (int i = 0; i < 3; ++i) t0[i] = st.t[i];
  const double prev_rms = st.prev_rms;
  if (tot[29] < double(prm.min_correspondences)) {  // :590-593
    st.degraded = 1;
    st.done = 1;
    return;
  }
  const double rms = sqrt(tot[27] / fmax(tot[28], 1e-300));
  const int iterations = st.iterations + 1;
  st.iterations = iterations;
  if (rms > prev_rms * (1.0 - fmax(prm.rel_tol, prm.min_improvement))) {  // :599-604: revert
    for (int i = 0; i < 9; ++i) st.R[i] = st.pR[i];
    for (int i = 0; i < 3; ++i) st.t[i] = st.pt[i];
    st.rms = prev_rms;
    st.converged = 1;
    st.done = 1;
    return;
  }
  for (int i = 0, k = 0; i < 6; ++i)
    for (int q = 0; q <= i; ++q, ++k) {
      h[i][q] = tot[k];
      h[q][i] = tot[k];
    }
  double dmax = h[0][0];
  for (int i = 1; i < 6; ++i) dmax = fmax(dmax, h[i][i]);
  const double damp = 1e-3 * dmax;  // :608
  for (int i = 0; i < 6; ++i) h[i][i] += damp;
  for (int i = 0; i < 6; ++i) mg[i] = -tot[21 + i];
  icp_ldlt_solve(h, mg, delta);
  M3 step = m3_identity();  // I + [omega]_x (:610-613)
  step.a[0][1] += -delta[2];
  step.a[0][2] += delta[1];
  step.a[1][0] += delta[2];
  step.a[1][2] += -delta[0];
  step.a[2][0] += -delta[1];
  step.a[2][1] += delta[0];
  M3 R;
  for (int i = 0; i < 9; ++i) R.a[i / 3][i % 3] = R0[i];
  const M3 Rn = icp_orthonormalize(mul(step, R));
  const V3 tn = mul(step, V3{t0[0], t0[1], t0[2]}) + V3{delta[3], delta[4], delta[5]};
  for (int i = 0; i < 9; ++i) st.pR[i] = R0[i];
  for (int i = 0; i < 3; ++i) st.pt[i] = t0[i];
  st.prev_rms = rms;
  st.rms = rms;
  for (int i = 0; i < 9; ++i) st.R[i] = Rn.a[i / 3][i % 3];
  st.t[0] = tn.x;
  st.t[1] = tn.y;
  st.t[2] = tn.z;
  if (iterations >= prm.max_iters) st.done = 1;
}

inline void icp_step_host(const double* tot, IcpDev& st, const wfk_icp_params& prm) {
  double h[6][6], mg[6], delta[6];
  icp_step(tot, st, prm, h, mg, delta);
}

}  // namespace wfk
