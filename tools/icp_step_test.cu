// Device vs host execution of the ICP step arithmetic (icp_math.cuh) on
// synthetic normal equations -- both compiled from the same source.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr
//        -I../paper_1603_08161_b200/csrc -o icp_step_test icp_step_test.cu
#include <cstdio>
#include <random>
#include <cstdlib>
#include "icp_math.cuh"
using namespace wfk;

__global__ void k_step(const double* tot, IcpDev* st, wfk_icp_params prm) {
  __shared__ double h[6][6], mg[6], delta[6];
  if (threadIdx.x == 0) {
    IcpDev local = *st;
    icp_step(tot, local, prm, h, mg, delta);
    *st = local;
  }
}
__global__ void k_step_global(const double* tot, IcpDev* st, wfk_icp_params prm) {
  __shared__ double h[6][6], mg[6], delta[6];
  if (threadIdx.x == 0) icp_step(tot, *st, prm, h, mg, delta);
}

__global__ void k_ldlt(const double* a36, const double* b, double* x) {
  if (threadIdx.x == 0) {
    double A[6][6];
    for (int i = 0; i < 36; ++i) A[i / 6][i % 6] = a36[i];
    icp_ldlt_solve(A, b, x);
  }
}
__global__ void k_orth(const double* m9, double* r9) {
  if (threadIdx.x == 0) {
    M3 m;
    for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = m9[i];
    const M3 r = icp_orthonormalize(m);
    for (int i = 0; i < 9; ++i) r9[i] = r.a[i / 3][i % 3];
  }
}
__global__ void k_mulv(const double* m9, const double* v3, double* o3) {
  if (threadIdx.x == 0) {
    M3 m;
    for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = m9[i];
    const V3 o = mul(m, V3{v3[0], v3[1], v3[2]}) + V3{1e-3, 2e-3, 3e-3};
    o3[0] = o.x; o3[1] = o.y; o3[2] = o.z;
  }
}

// icp_step's solve and update, with the intermediates written out
__global__ void k_step_dbg(const double* tot, const IcpDev* st0, double* dbg) {
  if (threadIdx.x != 0) return;
  IcpDev st = *st0;
  double h[6][6];
  int t = 0;
  for (int i = 0; i < 6; ++i)
    for (int q = 0; q <= i; ++q) {
      h[i][q] = tot[t];
      h[q][i] = tot[t];
      ++t;
    }
  double dmax = h[0][0];
  for (int i = 1; i < 6; ++i) dmax = fmax(dmax, h[i][i]);
  const double damp = 1e-3 * dmax;
  for (int i = 0; i < 6; ++i) h[i][i] += damp;
  double mg[6], delta[6];
  for (int i = 0; i < 6; ++i) mg[i] = -tot[21 + i];
  icp_ldlt_solve(h, mg, delta);
  for (int i = 0; i < 6; ++i) dbg[i] = delta[i];
  M3 step = m3_identity();
  step.a[0][1] += -delta[2];
  step.a[0][2] += delta[1];
  step.a[1][0] += delta[2];
  step.a[1][2] += -delta[0];
  step.a[2][0] += -delta[1];
  step.a[2][1] += delta[0];
  M3 R;
  for (int i = 0; i < 9; ++i) R.a[i / 3][i % 3] = st.R[i];
  const M3 Rn = icp_orthonormalize(mul(step, R));
  const V3 tn = mul(step, V3{st.t[0], st.t[1], st.t[2]}) + V3{delta[3], delta[4], delta[5]};
  for (int i = 0; i < 9; ++i) dbg[6 + i] = Rn.a[i / 3][i % 3];
  dbg[15] = tn.x; dbg[16] = tn.y; dbg[17] = tn.z;
}

int main() {
  {
    std::mt19937 g2(9);
    std::uniform_real_distribution<double> u2(-1, 1);
    double a[36], b[6], xh[6], xd[6], m9[9], rh[9], rd[9], v3[3] = {0.3, -0.2, 0.1}, oh[3], od[3];
    for (int i = 0; i < 6; ++i)
      for (int k = 0; k <= i; ++k) a[i * 6 + k] = a[k * 6 + i] = u2(g2) + (i == k ? 6.0 : 0.0);
    for (double& x : b) x = u2(g2);
    for (int i = 0; i < 9; ++i) m9[i] = (i % 4 == 0 ? 1.0 : 0.0) + 0.01 * u2(g2);
    double A[6][6];
    for (int i = 0; i < 36; ++i) A[i / 6][i % 6] = a[i];
    icp_ldlt_solve(A, b, xh);
    M3 m;
    for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = m9[i];
    const M3 r = icp_orthonormalize(m);
    for (int i = 0; i < 9; ++i) rh[i] = r.a[i / 3][i % 3];
    const V3 o = mul(m, V3{v3[0], v3[1], v3[2]}) + V3{1e-3, 2e-3, 3e-3};
    oh[0] = o.x; oh[1] = o.y; oh[2] = o.z;
    double *da, *db, *dx, *dm, *dr, *dv, *dout;
    cudaMalloc(&da, 288); cudaMalloc(&db, 48); cudaMalloc(&dx, 48); cudaMalloc(&dm, 72); cudaMalloc(&dr, 72);
    cudaMalloc(&dv, 24); cudaMalloc(&dout, 24);
    cudaMemcpy(da, a, 288, cudaMemcpyHostToDevice); cudaMemcpy(db, b, 48, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, m9, 72, cudaMemcpyHostToDevice); cudaMemcpy(dv, v3, 24, cudaMemcpyHostToDevice);
    k_ldlt<<<1, 32>>>(da, db, dx);
    k_orth<<<1, 32>>>(dm, dr);
    k_mulv<<<1, 32>>>(dm, dv, dout);
    cudaMemcpy(xd, dx, 48, cudaMemcpyDeviceToHost); cudaMemcpy(rd, dr, 72, cudaMemcpyDeviceToHost);
    cudaMemcpy(od, dout, 24, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0, e3 = 0;
    for (int i = 0; i < 6; ++i) e1 = fmax(e1, fabs(xh[i] - xd[i]));
    for (int i = 0; i < 9; ++i) e2 = fmax(e2, fabs(rh[i] - rd[i]));
    for (int i = 0; i < 3; ++i) e3 = fmax(e3, fabs(oh[i] - od[i]));
    printf("ldlt %.3e  orth %.3e  mulv %.3e\n", e1, e2, e3);
    printf("od %g %g %g oh %g %g %g\n", od[0], od[1], od[2], oh[0], oh[1], oh[2]);
  }
  std::mt19937 gen(3);
  std::uniform_real_distribution<double> u(-1, 1);
  int bad = 0;
  for (int trial = 0; trial < 20; ++trial) {
    double tot[kIcpVals] = {};
    for (int s = 0; s < 200; ++s) {  // sum_w w J J^T over random sources
      double j[6];
      for (double& x : j) x = u(gen);
      const double w = 0.5 + 0.5 * u(gen), r = 1e-3 * u(gen);
      int t = 0;
      for (int i = 0; i < 6; ++i) {
        for (int q = 0; q <= i; ++q) tot[t++] += w * j[i] * j[q];
        tot[21 + i] += w * j[i] * r;
      }
      tot[27] += w * r * r;
      tot[28] += w;
      tot[29] += 1;
    }
    IcpDev h0{};
    for (int i = 0; i < 9; ++i) h0.R[i] = h0.pR[i] = (i % 4 == 0) ? 1.0 : 0.0;
    h0.t[0] = 0.01 * trial;
    h0.prev_rms = 1e300;
    wfk_icp_params prm{};
    prm.max_iters = 20;
    prm.min_correspondences = 6;
    prm.rel_tol = 1e-6;
    IcpDev host = h0;
    icp_step_host(tot, host, prm);
    double* dtot;
    IcpDev* dst;
    cudaMalloc(&dtot, sizeof(tot));
    cudaMalloc(&dst, sizeof(IcpDev));
    cudaMemcpy(dtot, tot, sizeof(tot), cudaMemcpyHostToDevice);
    cudaMemcpy(dst, &h0, sizeof(IcpDev), cudaMemcpyHostToDevice);
    double* ddbg;
    cudaMalloc(&ddbg, 18 * 8);
    k_step_dbg<<<1, 32>>>(dtot, dst, ddbg);
    double dbg[18];
    cudaMemcpy(dbg, ddbg, sizeof(dbg), cudaMemcpyDeviceToHost);
    if (trial == 0)
      printf("dbg delta %g %g %g %g %g %g  tn %g %g %g\n", dbg[0], dbg[1], dbg[2], dbg[3], dbg[4], dbg[5], dbg[15],
             dbg[16], dbg[17]);
    if (getenv("GLOBAL")) k_step_global<<<1, 32>>>(dtot, dst, prm); else k_step<<<1, 32>>>(dtot, dst, prm);
    IcpDev dev;
    cudaMemcpy(&dev, dst, sizeof(IcpDev), cudaMemcpyDeviceToHost);
    if (trial == 0) printf("dev R %g %g %g / %g %g %g / %g %g %g  rms %g it %d done %d\n", dev.R[0], dev.R[1], dev.R[2], dev.R[3], dev.R[4], dev.R[5], dev.R[6], dev.R[7], dev.R[8], dev.rms, dev.iterations, dev.done);
    double err = 0;
    for (int i = 0; i < 9; ++i) err = fmax(err, fabs(dev.R[i] - host.R[i]));
    for (int i = 0; i < 3; ++i) err = fmax(err, fabs(dev.t[i] - host.t[i]));
    if (err > 1e-12) ++bad;
    printf("trial %2d  max |dev - host| %.3e   t host %.6g %.6g %.6g  dev %.6g %.6g %.6g (%s)\n", trial, err, host.t[0],
           host.t[1], host.t[2], dev.t[0], dev.t[1], dev.t[2], cudaGetErrorString(cudaGetLastError()));
    cudaFree(dtot);
    cudaFree(dst);
  }
  printf("%d mismatching trials\n", bad);
  return bad ? 1 : 0;
}
