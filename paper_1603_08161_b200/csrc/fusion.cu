// Deformed-TSDF fusion on sm_100a (proj/src/fusion.cpp:7-126) and the active
// set it grows (proj/src/solver.cpp:32-69).
//
// All per-lattice-point work is one thread per point over the x-fastest SoA
// lattice (coalesced float / double streams).  The warp S(x) and the
// projective depth lookup are evaluated in fp64 with separately rounded
// operations in the reference order, so gate classes, fused values and the
// four FusionStats counters are bit-identical to the CPU reference.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"
#include "volume_math.cuh"

namespace wfk {

// cells with all 8 corners observed and a sign change mark their corners
// (solver.cpp:35-54)
__global__ void k_surface_cells(Grid g, const float* tsdf, const float* weight, uint8_t* on_surface) {
  const int64_t ncell = int64_t(g.nx - 1) * (g.ny - 1) * (g.nz - 1);
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
    const int cx = int(c % (g.nx - 1));
    const int cy = int((c / (g.nx - 1)) % (g.ny - 1));
    const int cz = int(c / (int64_t(g.nx - 1) * (g.ny - 1)));
    bool pos = false, neg = false, observed = true;
    int corners[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = g.lin(cx + (k & 1), cy + ((k >> 1) & 1), cz + (k >> 2));
      corners[k] = i;
      if (weight[i] <= 0.f) observed = false;
      if (tsdf[i] < 0)
        neg = true;
      else
        pos = true;
    }
    if (!observed || !pos || !neg) continue;
#pragma unroll
    for (int k = 0; k < 8; ++k) on_surface[corners[k]] = 1;
  }
}

// one-ring dilation, grow-only OR into active (solver.cpp:56-64)
__global__ void k_dilate(Grid g, const uint8_t* on_surface, uint8_t* active) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < g.n(); i += int64_t(gridDim.x) * blockDim.x) {
    if (!on_surface[i]) continue;
    active[i] = 1;
    int x, y, z;
    g.idx3(int(i), x, y, z);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int a = x + kFace[k][0], b = y + kFace[k][1], c = z + kFace[k][2];
      if (g.in_grid(a, b, c)) active[g.lin(a, b, c)] = 1;
    }
  }
}

static void active_set_device(wfk_ctx* c) {
  VolumeDev& v = c->vol;
  cudaStream_t s = c->stream;
  uint8_t* on = c->mask.ensure(size_t(2 * v.n));
  WFK_CUDA(cudaMemsetAsync(on, 0, size_t(v.n), s));
  const int64_t ncell = int64_t(v.g.nx - 1) * (v.g.ny - 1) * (v.g.nz - 1);
  k_surface_cells<<<grid_for(ncell), kBlock, 0, s>>>(v.g, v.tsdf, v.weight, on);
  k_dilate<<<grid_for(v.n), kBlock, 0, s>>>(v.g, on, v.active);
  count_launch(c, 2);
  ++v.active_gen;
  WFK_CUDA(cudaGetLastError());
}

void fusion_compute_active_set(wfk_ctx* c, int32_t* out, int64_t cap, int64_t* n_out) {
  if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  active_set_device(c);
  VolumeDev& v = c->vol;
  cudaStream_t s = c->stream;
  int32_t* list = c->ivec.ensure(size_t(v.n) + 32);
  int32_t* d_count = list + v.n + 8;
  size_t tmp = 0;
  thrust::counting_iterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmp, it, v.active.p, list, d_count, int(v.n), s);
  c->temp.ensure(tmp);
  WFK_CUDA(cub::DeviceSelect::Flagged(c->temp.p, tmp, it, v.active.p, list, d_count, int(v.n), s));
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, d_count, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  const int64_t n = c->h_pinned[0];
  if (n_out) *n_out = n;
  if (out) {
    if (n > cap) throw Error(WFK_E_CAPACITY, "active list buffer too small");
    WFK_CUDA(cudaMemcpyAsync(out, list, size_t(n) * 4, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  }
}

// integrate_frame (fusion.cpp:15-68), one lattice point per thread
struct IntegrateArgs {
  Grid g;
  double mu;
  PoseD pose;
  wfk_intrinsics K;
  const float* depth;
  const float* color;
  int k_min, bootstrap;
  double w_max, sample_weight;
  float* tsdf;
  float* weight;
  float* vcolor;
  const double* deformed;
  const int32_t* age;
  const uint8_t* active;
  int32_t* counts;  // fused, gate, frustum, occluded
};

__global__ void k_integrate(IntegrateArgs a) {
  int cnt[4] = {0, 0, 0, 0};
  const int W = a.K.width, H = a.K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.g.n(); i += int64_t(gridDim.x) * blockDim.x) {
    if (!a.bootstrap && (!a.active[i] || a.age[i] < a.k_min)) {
      ++cnt[1];
      continue;
    }
    const V3 warped = a.pose.apply(a.g.interpolate(a.deformed, a.g.canonical(int(i))));
    if (warped.z <= 0) {
      ++cnt[2];
      continue;
    }
    const double ux = a.K.fx * warped.x / warped.z + a.K.cx;
    const double uy = a.K.fy * warped.y / warped.z + a.K.cy;
    const int u = int(llround(ux));
    const int v = int(llround(uy));
    if (u < 0 || v < 0 || u >= W || v >= H) {
      ++cnt[2];
      continue;
    }
    double depth = a.depth[int64_t(v) * W + u];
    {
      const int u0 = clampi(int(floor(ux)), 0, W - 2);
      const int v0 = clampi(int(floor(uy)), 0, H - 2);
      const float d00 = a.depth[int64_t(v0) * W + u0], d10 = a.depth[int64_t(v0) * W + u0 + 1];
      const float d01 = a.depth[int64_t(v0 + 1) * W + u0], d11 = a.depth[int64_t(v0 + 1) * W + u0 + 1];
      if (d00 > 0 && d10 > 0 && d01 > 0 && d11 > 0) {
        const double fu = clampd(ux - u0, 0.0, 1.0);
        const double fv = clampd(uy - v0, 0.0, 1.0);
        depth = (1 - fv) * ((1 - fu) * d00 + fu * d10) + fv * ((1 - fu) * d01 + fu * d11);
      }
    }
    if (depth <= 0) {
      ++cnt[2];
      continue;
    }
    const double sdf = double(depth) - warped.z;
    if (sdf < -a.mu) {
      ++cnt[3];
      continue;
    }
    const double d = fmin(sdf, a.mu);
    const double w = a.sample_weight;
    const double w_old = a.weight[i];
    a.tsdf[i] = float((w_old * a.tsdf[i] + w * d) / (w_old + w));
    if (a.color) {
      const int64_t pix = 3 * (int64_t(v) * W + u);
      for (int k = 0; k < 3; ++k) {
        const float ck = (float(w_old) * a.vcolor[3 * i + k] + float(w) * a.color[pix + k]) / float(w_old + w);
        a.vcolor[3 * i + k] = clampf(ck, 0.f, 255.f);
      }
    }
    a.weight[i] = float(fmin(w_old + w, a.w_max));
    ++cnt[0];
  }
  // integer stats: warp then block aggregation, 4 atomics per block
  __shared__ int sc[4];
  if (threadIdx.x < 4) sc[threadIdx.x] = 0;
  __syncthreads();
  for (int k = 0; k < 4; ++k) {
    int v = cnt[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sc[k], v);
  }
  __syncthreads();
  if (threadIdx.x < 4 && sc[threadIdx.x]) atomicAdd(&a.counts[threadIdx.x], sc[threadIdx.x]);
}

void fusion_integrate(wfk_ctx* c, const wfk_pose* pose, const wfk_fusion_params& p, wfk_fusion_stats* out) {
  VolumeDev& v = c->vol;
  if (!v.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  if (c->frame.K.width <= 0) throw Error(WFK_E_INVALID_ARG, "no frame uploaded");
  cudaStream_t s = c->stream;
  int32_t* counts = c->flags.ensure(16);
  WFK_CUDA(cudaMemsetAsync(counts, 0, 4 * sizeof(int32_t), s));
  IntegrateArgs a;
  a.g = v.g;
  a.mu = v.mu;
  a.pose = pose_dev(pose);
  a.K = c->frame.K;
  a.depth = c->frame.depth;
  a.color = c->frame.has_color ? c->frame.color : nullptr;
  a.k_min = p.k_min;
  a.bootstrap = p.bootstrap;
  a.w_max = p.w_max;
  a.sample_weight = p.sample_weight;
  a.tsdf = v.tsdf;
  a.weight = v.weight;
  a.vcolor = v.color;
  a.deformed = v.deformed;
  a.age = v.age;
  a.active = v.active;
  a.counts = counts;
  k_integrate<<<std::min(grid_for(v.n), c->num_sms * 16), kBlock, 0, s>>>(a);
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, counts, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  if (out) {
    out->fused = c->h_pinned[0];
    out->skipped_gate = c->h_pinned[1];
    out->skipped_frustum = c->h_pinned[2];
    out->skipped_occluded = c->h_pinned[3];
  }
}

// expand_grid extrapolation for newly active points (fusion.cpp:96-120)
__global__ void k_expand(Grid g, const uint8_t* was, const uint8_t* active, double* deformed, double* euler,
                         int32_t* age, int32_t* counts) {
  int act = 0, orph = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < g.n(); i += int64_t(gridDim.x) * blockDim.x) {
    if (!active[i] || was[i]) continue;
    ++act;
    int x, y, z;
    g.idx3(int(i), x, y, z);
    const V3 can = g.canonical(int(i));
    V3 sum{0, 0, 0};
    int found = 0, nearest = -1;
    for (int k = 0; k < 6; ++k) {
      const int a = x + kFace[k][0], b = y + kFace[k][1], c = z + kFace[k][2];
      if (!g.in_grid(a, b, c)) continue;
      const int j = g.lin(a, b, c);
      if (!was[j]) continue;
      sum += ld3(deformed, j) + mul(euler_to_matrix(ld3(euler, j)), can - g.canonical(j));
      if (nearest < 0) nearest = j;
      ++found;
    }
    age[i] = 0;
    if (found > 0) {
      st3(deformed, i, sum / double(found));
      st3(euler, i, ld3(euler, nearest));
    } else {
      st3(deformed, i, can);
      st3(euler, i, V3{0, 0, 0});
      ++orph;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    act += __shfl_xor_sync(0xffffffffu, act, o);
    orph += __shfl_xor_sync(0xffffffffu, orph, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (act) atomicAdd(&counts[0], act);
    if (orph) atomicAdd(&counts[1], orph);
  }
}

void fusion_expand(wfk_ctx* c, wfk_expansion_stats* out) {
  VolumeDev& v = c->vol;
  if (!v.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  cudaStream_t s = c->stream;
  uint8_t* buf = c->mask.ensure(size_t(2 * v.n));
  uint8_t* was = buf + v.n;
  WFK_CUDA(cudaMemcpyAsync(was, v.active.p, size_t(v.n), cudaMemcpyDeviceToDevice, s));
  active_set_device(c);
  int32_t* counts = c->flags.ensure(16) + 4;
  WFK_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s));
  k_expand<<<std::min(grid_for(v.n), c->num_sms * 16), kBlock, 0, s>>>(v.g, was, v.active, v.deformed, v.euler,
                                                                       v.age, counts);
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, counts, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  if (out) {
    out->activated = c->h_pinned[0];
    out->orphans = c->h_pinned[1];
  }
}

__global__ void k_ages_list(const int32_t* idx, int64_t n, int32_t* age) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(&age[idx[k]], 1);
}
__global__ void k_ages_active(int64_t n, const uint8_t* active, int32_t* age) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (active[i]) age[i] += 1;
}

void fusion_advance_ages(wfk_ctx* c, const int32_t* idx, int64_t n) {
  VolumeDev& v = c->vol;
  if (!v.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  if (n <= 0) return;
  int32_t* d = c->ivec.ensure(size_t(n) + 32);
  WFK_CUDA(cudaMemcpyAsync(d, idx, size_t(n) * 4, cudaMemcpyHostToDevice, c->stream));
  k_ages_list<<<grid_for(n), kBlock, 0, c->stream>>>(d, n, v.age);
  count_launch(c);
  WFK_CUDA(cudaStreamSynchronize(c->stream));
}

void fusion_advance_active_ages(wfk_ctx* c) {
  VolumeDev& v = c->vol;
  if (!v.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  k_ages_active<<<grid_for(v.n), kBlock, 0, c->stream>>>(v.n, v.active, v.age);
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// DeformableVolume::invert_warp (volume.cpp:68-126), one thread per point
// ---------------------------------------------------------------------------
__global__ void k_invert_warp(Grid g, const double* deformed, PoseD pose, int64_t n, const double* y,
                              const double* seed, int max_iters, double tol, double* xo, uint8_t* ok) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    V3 out;
    ok[i] = invert_warp_point(g, deformed, pose, ld3(y, i), ld3(seed, i), max_iters, tol, out) ? 1 : 0;
    st3(xo, i, out);
  }
}

void volume_invert_warp(wfk_ctx* c, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                        int32_t max_iters, double tol, double* x, uint8_t* ok) {
  if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  if (n <= 0) return;
  cudaStream_t s = c->stream;
  double* d = c->dvec.ensure(9 * size_t(n));
  uint8_t* dok = c->mask.ensure(size_t(n));
  WFK_CUDA(cudaMemcpyAsync(d, y, 3 * size_t(n) * 8, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(d + 3 * n, seed, 3 * size_t(n) * 8, cudaMemcpyHostToDevice, s));
  PoseD pd;
  for (int i = 0; i < 9; ++i) pd.r.a[i / 3][i % 3] = pose ? pose->rotation[i] : (i % 4 == 0 ? 1.0 : 0.0);
  pd.t = pose ? V3{pose->translation[0], pose->translation[1], pose->translation[2]} : V3{0, 0, 0};
  k_invert_warp<<<grid_for(n), kBlock, 0, s>>>(c->vol.g, c->vol.deformed, pd, n, d, d + 3 * n, max_iters, tol,
                                               d + 6 * n, dok);
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(x, d + 6 * n, 3 * size_t(n) * 8, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(ok, dok, size_t(n), cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
}

}  // namespace wfk
