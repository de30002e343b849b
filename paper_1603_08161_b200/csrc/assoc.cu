// Correspondence generation on sm_100a: depth back-projection
// (proj/src/correspond.cpp:7-57), marching cubes + normals
// (proj/src/isosurface.cpp:39-112), z-buffered rasterisation
// (proj/src/rasterize.cpp:29-137) and projective association
// (proj/src/correspond.cpp:59-150) -- the reference's "raycast".
//
// Integer outputs (vertex numbering, triangle order, coverage, z-test winner,
// correspondence selection and order) are bit-identical to the reference:
//  * marching cubes numbers vertices by first use in z-y-x cell scan order:
//    an edge's vertex is created by the first valid cell (scan order) sharing
//    the edge, at that cell's first reference in its case list; three passes
//    (case -> counts -> scan -> vertices -> triangles) reproduce it without a
//    hash map;
//  * normals gather incident triangles in ascending triangle index (the
//    reference's scatter order) through a vertex->triangle CSR;
//  * the z-test keeps the lowest triangle index among equal float depths with
//    one 64-bit atomicMin on (float depth bits, triangle index) per covered
//    pixel, then the winner's attributes are resolved per pixel;
//  * association compacts per-pixel candidates in row-major order.
#include <mutex>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "../../include/wfk_mc_cases.h"
#include "wfk_context.cuh"
#include "wfk_solver.cuh"
#include "icp_math.cuh"

namespace wfk {

// ---------------------------------------------------------------------------
// marching-cubes tables in constant memory
// ---------------------------------------------------------------------------
struct McTables {
  int8_t edges[256][16];  // case -> edge list (-1 terminated)
  int8_t ntri[256];
  int8_t edge_corner[12][2];
  int8_t edge_lower[12];  // lower corner of the edge along its axis
  int8_t edge_axis[12];
  int8_t corner_off[8][3];
};
__constant__ McTables c_mc;
// __constant__ memory is per device: upload once per device, under a lock
static std::mutex g_mc_mu;
static unsigned long long g_mc_ready = 0;  // bit d: tables uploaded to device d

static void mc_tables_init() {
  int dev = 0;
  WFK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_mc_mu);
  if (g_mc_ready & (1ull << (dev & 63))) return;
  McTables t;
  for (int c = 0; c < 256; ++c) {
    const char* s = kWfMcCases[c];
    int n = 0;
    for (; s[n]; ++n) t.edges[c][n] = int8_t(s[n] <= '9' ? s[n] - '0' : s[n] - 'a' + 10);
    for (int k = n; k < 16; ++k) t.edges[c][k] = -1;
    t.ntri[c] = int8_t(n / 3);
  }
  for (int e = 0; e < 12; ++e) {
    const int a = kWfMcEdgeCorners[e][0], b = kWfMcEdgeCorners[e][1];
    t.edge_corner[e][0] = int8_t(a);
    t.edge_corner[e][1] = int8_t(b);
    // isosurface.cpp:25-35 classify_edge
    int axis = 0, lower = a;
    for (int k = 0; k < 3; ++k)
      if (kWfMcCornerOffset[a][k] != kWfMcCornerOffset[b][k]) {
        axis = k;
        lower = kWfMcCornerOffset[a][k] < kWfMcCornerOffset[b][k] ? a : b;
        break;
      }
    t.edge_axis[e] = int8_t(axis);
    t.edge_lower[e] = int8_t(lower);
  }
  for (int c = 0; c < 8; ++c)
    for (int k = 0; k < 3; ++k) t.corner_off[c][k] = int8_t(kWfMcCornerOffset[c][k]);
  WFK_CUDA(cudaMemcpyToSymbol(c_mc, &t, sizeof(t)));
  g_mc_ready |= 1ull << (dev & 63);
}

// ---------------------------------------------------------------------------
// backproject_depth (correspond.cpp:7-57), one pixel per thread
// ---------------------------------------------------------------------------
WF_D bool bp_point(const float* depth, const wfk_intrinsics& K, int x, int y, V3& p) {
  const float d = depth[int64_t(y) * K.width + x];
  if (d <= 0.f) return false;
  const double dd = d;
  p = V3{(double(x) - K.cx) / K.fx * dd, (double(y) - K.cy) / K.fy * dd, dd};
  return true;
}

__global__ void k_backproject(wfk_intrinsics K, const float* depth, double* point, double* normal, uint8_t* pv,
                              uint8_t* nv) {
  const int64_t npx = int64_t(K.width) * K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(i % K.width), y = int(i / K.width);
    V3 p{0, 0, 0};
    const bool ok = bp_point(depth, K, x, y, p);
    st3(point, i, p);
    pv[i] = ok ? 1 : 0;
    V3 n{0, 0, 0};
    uint8_t nok = 0;
    if (ok && y > 0 && y < K.height - 1 && x > 0 && x < K.width - 1) {
      V3 pl, pr, pu, pd;
      if (bp_point(depth, K, x - 1, y, pl) && bp_point(depth, K, x + 1, y, pr) && bp_point(depth, K, x, y - 1, pu) &&
          bp_point(depth, K, x, y + 1, pd)) {
        const V3 du = pr - pl;
        const V3 dv = pd - pu;
        V3 nn = cross(du, dv);
        const double len = norm3(nn);
        if (!(len < 1e-20)) {
          nn = nn / len;
          if (dot(nn, p) > 0) nn = -nn;
          n = nn;
          nok = 1;
        }
      }
    }
    st3(normal, i, n);
    nv[i] = nok;
  }
}

void assoc_backproject(wfk_ctx* c, wfk_point_normal_map* out) {
  FrameDev& f = c->frame;
  if (f.K.width <= 0) throw Error(WFK_E_INVALID_ARG, "no frame uploaded");
  const int64_t npx = int64_t(f.K.width) * f.K.height;
  f.point.ensure(3 * size_t(npx));
  f.normal.ensure(3 * size_t(npx));
  f.pvalid.ensure(size_t(npx));
  f.nvalid.ensure(size_t(npx));
  k_backproject<<<grid_for(npx), kBlock, 0, c->stream>>>(f.K, f.depth, f.point, f.normal, f.pvalid, f.nvalid);
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
  f.maps_valid = true;
  if (out) {
    cudaStream_t s = c->stream;
    out->width = f.K.width;
    out->height = f.K.height;
    if (out->point) WFK_CUDA(cudaMemcpyAsync(out->point, f.point, 3 * size_t(npx) * 8, cudaMemcpyDeviceToHost, s));
    if (out->normal)
      WFK_CUDA(cudaMemcpyAsync(out->normal, f.normal, 3 * size_t(npx) * 8, cudaMemcpyDeviceToHost, s));
    if (out->point_valid)
      WFK_CUDA(cudaMemcpyAsync(out->point_valid, f.pvalid, size_t(npx), cudaMemcpyDeviceToHost, s));
    if (out->normal_valid)
      WFK_CUDA(cudaMemcpyAsync(out->normal_valid, f.nvalid, size_t(npx), cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  }
}

// ---------------------------------------------------------------------------
// marching cubes (isosurface.cpp:39-97)
// ---------------------------------------------------------------------------
struct CellGrid {
  int cx, cy, cz;  // cells per axis
  WF_HD int64_t n() const { return int64_t(cx) * cy * cz; }
};

// pass 1: case of every cell, -1 when unobserved or empty (isosurface.cpp:47-64)
__global__ void k_mc_case(Grid g, CellGrid cgd, const float* tsdf, const float* weight, int32_t* cell_case) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cgd.n(); c += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(c % cgd.cx), y = int((c / cgd.cx) % cgd.cy), z = int(c / (int64_t(cgd.cx) * cgd.cy));
    int cube = 0;
    bool observed = true;
    for (int k = 0; k < 8; ++k) {
      const int i = g.lin(x + c_mc.corner_off[k][0], y + c_mc.corner_off[k][1], z + c_mc.corner_off[k][2]);
      if (weight[i] <= 0.f) {
        observed = false;
        break;
      }
      if (double(tsdf[i]) < 0) cube |= 1 << k;
    }
    cell_case[c] = (!observed || cube == 0 || cube == 255) ? -1 : cube;
  }
}

// owner cell of a lattice edge: the first valid cell in scan order among the
// (up to four) cells sharing it
WF_D int64_t edge_owner(const CellGrid& cgd, const int32_t* cell_case, int px, int py, int pz, int axis) {
  int oa[4][3];
  if (axis == 0) {
    const int t[4][3] = {{0, -1, -1}, {0, 0, -1}, {0, -1, 0}, {0, 0, 0}};
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 3; ++k) oa[i][k] = t[i][k];
  } else if (axis == 1) {
    const int t[4][3] = {{-1, 0, -1}, {0, 0, -1}, {-1, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 3; ++k) oa[i][k] = t[i][k];
  } else {
    const int t[4][3] = {{-1, -1, 0}, {0, -1, 0}, {-1, 0, 0}, {0, 0, 0}};
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 3; ++k) oa[i][k] = t[i][k];
  }
  for (int i = 0; i < 4; ++i) {
    const int x = px + oa[i][0], y = py + oa[i][1], z = pz + oa[i][2];
    if (x < 0 || y < 0 || z < 0 || x >= cgd.cx || y >= cgd.cy || z >= cgd.cz) continue;
    const int64_t c = x + int64_t(cgd.cx) * (y + int64_t(cgd.cy) * z);
    if (cell_case[c] >= 0) return c;
  }
  return -1;
}

// pass 2: per valid cell, triangle slots and the number of vertices it creates
__global__ void k_mc_count(CellGrid cgd, const int32_t* cell_case, int32_t* ntri, int32_t* nvert) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cgd.n(); c += int64_t(gridDim.x) * blockDim.x) {
    const int cs = cell_case[c];
    if (cs < 0) {
      ntri[c] = 0;
      nvert[c] = 0;
      continue;
    }
    const int x = int(c % cgd.cx), y = int((c / cgd.cx) % cgd.cy), z = int(c / (int64_t(cgd.cx) * cgd.cy));
    unsigned seen = 0;
    int nv = 0;
    for (int k = 0; k < 16 && c_mc.edges[cs][k] >= 0; ++k) {
      const int e = c_mc.edges[cs][k];
      if (seen & (1u << e)) continue;
      seen |= 1u << e;
      const int lc = c_mc.edge_lower[e];
      const int ax = c_mc.edge_axis[e];
      if (edge_owner(cgd, cell_case, x + c_mc.corner_off[lc][0], y + c_mc.corner_off[lc][1],
                     z + c_mc.corner_off[lc][2], ax) == c)
        ++nv;
    }
    ntri[c] = c_mc.ntri[cs];
    nvert[c] = nv;
  }
}

// pass 3: create the owned vertices (isosurface.cpp:73-88)
struct McVertArgs {
  Grid g;
  CellGrid cgd;
  PoseD pose;
  const int32_t* cell_case;
  const int32_t* vert_off;
  const float* tsdf;
  const float* color;
  const double* deformed;
  int32_t* edge_vertex;  // 3n
  double *can, *def;
  float* col;
};

__global__ void k_mc_vertices(McVertArgs a) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < a.cgd.n(); c += int64_t(gridDim.x) * blockDim.x) {
    const int cs = a.cell_case[c];
    if (cs < 0) continue;
    const int x = int(c % a.cgd.cx), y = int((c / a.cgd.cx) % a.cgd.cy), z = int(c / (int64_t(a.cgd.cx) * a.cgd.cy));
    int ci[8];
    double cv[8];
    for (int k = 0; k < 8; ++k) {
      ci[k] = a.g.lin(x + c_mc.corner_off[k][0], y + c_mc.corner_off[k][1], z + c_mc.corner_off[k][2]);
      cv[k] = a.tsdf[ci[k]];
    }
    unsigned seen = 0;
    int vid = a.vert_off[c];
    for (int k = 0; k < 16 && c_mc.edges[cs][k] >= 0; ++k) {
      const int e = c_mc.edges[cs][k];
      if (seen & (1u << e)) continue;
      seen |= 1u << e;
      const int lc = c_mc.edge_lower[e];
      const int ax = c_mc.edge_axis[e];
      if (edge_owner(a.cgd, a.cell_case, x + c_mc.corner_off[lc][0], y + c_mc.corner_off[lc][1],
                     z + c_mc.corner_off[lc][2], ax) != c)
        continue;
      const int ea = c_mc.edge_corner[e][0], eb = c_mc.edge_corner[e][1];
      const double va = cv[ea], vb = cv[eb];
      const V3 pa = a.g.canonical(ci[ea]);
      const V3 pb = a.g.canonical(ci[eb]);
      const double s = va / (va - vb);
      const V3 p = pa + s * (pb - pa);
      st3(a.can, vid, p);
      st3(a.def, vid, a.pose.apply(a.g.interpolate(a.deformed, p)));
      // sample_tsdf(p).color (volume.cpp:128-137): float accumulation
      int idx[8];
      double w[8];
      a.g.anchors(p, idx, w);
      float cr = 0.f, cgc = 0.f, cb = 0.f;
      for (int q = 0; q < 8; ++q) {
        const float fw = static_cast<float>(w[q]);
        cr += fw * a.color[3 * int64_t(idx[q])];
        cgc += fw * a.color[3 * int64_t(idx[q]) + 1];
        cb += fw * a.color[3 * int64_t(idx[q]) + 2];
      }
      a.col[3 * int64_t(vid)] = cr;
      a.col[3 * int64_t(vid) + 1] = cgc;
      a.col[3 * int64_t(vid) + 2] = cb;
      a.edge_vertex[3 * int64_t(ci[lc]) + ax] = vid;
      ++vid;
    }
  }
}

// pass 4: triangles in cell scan order then table order, winding swapped
// (isosurface.cpp:89-93)
__global__ void k_mc_triangles(Grid g, CellGrid cgd, const int32_t* cell_case, const int32_t* tri_off,
                               const int32_t* edge_vertex, int32_t* tri, uint8_t* keep) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < cgd.n(); c += int64_t(gridDim.x) * blockDim.x) {
    const int cs = cell_case[c];
    if (cs < 0) continue;
    const int x = int(c % cgd.cx), y = int((c / cgd.cx) % cgd.cy), z = int(c / (int64_t(cgd.cx) * cgd.cy));
    int t0 = tri_off[c];
    for (int n = 0; n < c_mc.ntri[cs]; ++n) {
      int t[3];
      for (int k = 0; k < 3; ++k) {
        const int e = c_mc.edges[cs][3 * n + k];
        const int lc = c_mc.edge_lower[e];
        const int p = g.lin(x + c_mc.corner_off[lc][0], y + c_mc.corner_off[lc][1], z + c_mc.corner_off[lc][2]);
        t[k] = edge_vertex[3 * int64_t(p) + c_mc.edge_axis[e]];
      }
      const int tmp = t[1];
      t[1] = t[2];
      t[2] = tmp;
      const int64_t slot = t0 + n;
      tri[3 * slot] = t[0];
      tri[3 * slot + 1] = t[1];
      tri[3 * slot + 2] = t[2];
      keep[slot] = (t[0] != t[1] && t[1] != t[2] && t[0] != t[2]) ? 1 : 0;
    }
  }
}

__global__ void k_compact_tri(int64_t T, const int32_t* tri, const uint8_t* keep, const int32_t* pos, int32_t* out) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < T; t += int64_t(gridDim.x) * blockDim.x) {
    if (!keep[t]) continue;
    const int64_t o = pos[t];
    out[3 * o] = tri[3 * t];
    out[3 * o + 1] = tri[3 * t + 1];
    out[3 * o + 2] = tri[3 * t + 2];
  }
}

struct U8ToInt {
  __host__ __device__ int32_t operator()(uint8_t k) const { return k; }
};

template <class T>
static void exclusive_scan(wfk_ctx* c, const T* in, T* out, int64_t n) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, int(n), c->stream);
  c->temp.ensure(tmp);
  WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tmp, in, out, int(n), c->stream));
  count_launch(c);
}

void assoc_extract_mesh(wfk_ctx* c, const wfk_pose* pose, int64_t* nv, int64_t* nt) {
  VolumeDev& v = c->vol;
  if (!v.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  mc_tables_init();
  MeshDev& m = c->mesh;
  cudaStream_t s = c->stream;
  const CellGrid cgd{v.g.nx - 1, v.g.ny - 1, v.g.nz - 1};
  const int64_t NC = cgd.n();
  m.cell_case.ensure(size_t(NC) + 1);
  int32_t* ntri = m.cell_tri_off.ensure(2 * (size_t(NC) + 1));
  int32_t* tri_off = ntri + NC + 1;
  int32_t* nvert = m.cell_vert_off.ensure(2 * (size_t(NC) + 1));
  int32_t* vert_off = nvert + NC + 1;
  k_mc_case<<<grid_for(NC), kBlock, 0, s>>>(v.g, cgd, v.tsdf, v.weight, m.cell_case);
  k_mc_count<<<grid_for(NC), kBlock, 0, s>>>(cgd, m.cell_case, ntri, nvert);
  count_launch(c, 2);
  WFK_CUDA(cudaMemsetAsync(ntri + NC, 0, 4, s));
  WFK_CUDA(cudaMemsetAsync(nvert + NC, 0, 4, s));
  exclusive_scan(c, ntri, tri_off, NC + 1);
  exclusive_scan(c, nvert, vert_off, NC + 1);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, tri_off + NC, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 1, vert_off + NC, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  const int64_t T0 = c->h_pinned[0], V = c->h_pinned[1];
  m.can.ensure(3 * size_t(V));
  m.def.ensure(3 * size_t(V));
  m.nrm.ensure(3 * size_t(V));
  m.col.ensure(3 * size_t(V));
  m.edge_vertex.ensure(3 * size_t(v.n));
  McVertArgs a;
  a.g = v.g;
  a.cgd = cgd;
  a.pose = pose_dev(pose);
  a.cell_case = m.cell_case;
  a.vert_off = vert_off;
  a.tsdf = v.tsdf;
  a.color = v.color;
  a.deformed = v.deformed;
  a.edge_vertex = m.edge_vertex;
  a.can = m.can;
  a.def = m.def;
  a.col = m.col;
  k_mc_vertices<<<grid_for(NC), kBlock, 0, s>>>(a);
  int32_t* tri_raw = c->ivec.ensure(3 * size_t(T0) + 8);
  uint8_t* keep = m.tri_keep.ensure(size_t(T0) + 1);
  k_mc_triangles<<<grid_for(NC), kBlock, 0, s>>>(v.g, cgd, m.cell_case, tri_off, m.edge_vertex, tri_raw, keep);
  count_launch(c, 2);
  // drop degenerate triangles, keeping order (isosurface.cpp:92)
  DevBuf<int32_t>& p32 = m.tri_pos;
  p32.ensure(size_t(T0) + 1);
  int64_t T = 0;
  if (T0 > 0) {
    thrust::transform_iterator<U8ToInt, const uint8_t*, int32_t> it(keep, U8ToInt());
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, p32.p, int(T0 + 1), s);
    c->temp.ensure(tmp);
    WFK_CUDA(cudaMemsetAsync(keep + T0, 0, 1, s));
    WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tmp, it, p32.p, int(T0 + 1), s));
    count_launch(c);
    WFK_CUDA(cudaMemcpyAsync(c->h_pinned, p32.p + T0, 4, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    T = c->h_pinned[0];
  }
  m.tri.ensure(3 * size_t(T) + 3);
  if (T > 0) {
    k_compact_tri<<<grid_for(T0), kBlock, 0, s>>>(T0, tri_raw, keep, p32, m.tri);
    count_launch(c);
  }
  WFK_CUDA(cudaGetLastError());
  m.V = V;
  m.T = T;
  m.normals_valid = false;
  m.adj_valid = false;
  if (nv) *nv = V;
  if (nt) *nt = T;
}

// redeform: deformed vertices from the current field (pipeline.cpp:167-169)
__global__ void k_mesh_warp(Grid g, PoseD pose, int64_t V, const double* deformed, const double* can, double* def) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < V; i += int64_t(gridDim.x) * blockDim.x)
    st3(def, i, pose.apply(g.interpolate(deformed, ld3(can, i))));
}

void assoc_mesh_warp(wfk_ctx* c, const wfk_pose* pose) {
  MeshDev& m = c->mesh;
  if (m.V == 0) return;
  k_mesh_warp<<<grid_for(m.V), kBlock, 0, c->stream>>>(c->vol.g, pose_dev(pose), m.V, c->vol.deformed, m.can, m.def);
  count_launch(c);
  m.normals_valid = false;
  WFK_CUDA(cudaGetLastError());
}

// compute_normals (isosurface.cpp:99-112): vertex -> triangle CSR in
// ascending triangle order, then a per-vertex gather
__global__ void k_adj_keys(int64_t T, const int32_t* tri, int32_t* key, int32_t* val, int32_t* cnt) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < T; t += int64_t(gridDim.x) * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      key[3 * t + k] = tri[3 * t + k];
      val[3 * t + k] = int32_t(t);
      atomicAdd(&cnt[tri[3 * t + k]], 1);
    }
}
__global__ void k_normals(int64_t V, const int32_t* ptr, const int32_t* tris, const int32_t* tri, const double* def,
                          double* nrm) {
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < V; v += int64_t(gridDim.x) * blockDim.x) {
    V3 n{0, 0, 0};
    for (int e = ptr[v]; e < ptr[v + 1]; ++e) {
      const int t = tris[e];
      const V3 a = ld3(def, tri[3 * t]), b = ld3(def, tri[3 * t + 1]), cc = ld3(def, tri[3 * t + 2]);
      n += cross(b - a, cc - a);
    }
    const double len = norm3(n);
    if (len > 1e-20) n = n / len;
    st3(nrm, v, n);
  }
}

void assoc_compute_normals(wfk_ctx* c) {
  MeshDev& m = c->mesh;
  cudaStream_t s = c->stream;
  m.nrm.ensure(3 * size_t(m.V) + 3);
  if (m.V == 0) {
    m.normals_valid = true;
    return;
  }
  if (!m.adj_valid) {
    const int64_t E = 3 * m.T;
    m.adj_ptr.ensure(size_t(m.V) + 1);
    m.adj_tri.ensure(size_t(E) + 1);
    DevBuf<int32_t>& key = m.adj_key;
    DevBuf<int32_t>& val = m.adj_val;
    DevBuf<int32_t>& key2 = m.adj_key2;
    DevBuf<int32_t>& cnt = m.adj_cnt;
    key.ensure(size_t(E) + 1);
    val.ensure(size_t(E) + 1);
    key2.ensure(size_t(E) + 1);
    cnt.ensure(size_t(m.V) + 1);
    WFK_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t(m.V) + 1) * 4, s));
    if (E > 0) {
      k_adj_keys<<<grid_for(m.T), kBlock, 0, s>>>(m.T, m.tri, key, val, cnt);
      count_launch(c);
      int bits = 1;
      while ((int64_t(1) << bits) <= m.V) ++bits;
      size_t tmp = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tmp, key.p, key2.p, val.p, m.adj_tri.p, int(E), 0, bits, s);
      c->temp.ensure(tmp);
      WFK_CUDA(cub::DeviceRadixSort::SortPairs(c->temp.p, tmp, key.p, key2.p, val.p, m.adj_tri.p, int(E), 0, bits, s));
      count_launch(c);
    }
    exclusive_scan(c, cnt.p, m.adj_ptr.p, m.V + 1);
    m.adj_valid = true;
  }
  k_normals<<<grid_for(m.V), kBlock, 0, s>>>(m.V, m.adj_ptr, m.adj_tri, m.tri, m.def, m.nrm);
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
  m.normals_valid = true;
}

// ---------------------------------------------------------------------------
// rasterize (rasterize.cpp:29-137)
// ---------------------------------------------------------------------------
struct TriSetup {
  double sx[3], sy[3];
  double inv_z[3];
  double inv_area;
  int vi[3];  // vertex ids in normalized order
  int xmin, xmax, ymin, ymax;
  int top_left;  // bit k: edge k is top-left
  int valid;
};

WF_D double edge_fn(double ax, double ay, double bx, double by, double px, double py) {
  return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

__global__ void k_tri_setup(int64_t T, const int32_t* tri, const double* def, wfk_intrinsics K, TriSetup* out) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < T; t += int64_t(gridDim.x) * blockDim.x) {
    TriSetup s;
    s.valid = 0;
    const int v0 = tri[3 * t], v1 = tri[3 * t + 1], v2 = tri[3 * t + 2];
    const V3 p[3] = {ld3(def, v0), ld3(def, v1), ld3(def, v2)};
    const int vv[3] = {v0, v1, v2};
    if (p[0].z < 1e-3 || p[1].z < 1e-3 || p[2].z < 1e-3) {
      out[t] = s;
      continue;
    }
    int order[3] = {0, 1, 2};
    for (int k = 0; k < 3; ++k) {
      s.sx[k] = K.fx * p[k].x / p[k].z + K.cx;
      s.sy[k] = K.fy * p[k].y / p[k].z + K.cy;
    }
    double area2 = edge_fn(s.sx[0], s.sy[0], s.sx[1], s.sy[1], s.sx[2], s.sy[2]);
    if (area2 == 0.0) {
      out[t] = s;
      continue;
    }
    if (area2 < 0) {
      double tmp = s.sx[1]; s.sx[1] = s.sx[2]; s.sx[2] = tmp;
      tmp = s.sy[1]; s.sy[1] = s.sy[2]; s.sy[2] = tmp;
      order[1] = 2;
      order[2] = 1;
      area2 = -area2;
    }
    for (int k = 0; k < 3; ++k) {
      s.vi[k] = vv[order[k]];
      s.inv_z[k] = 1.0 / p[order[k]].z;
    }
    s.inv_area = 1.0 / area2;
    double uxmin = s.sx[0], uxmax = s.sx[0], uymin = s.sy[0], uymax = s.sy[0];
    for (int k = 1; k < 3; ++k) {
      uxmin = fmin(uxmin, s.sx[k]);
      uxmax = fmax(uxmax, s.sx[k]);
      uymin = fmin(uymin, s.sy[k]);
      uymax = fmax(uymax, s.sy[k]);
    }
    s.xmin = max(0, int(ceil(uxmin)));
    s.xmax = min(K.width - 1, int(floor(uxmax)));
    s.ymin = max(0, int(ceil(uymin)));
    s.ymax = min(K.height - 1, int(floor(uymax)));
    if (s.xmin > s.xmax || s.ymin > s.ymax) {
      out[t] = s;
      continue;
    }
    s.top_left = 0;
    for (int k = 0; k < 3; ++k) {
      const double ax = s.sx[k], ay = s.sy[k], bx = s.sx[(k + 1) % 3], by = s.sy[(k + 1) % 3];
      if ((ay == by && bx > ax) || (by < ay)) s.top_left |= 1 << k;
    }
    s.valid = 1;
    out[t] = s;
  }
}

// inside test + perspective-correct barycentrics (rasterize.cpp:96-110)
WF_D bool tri_sample(const TriSetup& t, int x, int y, double& l0, double& l1, double& l2, double& z) {
  const double px = double(x), py = double(y);
  double w[3];
  for (int k = 0; k < 3; ++k) {
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    w[k] = edge_fn(t.sx[a], t.sy[a], t.sx[b], t.sy[b], px, py);
    if (w[k] < 0 || (w[k] == 0 && !((t.top_left >> ((k + 1) % 3)) & 1))) return false;
  }
  l0 = w[0] * t.inv_area;
  l1 = w[1] * t.inv_area;
  l2 = 1.0 - l0 - l1;
  const double inv_z = l0 * t.inv_z[0] + l1 * t.inv_z[1] + l2 * t.inv_z[2];
  z = 1.0 / inv_z;
  return true;
}

__global__ void k_raster_z(int64_t T, const TriSetup* setups, int W, unsigned long long* zkey) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < T; t += int64_t(gridDim.x) * blockDim.x) {
    const TriSetup s = setups[t];
    if (!s.valid) continue;
    for (int y = s.ymin; y <= s.ymax; ++y)
      for (int x = s.xmin; x <= s.xmax; ++x) {
        double l0, l1, l2, z;
        if (!tri_sample(s, x, y, l0, l1, l2, z)) continue;
        const float fz = float(z);
        if (!(fz < __int_as_float(0x7f800000))) continue;  // float(z) < +inf
        const unsigned long long key =
            (static_cast<unsigned long long>(__float_as_uint(fz)) << 32) | static_cast<unsigned int>(t);
        atomicMin(&zkey[int64_t(y) * W + x], key);
      }
  }
}

__global__ void k_raster_resolve(int W, int H, const unsigned long long* zkey, const TriSetup* setups,
                                 const double* can, const double* def, const double* nrm, int have_normals,
                                 float* depth, double* point, double* normal, double* canonical) {
  const int64_t npx = int64_t(W) * H;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long key = zkey[i];
    const unsigned int hi = static_cast<unsigned int>(key >> 32);
    if (hi >= 0x7f800000u) {
      depth[i] = __int_as_float(0x7f800000);
      st3(point, i, V3{0, 0, 0});
      st3(normal, i, V3{0, 0, 0});
      st3(canonical, i, V3{0, 0, 0});
      continue;
    }
    const int t = int(key & 0xffffffffu);
    const TriSetup s = setups[t];
    double l0, l1, l2, z;
    tri_sample(s, int(i % W), int(i / W), l0, l1, l2, z);
    depth[i] = float(z);
    V3 pt{0, 0, 0}, nn{0, 0, 0}, cn{0, 0, 0};
    const double lw[3] = {l0, l1, l2};
    V3 poz[3], noz[3], coz[3];
    for (int k = 0; k < 3; ++k) {
      const double zk = 1.0 / s.inv_z[k];
      (void)zk;
      const V3 pv = ld3(def, s.vi[k]);
      poz[k] = pv / pv.z;
      noz[k] = (have_normals ? ld3(nrm, s.vi[k]) : V3{0, 0, 0}) / pv.z;
      coz[k] = ld3(can, s.vi[k]) / pv.z;
    }
    pt = (lw[0] * poz[0] + lw[1] * poz[1] + lw[2] * poz[2]) * z;
    nn = (lw[0] * noz[0] + lw[1] * noz[1] + lw[2] * noz[2]) * z;
    cn = (lw[0] * coz[0] + lw[1] * coz[1] + lw[2] * coz[2]) * z;
    const double nl = norm3(nn);
    st3(point, i, pt);
    st3(normal, i, nl > 1e-20 ? nn / nl : V3{0, 0, 0});
    st3(canonical, i, cn);
  }
}

__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) p[i] = v;
}

void assoc_rasterize(wfk_ctx* c, const wfk_intrinsics& K, wfk_geometry_buffer* out) {
  if (!(K.fx > 0 && K.fy > 0 && K.width > 0 && K.height > 0))
    throw Error(WFK_E_INVALID_ARG, "rasterize: invalid intrinsics");
  MeshDev& m = c->mesh;
  GBufDev& b = c->gbuf;
  cudaStream_t s = c->stream;
  const int64_t npx = int64_t(K.width) * K.height;
  b.w = K.width;
  b.h = K.height;
  b.depth.ensure(size_t(npx));
  b.point.ensure(3 * size_t(npx));
  b.normal.ensure(3 * size_t(npx));
  b.canonical.ensure(3 * size_t(npx));
  b.zkey.ensure(size_t(npx));
  k_fill_u64<<<grid_for(npx), kBlock, 0, s>>>(b.zkey, npx, ~0ull);
  count_launch(c);
  TriSetup* setups = reinterpret_cast<TriSetup*>(b.setup.ensure((sizeof(TriSetup) / 8 + 1) * (size_t(m.T) + 1)));
  if (m.T > 0) {
    k_tri_setup<<<grid_for(m.T), kBlock, 0, s>>>(m.T, m.tri, m.def, K, setups);
    k_raster_z<<<grid_for(m.T, 128), 128, 0, s>>>(m.T, setups, K.width, b.zkey);
    count_launch(c, 2);
  }
  k_raster_resolve<<<grid_for(npx), kBlock, 0, s>>>(K.width, K.height, b.zkey, setups, m.can, m.def, m.nrm,
                                                    m.normals_valid ? 1 : 0, b.depth, b.point, b.normal, b.canonical);
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
  b.valid = true;
  if (out) {
    out->width = K.width;
    out->height = K.height;
    if (out->depth) WFK_CUDA(cudaMemcpyAsync(out->depth, b.depth, size_t(npx) * 4, cudaMemcpyDeviceToHost, s));
    if (out->point) WFK_CUDA(cudaMemcpyAsync(out->point, b.point, 3 * size_t(npx) * 8, cudaMemcpyDeviceToHost, s));
    if (out->normal) WFK_CUDA(cudaMemcpyAsync(out->normal, b.normal, 3 * size_t(npx) * 8, cudaMemcpyDeviceToHost, s));
    if (out->canonical)
      WFK_CUDA(cudaMemcpyAsync(out->canonical, b.canonical, 3 * size_t(npx) * 8, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  }
}

// ---------------------------------------------------------------------------
// find_dense_correspondences (correspond.cpp:114-150)
// ---------------------------------------------------------------------------
struct AssocArgs {
  wfk_intrinsics K;
  wfk_correspond_params p;
  Grid g;
  const float* depth;
  const double *bpoint, *bnormal, *bcanon;
  const double *mpoint, *mnormal;
  const uint8_t *pv, *nv;
  const uint8_t* active;
  int drop_inactive;
  uint8_t* flag;
};

// sample_point_normal (correspond.cpp:69-112)
WF_D bool sample_pn(const AssocArgs& a, double ux, double uy, V3& point, V3& normal) {
  const int W = a.K.width, H = a.K.height;
  const int tu = int(llround(ux));
  const int tv = int(llround(uy));
  if (tu < 0 || tv < 0 || tu >= W || tv >= H) return false;
  const int u0 = clampi(int(floor(ux)), 0, W - 2);
  const int v0 = clampi(int(floor(uy)), 0, H - 2);
  bool smooth = true;
  double zmin = __longlong_as_double(0x7ff0000000000000ll), zmax = -zmin;
  for (int dy = 0; dy < 2 && smooth; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      const int64_t p = int64_t(v0 + dy) * W + (u0 + dx);
      if (!a.pv[p] || !a.nv[p]) {
        smooth = false;
        break;
      }
      zmin = fmin(zmin, a.mpoint[3 * p + 2]);
      zmax = fmax(zmax, a.mpoint[3 * p + 2]);
    }
  if (smooth && zmax - zmin < 0.05) {
    const double fu = clampd(ux - u0, 0.0, 1.0);
    const double fv = clampd(uy - v0, 0.0, 1.0);
    V3 pt{0, 0, 0}, nn{0, 0, 0};
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const double w = (dx ? fu : 1 - fu) * (dy ? fv : 1 - fv);
        const int64_t p = int64_t(v0 + dy) * W + (u0 + dx);
        pt += w * ld3(a.mpoint, p);
        nn += w * ld3(a.mnormal, p);
      }
    const double len = norm3(nn);
    if (len > 1e-12) {
      point = pt;
      normal = nn / len;
      return true;
    }
  }
  const int64_t tp = int64_t(tv) * W + tu;
  if (!a.pv[tp] || !a.nv[tp]) return false;
  point = ld3(a.mpoint, tp);
  normal = ld3(a.mnormal, tp);
  return true;
}

WF_D double kernel_phi(double r, double eps) { return 1.0 - r / eps; }

struct Cand {
  V3 canonical, target, normal;
  double conf;
  int idx[8];
  double w[8];
};

WF_D bool candidate(const AssocArgs& a, int64_t i, Cand& out) {
  if (!isfinite(a.depth[i])) return false;  // GeometryBuffer::valid (isosurface.hpp:42)
  const V3 pc = ld3(a.bpoint, i);
  const V3 nc = ld3(a.bnormal, i);
  if (sqnorm(nc) < 0.5) return false;
  const double ux = a.K.fx * pc.x / pc.z + a.K.cx;
  const double uy = a.K.fy * pc.y / pc.z + a.K.cy;
  V3 pa, na;
  if (!sample_pn(a, ux, uy, pa, na)) return false;
  const double zz = sqnorm(pc);
  const V3 vdir = -(zz > 0 ? pc / sqrt(zz) : pc);
  const double kd = kernel_phi(norm3(pc - pa), a.p.eps_d);
  const double kn = kernel_phi(1.0 - dot(nc, na), a.p.eps_n);
  const double kv = kernel_phi(1.0 - dot(nc, vdir), a.p.eps_v);
  double w = 0.0;
  if (!(kd < 0 || kn < 0 || kv < 0)) {
    const double avg = (kd + kn + kv) / 3.0;
    w = avg * avg;
  }
  if (w <= 0) return false;
  const V3 can = ld3(a.bcanon, i);
  if (!a.g.contains(can)) return false;
  a.g.anchors(can, out.idx, out.w);
  if (a.drop_inactive)
    for (int k = 0; k < 8; ++k)
      if (!a.active[out.idx[k]]) return false;
  out.canonical = can;
  out.target = pa;
  out.normal = na;
  out.conf = w;
  return true;
}

__global__ void k_assoc_flag(AssocArgs a) {
  const int64_t npx = int64_t(a.K.width) * a.K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x) {
    Cand cd;
    a.flag[i] = candidate(a, i, cd) ? 1 : 0;
  }
}

struct ConOut {
  int32_t* kind;
  double* canonical;
  int32_t* anchor;
  double* weight;
  double* target;
  double* normal;
  double* conf;
};

__global__ void k_assoc_write(AssocArgs a, const int32_t* pos, ConOut o) {
  const int64_t npx = int64_t(a.K.width) * a.K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x) {
    if (!a.flag[i]) continue;
    Cand cd;
    candidate(a, i, cd);
    const int64_t k = pos[i];
    o.kind[k] = WFK_DENSE_PLANE;
    st3(o.canonical, k, cd.canonical);
    for (int q = 0; q < 8; ++q) {
      o.anchor[8 * k + q] = cd.idx[q];
      o.weight[8 * k + q] = cd.w[q];
    }
    st3(o.target, k, cd.target);
    st3(o.normal, k, cd.normal);
    o.conf[k] = cd.conf;
  }
}

void assoc_find_dense(wfk_ctx* c, const wfk_intrinsics& K, const wfk_correspond_params& p, bool drop_inactive,
                      int64_t* n_out) {
  FrameDev& f = c->frame;
  GBufDev& b = c->gbuf;
  if (!f.maps_valid) throw Error(WFK_E_INVALID_ARG, "no point/normal maps (call backproject first)");
  if (!b.valid) throw Error(WFK_E_INVALID_ARG, "no geometry buffer (call rasterize first)");
  if (b.w != f.K.width || b.h != f.K.height)
    throw Error(WFK_E_INVALID_ARG, "find_dense_correspondences: size mismatch");
  cudaStream_t s = c->stream;
  const int64_t npx = int64_t(b.w) * b.h;
  AssocArgs a;
  a.K = K;
  a.K.width = b.w;
  a.K.height = b.h;
  a.p = p;
  a.g = c->vol.g;
  a.depth = b.depth;
  a.bpoint = b.point;
  a.bnormal = b.normal;
  a.bcanon = b.canonical;
  a.mpoint = f.point;
  a.mnormal = f.normal;
  a.pv = f.pvalid;
  a.nv = f.nvalid;
  a.active = c->vol.active;
  a.drop_inactive = drop_inactive ? 1 : 0;
  a.flag = c->mask.ensure(size_t(std::max<int64_t>(npx, 2 * c->vol.n)) + 1);
  k_assoc_flag<<<grid_for(npx), kBlock, 0, s>>>(a);
  count_launch(c);
  DevBuf<int32_t>& pos = c->gbuf.assoc_pos;
  pos.ensure(size_t(npx) + 1);
  WFK_CUDA(cudaMemsetAsync(a.flag + npx, 0, 1, s));
  thrust::transform_iterator<U8ToInt, const uint8_t*, int32_t> it(a.flag, U8ToInt());
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, pos.p, int(npx + 1), s);
  c->temp.ensure(tmp);
  WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tmp, it, pos.p, int(npx + 1), s));
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, pos.p + npx, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  const int64_t n = c->h_pinned[0];
  ConIn& ci = c->cons;
  const size_t cap = size_t(n) + 1;
  ci.kind.ensure(cap);
  ci.canonical.ensure(3 * cap);
  ci.anchor.ensure(8 * cap);
  ci.weight.ensure(8 * cap);
  ci.target.ensure(3 * cap);
  ci.normal.ensure(3 * cap);
  ci.conf.ensure(cap);
  ConOut o{ci.kind, ci.canonical, ci.anchor, ci.weight, ci.target, ci.normal, ci.conf};
  if (n > 0) {
    k_assoc_write<<<grid_for(npx), kBlock, 0, s>>>(a, pos, o);
    count_launch(c);
  }
  WFK_CUDA(cudaStreamSynchronize(s));
  ci.count = n;
  ci.n_sparse = 0;  // the dense association replaces every constraint
  if (n_out) *n_out = n;
}

// ---------------------------------------------------------------------------
// estimate_global_pose (solver.cpp:536-614): dense projective point-to-plane ICP
// ---------------------------------------------------------------------------
// Sources (valid buffer samples, solver.cpp:549-558) are compacted in pixel
// order; each iteration is one accumulation launch (per-block partial sums of
// the 6x6 normal equations' lower triangle, g, error, weight and count) and
// one single-warp update launch that sums the partials in fixed block order,
// applies the reference's degraded / revert-and-converge rules, damps, solves
// with the restated Eigen LDLT and updates the pose -- all on the device, so a
// whole ICP costs no host round trip until the result is read.
WF_D bool icp_source(const AssocArgs& a, int64_t i) {
  if (!isfinite(a.depth[i])) return false;  // GeometryBuffer::valid
  if (sqnorm(ld3(a.bnormal, i)) < 0.5) return false;
  return a.g.contains(ld3(a.bcanon, i));
}
__global__ void k_icp_flag(AssocArgs a) {
  const int64_t npx = int64_t(a.K.width) * a.K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x)
    a.flag[i] = icp_source(a, i) ? 1 : 0;
}
// source k: q = interpolate_deformed(canonical) (volume.cpp:61-66), n0 = R0^T n
__global__ void k_icp_write(AssocArgs a, const int32_t* pos, const double* deformed, M3 r0t, double* src) {
  const int64_t npx = int64_t(a.K.width) * a.K.height;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npx; i += int64_t(gridDim.x) * blockDim.x) {
    if (!a.flag[i]) continue;
    const int64_t k = pos[i];
    st3(src, 2 * k, a.g.interpolate(deformed, ld3(a.bcanon, i)));
    st3(src, 2 * k + 1, mul(r0t, ld3(a.bnormal, i)));
  }
}

__global__ void k_icp_accumulate(AssocArgs a, const double* src, const int32_t* n_src, const IcpDev* st,
                                 double* partials) {
  __shared__ double sm[kIcpVals][kBlock / 32];
  if (st->done) return;
  PoseD pose;
  for (int i = 0; i < 9; ++i) pose.r.a[i / 3][i % 3] = st->R[i];
  pose.t = V3{st->t[0], st->t[1], st->t[2]};
  double acc[kIcpVals];
#pragma unroll
  for (int v = 0; v < kIcpVals; ++v) acc[v] = 0;
  const int64_t S = *n_src;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < S; k += int64_t(gridDim.x) * blockDim.x) {
    const V3 p = pose.apply(ld3(src, 2 * k));  // solver.cpp:567-589
    const double ux = a.K.fx * p.x / p.z + a.K.cx;
    const double uy = a.K.fy * p.y / p.z + a.K.cy;
    V3 pa, na;
    if (!sample_pn(a, ux, uy, pa, na)) continue;
    const V3 nc = mul(pose.r, ld3(src, 2 * k + 1));
    const double zz = sqnorm(p);
    const V3 v = -(zz > 0 ? p / sqrt(zz) : p);
    const double kd = kernel_phi(norm3(p - pa), a.p.eps_d);
    const double kn = kernel_phi(1.0 - dot(nc, na), a.p.eps_n);
    const double kv = kernel_phi(1.0 - dot(nc, v), a.p.eps_v);
    double w = 0.0;
    if (!(kd < 0 || kn < 0 || kv < 0)) {
      const double avg = (kd + kn + kv) / 3.0;
      w = avg * avg;
    }
    if (w <= 0) continue;
    const V3 c = cross(p, na);
    const double j[6] = {c.x, c.y, c.z, na.x, na.y, na.z};
    const double r = dot(na, p - pa);
    int t = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const double wj = w * j[i];
#pragma unroll
      for (int q = 0; q <= i; ++q) acc[t++] += wj * j[q];  // H(i, q), lower triangle
      acc[21 + i] += wj * r;
    }
    acc[27] += w * r * r;
    acc[28] += w;
    acc[29] += 1.0;
  }
  // fixed-order block sum: warp trees, then the warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < kIcpVals; ++v) {
    const double x = warp_sum(acc[v]);
    if (lane == 0) sm[v][warp] = x;
  }
  __syncthreads();
  if (threadIdx.x < kIcpVals) {
    double t = 0;
    for (int w2 = 0; w2 < int(blockDim.x >> 5); ++w2) t += sm[threadIdx.x][w2];
    partials[size_t(blockIdx.x) * kIcpVals + threadIdx.x] = t;
  }
}

// one warp per accumulated value: lanes sum strided block partials, then a
// fixed shuffle tree (run-to-run identical); thread 0 takes the step.  After
// convergence the remaining launches of the fixed-length loop return at once.
constexpr int kIcpUpdateThreads = 32 * kIcpVals;
__global__ void __launch_bounds__(kIcpUpdateThreads) k_icp_update(const double* partials, int nblk, IcpDev* st,
                                                                  wfk_icp_params prm, double* tot_out) {
  __shared__ double tot[kIcpVals];
  __shared__ double h[6][6], mg[6], delta[6];
  if (st->done) return;
  const int v = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double t = 0;
  for (int b = lane; b < nblk; b += 32) t += partials[size_t(b) * kIcpVals + v];
  t = warp_sum(t);
  if (lane == 0) {
    tot[v] = t;
    if (tot_out) tot_out[v] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    IcpDev local = *st;
    icp_step(tot, local, prm, h, mg, delta);
    *st = local;
  }
}

// Split in two so wfk_process_frame can queue other work (the feature
// detection on a side stream) between the ICP launches and the readback of
// the pose: begin enqueues every ICP kernel and the asynchronous state
// readback, end waits for it.
void assoc_estimate_pose_begin(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& initial,
                               const wfk_icp_params& prm);
void assoc_estimate_pose_end(wfk_ctx* c, wfk_icp_result* out);

void assoc_estimate_pose(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& initial, const wfk_icp_params& prm,
                         wfk_icp_result* out) {
  assoc_estimate_pose_begin(c, K, initial, prm);
  assoc_estimate_pose_end(c, out);
}

void assoc_estimate_pose_begin(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& initial,
                               const wfk_icp_params& prm) {
  FrameDev& f = c->frame;
  GBufDev& b = c->gbuf;
  if (!f.maps_valid) throw Error(WFK_E_INVALID_ARG, "no point/normal maps (call backproject first)");
  if (!b.valid) throw Error(WFK_E_INVALID_ARG, "no geometry buffer (call rasterize first)");
  if (b.w != f.K.width || b.h != f.K.height) throw Error(WFK_E_INVALID_ARG, "estimate_global_pose: size mismatch");
  if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  cudaStream_t s = c->stream;
  const int64_t npx = int64_t(b.w) * b.h;
  AssocArgs a;
  a.K = K;
  a.K.width = b.w;
  a.K.height = b.h;
  a.p = prm.corr;
  a.g = c->vol.g;
  a.depth = b.depth;
  a.bpoint = b.point;
  a.bnormal = b.normal;
  a.bcanon = b.canonical;
  a.mpoint = f.point;
  a.mnormal = f.normal;
  a.pv = f.pvalid;
  a.nv = f.nvalid;
  a.active = c->vol.active;
  a.drop_inactive = 0;
  a.flag = c->mask.ensure(size_t(std::max<int64_t>(npx, 2 * c->vol.n)) + 1);
  k_icp_flag<<<grid_for(npx), kBlock, 0, s>>>(a);
  WFK_CUDA(cudaMemsetAsync(a.flag + npx, 0, 1, s));
  int32_t* pos = c->icp_pos.ensure(size_t(npx) + 1);
  thrust::transform_iterator<U8ToInt, const uint8_t*, int32_t> it(a.flag, U8ToInt());
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, it, pos, int(npx + 1), s);
  c->temp.ensure(tmp);
  WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tmp, it, pos, int(npx + 1), s));
  double* src = c->icp_src.ensure(6 * size_t(npx) + 6);
  M3 r0;
  for (int i = 0; i < 9; ++i) r0.a[i / 3][i % 3] = initial.rotation[i];
  k_icp_write<<<grid_for(npx), kBlock, 0, s>>>(a, pos, c->vol.deformed, transpose(r0), src);
  count_launch(c, 3);
  // state: pose = initial, prev_rms = +inf
  IcpDev h0{};
  for (int i = 0; i < 9; ++i) h0.R[i] = h0.pR[i] = initial.rotation[i];
  for (int i = 0; i < 3; ++i) h0.t[i] = h0.pt[i] = initial.translation[i];
  h0.prev_rms = __builtin_huge_val();
  h0.done = prm.max_iters <= 0 ? 1 : 0;
  IcpDev* st = reinterpret_cast<IcpDev*>(c->icp_state.ensure(sizeof(IcpDev)));
  IcpDev* hst = reinterpret_cast<IcpDev*>(c->h_pinned + 1024);  // pinned staging (second 4 KB)
  *hst = h0;
  WFK_CUDA(cudaMemcpyAsync(st, hst, sizeof(IcpDev), cudaMemcpyHostToDevice, s));
  const int nblk = c->num_sms * 2;
  double* part = c->icp_part.ensure(size_t(nblk) * kIcpVals);
  static const bool hostcheck = getenv("WFK_ICP_HOSTCHECK") != nullptr;
  double* tot_dbg = hostcheck ? c->dvec.ensure(64) : nullptr;
  IcpDev hcheck = h0;
  for (int i = 0; i < prm.max_iters; ++i) {
    k_icp_accumulate<<<nblk, kBlock, 0, s>>>(a, src, pos + npx, st, part);
    k_icp_update<<<1, kIcpUpdateThreads, 0, s>>>(part, nblk, st, prm, tot_dbg);
    count_launch(c, 2);
    if (hostcheck) {  // debug: the same step on the host from the device's totals
      double tot[kIcpVals];
      IcpDev dev;
      WFK_CUDA(cudaMemcpyAsync(tot, tot_dbg, sizeof(tot), cudaMemcpyDeviceToHost, s));
      WFK_CUDA(cudaMemcpyAsync(&dev, st, sizeof(IcpDev), cudaMemcpyDeviceToHost, s));
      WFK_CUDA(cudaStreamSynchronize(s));
      if (!hcheck.done) icp_step_host(tot, hcheck, prm);
      fprintf(stderr, "[icp check] it %d host t %.9g %.9g %.9g dev t %.9g %.9g %.9g host R0 %.9g dev R0 %.9g\n", i,
              hcheck.t[0], hcheck.t[1], hcheck.t[2], dev.t[0], dev.t[1], dev.t[2], hcheck.R[0], dev.R[0]);
    }
  }
  WFK_CUDA(cudaMemcpyAsync(hst, st, sizeof(IcpDev), cudaMemcpyDeviceToHost, s));
}

void assoc_estimate_pose_end(wfk_ctx* c, wfk_icp_result* out) {
  const IcpDev* hst = reinterpret_cast<const IcpDev*>(c->h_pinned + 1024);
  WFK_CUDA(cudaStreamSynchronize(c->stream));
  std::memset(out, 0, sizeof(*out));
  for (int i = 0; i < 9; ++i) out->pose.rotation[i] = hst->R[i];
  for (int i = 0; i < 3; ++i) out->pose.translation[i] = hst->t[i];
  out->converged = hst->converged;
  out->degraded = hst->degraded;
  out->rms = hst->rms;
  out->iterations = hst->iterations;
}

}  // namespace wfk
