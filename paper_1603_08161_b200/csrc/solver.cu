// Non-rigid alignment solver on sm_100a: the reference's flip-flop
// position-PCG / Procrustes loop over the deformation lattice, coarse to fine
// (proj/src/solver.cpp:32-534), as
//
//   * per-level setup kernels: active-row compaction (ascending lattice order,
//     solver.cpp:115-119), 6-neighbour row table, lock-free union-find for the
//     frozen components (solver.cpp:124-144), constraint preparation and a
//     row-major transpose of the constraint->anchor incidence built with a
//     stable radix sort, so each row gathers its data term without atomics
//     in exactly the reference's accumulation order (solver.cpp:185-195);
//   * ONE cooperative persistent kernel per flip_flop_solve (solver.cpp:419-453)
//     that runs energy, rhs/diagonal assembly, the Jacobi-PCG loop, write-back,
//     the Procrustes rotation fit and the energy trace with grid-wide barriers
//     instead of kernel launches.  The PCG operator is matrix-free: per
//     iteration one pass over the constraints (q_c = sum_k a_k p[a_k],
//     u_c = coef (g.q_c) g) and one pass over rows (sum of a_i u_c over the
//     row's incidence list + the 6-neighbour ARAP Laplacian), replacing the
//     27 x 3x3 fp64 block rows the reference stores (2,081 B per row).
//     Dot products are deterministic two-level reductions (warp shuffle ->
//     per-block partial -> fixed-order sum).
#include <cooperative_groups.h>
#include <chrono>
#include <mutex>
#include <string>

#include <cub/cub.cuh>
#include <type_traits>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"

namespace cg = cooperative_groups;

namespace wfk {

// ============================================================================
// setup kernels
// ============================================================================


__global__ void k_scatter_node_row(const int32_t* rows, int N, int32_t* node_row) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) node_row[rows[r]] = r;
}

// 6 face neighbours per row in the reference's kFaceNeighbors order
// (solver.cpp:17-18); -1 when outside the grid or inactive.
__global__ void k_row_neighbours(Grid g, const int32_t* rows, int N, const int32_t* node_row, int32_t* nbr,
                                 int32_t* uf) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    int x, y, z;
    g.idx3(rows[r], x, y, z);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int a = x + kFace[k][0], b = y + kFace[k][1], c = z + kFace[k][2];
      nbr[int64_t(k) * N + r] = g.in_grid(a, b, c) ? node_row[g.lin(a, b, c)] : -1;
    }
    int m = r;  // hook to the smallest neighbour: parents stay <= children
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int j = nbr[int64_t(k) * N + r];
      if (j >= 0 && j < m) m = j;
    }
    uf[r] = m;
  }
}

// Lock-free union-find (ECL-CC style): a parent is never larger than its
// child, so a set's root is its smallest row and the final labels are
// independent of the race order.  find() halves paths as it walks.
__device__ __forceinline__ int uf_find(int32_t* uf_, int x) {
  volatile int32_t* uf = uf_;
  int cur = uf[x];
  if (cur != x) {
    int next, prev = x;
    while (cur > (next = uf[cur])) {
      uf[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}
__global__ void k_union(const int32_t* nbr, int N, int32_t* uf) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 6; k += 2) {  // +x, +y, +z edges cover every edge once
      const int j = nbr[int64_t(k) * N + r];
      if (j < 0) continue;
      int a = uf_find(uf, r), b = uf_find(uf, j);
      while (a != b) {
        if (a < b) {
          const int t = a;
          a = b;
          b = t;
        }
        const int old = atomicCAS(&uf[a], a, b);
        if (old == a) break;
        a = uf_find(uf, old);
        b = uf_find(uf, b);
      }
    }
  }
}
__global__ void k_uf_compress(int N, int32_t* uf, uint8_t* comp_flag) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    uf[r] = uf_find(uf, r);
    comp_flag[r] = 0;
  }
}

// Per-constraint preparation at one level: anchor rows, g = R^T n and the
// constant of the rhs (solver.cpp:203-226), constrained-component marks
// (solver.cpp:136-141) and the incidence keys of the row transpose.
__global__ void k_con_prepare(int64_t C, const int32_t* kind, const double* target, const double* normal,
                              const double* conf, const int32_t* c_node, const double* c_w,
                              const int32_t* node_row, const int32_t* uf, PoseD pose, double w_d, double w_s,
                              int N, int32_t* c_row, double* c_g, double* c_b, int32_t* c_kind,
                              uint8_t* comp_flag, int32_t* key, int32_t* val) {
  // one thread per (constraint, corner); corner 0 also does the constraint's g
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < 8 * C; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = i >> 3;
    const int k = int(i & 7);
    if (k == 0) {
      const M3 rt = transpose(pose.r);
      const bool dense = kind[c] == WFK_DENSE_PLANE;
      c_kind[c] = kind[c];
      const V3 n = ld3(normal, c), f = ld3(target, c);
      if (dense) {
        const V3 gv = mul(rt, n);
        c_g[4 * c] = gv.x;
        c_g[4 * c + 1] = gv.y;
        c_g[4 * c + 2] = gv.z;
        c_g[4 * c + 3] = w_d * conf[c];
        c_b[c] = dot(n, pose.t - f);
      } else {
        const V3 v = mul(rt, f - pose.t);
        c_g[4 * c] = v.x;
        c_g[4 * c + 1] = v.y;
        c_g[4 * c + 2] = v.z;
        c_g[4 * c + 3] = w_s * conf[c];
        c_b[c] = 0.0;
      }
    }
    const int row = node_row[c_node[i]];
    const double w = c_w[i];
    c_row[i] = row;
    if (row >= 0 && w > 0) comp_flag[uf[row]] = 1;
    // incidence entry unless alpha_i == 0 (solver.cpp:202)
    key[i] = (row >= 0 && w != 0) ? row * 8 + (7 - k) : N * 8;  // cell order of solver.cpp:185-187; sentinel last
    val[i] = int32_t(i);
  }
}

// sort keys of the pipelined row order: incidences per row (clamped to 16 bits)
__global__ void k_row_count_keys(int N, const int32_t* row_ptr, int32_t* key, int32_t* val) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    key[r] = min(row_ptr[r + 1] - row_ptr[r], 65535);
    val[r] = r;
  }
}

// row_ptr from the sorted incidence keys (row * 8 + corner; sentinel N * 8):
// position e starts every row in (row(e - 1), row(e)], position E8 closes the
// rest, so row_ptr[N] = E (the sentinels sort last).
__global__ void k_row_ptr_from_keys(int64_t E8, const int32_t* key, int N, int32_t* row_ptr) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e <= E8; e += int64_t(gridDim.x) * blockDim.x) {
    const int row = e < E8 ? min(key[e] >> 3, N) : N;
    const int prev = e > 0 ? min(key[e - 1] >> 3, N) : -1;
    for (int r = prev + 1; r <= row; ++r) row_ptr[r] = int32_t(e);
  }
}

__global__ void k_frozen(int N, const int32_t* uf, const uint8_t* comp_flag, uint8_t* frozen) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    frozen[r] = comp_flag[uf[r]] ? 0 : 1;
}

__global__ void k_entries(const int32_t* n_ent, const int32_t* sorted_val, const double* c_w, int32_t* ent_con,
                          uint8_t* ent_k, double* ent_w, int32_t* c_pos) {
  const int64_t E = *n_ent;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < E; e += int64_t(gridDim.x) * blockDim.x) {
    const int v = sorted_val[e];
    ent_con[e] = v >> 3;
    ent_k[e] = uint8_t(v & 7);
    ent_w[e] = c_w[v];
    c_pos[v] = int32_t(e);
  }
}

// work items of the balanced matrix-free row pass (see item_pass)
__global__ void k_item_count(int N, const int32_t* row_ptr, int32_t* n_extra) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const int cnt = row_ptr[r + 1] - row_ptr[r];
    n_extra[r] = cnt > kItemLen ? (cnt - 1) / kItemLen : 0;  // items beyond the row's first
  }
}
__global__ void k_item_write(int N, const int32_t* row_ptr, const int32_t* xptr, int4* xitems, int2* xrange) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const int e0 = row_ptr[r], e1 = row_ptr[r + 1];
    const int x0 = xptr[r], x1 = xptr[r + 1];
    for (int i = x0, k = 1; i < x1; ++i, ++k)
      xitems[i] = make_int4(r, e0 + k * kItemLen, min(e1, e0 + (k + 1) * kItemLen), 0);
    xrange[r] = make_int2(x0, x1 - x0);
  }
}

// Assembled levels: B^T B (solver.cpp:196-226) and the ConstraintCache
// (solver.hpp:66-70).  A block of kAsmWarps warps takes its rows in groups
// of kAsmWarps: a row with at most kAsmLong incidences is summed by one warp,
// a longer one by all warps of the block on contiguous segments whose
// partials are added in segment order (deterministic).  Inside a segment every
// value is summed sequentially in incidence order (cell order,
// solver.cpp:185-195).  The incidences are sorted by the row's corner ki
// inside the cell, so a run of equal ki touches the same 8 stencil slots:
// lane 3j + p (j < 8, p < 3) owns values 2p, 2p + 1 of the slot pairing the
// row with cell corner j, keeps them in registers for the run and swaps them
// through the warp's slot table when ki changes; lanes 24..29 own the six
// cache terms (rhs xyz, diagonal xyz).  Every lane runs the same
// instruction stream -- acc += (P w) Q with P, w, Q picked from the staged
// incidence by a per-lane column (1.0 / 0.0 columns stand for the terms a
// kind does not have) -- and the next chunk's incidences are loaded while
// the current one is summed.
constexpr int kAsmWarps = 8;
constexpr int kAsmLong = 128;  // rows above this many incidences are split over the block
enum { kTsc, kTsd, kTnf, kTggt, kTg = kTggt + 6, kTone = kTg + 3, kTzero, kTcols };
struct AsmStage {
  double t[kTcols][33];  // sc = coef a, sd = coef a^2, -coef a c_b, g g^T, g, 1, 0
  double w[9][33];       // the constraint's 8 corner weights, 1
  int k[32], dense[32];
  double acc[28][6];     // the segment's slot blocks (27) and cache terms (row 27)
};
constexpr size_t kAsmSmem = sizeof(AsmStage) * kAsmWarps;
__device__ __forceinline__ int asm_slot(int ki, int j) {
  return ((j & 1) - (ki & 1) + 1) + 3 * (((j >> 1) & 1) - ((ki >> 1) & 1) + 1) + 9 * ((j >> 2) - (ki >> 2) + 1);
}
struct AsmCon {  // one incidence's constraint data in flight
  int k, dense;
  double a, coef, cb, g[3], w[8];
};
struct AsmIn {
  const int32_t* ent_con;
  const uint8_t* ent_k;
  const double *ent_w, *c_w, *c_g, *c_b;
  const int32_t* c_kind;
};
__device__ __forceinline__ void asm_load(const AsmIn& in, int e, int c, AsmCon& x) {
  x.k = in.ent_k[e];
  x.a = in.ent_w[e];
  x.g[0] = in.c_g[4 * c];
  x.g[1] = in.c_g[4 * c + 1];
  x.g[2] = in.c_g[4 * c + 2];
  x.coef = in.c_g[4 * c + 3];
  x.cb = in.c_b[c];
  x.dense = in.c_kind[c] == WFK_DENSE_PLANE;
#pragma unroll
  for (int k = 0; k < 8; ++k) x.w[k] = in.c_w[8 * int64_t(c) + k];
}
// Sums incidences [s0, s1) of one row into st.acc (zeroed here).
__device__ __forceinline__ void asm_segment(const AsmIn& in, AsmStage& st, int s0, int s1) {
  const int L = threadIdx.x & 31;
  const int j = L / 3, pm = L % 3, cm = L - 24;
  // per-lane columns: (P, w, Q0, Q1) for a dense-plane and for a point incidence
  int pD, pN, wc, q0D, q0N, q1D, q1N;
  if (L < 24) {
    pD = pN = kTsc;
    wc = j;
    q0D = kTggt + 2 * pm;
    q1D = kTggt + 2 * pm + 1;
    q0N = pm == 0 ? kTone : kTzero;  // point: B^T B gains coef a_i a_j I (xx, yy, zz)
    q1N = pm == 0 ? kTzero : kTone;
  } else if (cm < 3) {
    pD = kTnf;
    pN = kTsc;
    wc = 8;
    q0D = q0N = kTg + cm;
    q1D = q1N = kTzero;
  } else if (cm < 6) {
    pD = pN = kTsd;
    wc = 8;
    q0D = kTggt + (cm == 3 ? 0 : cm == 4 ? 3 : 5);
    q0N = kTone;
    q1D = q1N = kTzero;
  } else {
    pD = pN = kTzero;
    wc = 8;
    q0D = q0N = q1D = q1N = kTzero;
  }
  for (int t = L; t < 28 * 6; t += 32) (&st.acc[0][0])[t] = 0.0;
  double a0 = 0, a1 = 0;
  int cur = -1;
  AsmCon nx;
  int c_next = -1;
  if (s0 + L < s1) {
    asm_load(in, s0 + L, in.ent_con[s0 + L], nx);
  }
  if (s0 + 32 + L < s1) c_next = in.ent_con[s0 + 32 + L];
  for (int base = s0; base < s1; base += 32) {
    __syncwarp();
    if (base + L < s1) {  // stage this chunk
      const double sc = nx.coef * nx.a;
      st.k[L] = nx.k;
      st.dense[L] = nx.dense;
      st.t[kTsc][L] = sc;
      st.t[kTsd][L] = sc * nx.a;
      st.t[kTnf][L] = -(sc * nx.cb);
      st.t[kTggt + 0][L] = nx.g[0] * nx.g[0];
      st.t[kTggt + 1][L] = nx.g[0] * nx.g[1];
      st.t[kTggt + 2][L] = nx.g[0] * nx.g[2];
      st.t[kTggt + 3][L] = nx.g[1] * nx.g[1];
      st.t[kTggt + 4][L] = nx.g[1] * nx.g[2];
      st.t[kTggt + 5][L] = nx.g[2] * nx.g[2];
      st.t[kTg + 0][L] = nx.g[0];
      st.t[kTg + 1][L] = nx.g[1];
      st.t[kTg + 2][L] = nx.g[2];
#pragma unroll
      for (int k = 0; k < 8; ++k) st.w[k][L] = nx.w[k];
    }
    // the next chunk's data in flight while this one is summed
    if (base + 32 + L < s1) asm_load(in, base + 32 + L, c_next, nx);
    if (base + 64 + L < s1) c_next = in.ent_con[base + 64 + L];
    __syncwarp();
    const int n = min(32, s1 - base);
    // runs of equal ki inside the chunk (the incidences are sorted by ki)
    const unsigned brk = __ballot_sync(0xffffffffu, L < n && (L == 0 || st.k[L] != st.k[L - 1])) | (n < 32 ? 1u << n : 0u);
    for (int i = 0; i < n;) {
      const int ki = st.k[i];
      const unsigned rest = brk & ~((2u << i) - 1u);
      const int iend = rest ? __ffs(rest) - 1 : 32;
      if (ki != cur) {  // warp-uniform: a new run of the row's corner
        if (cur >= 0 && L < 24) {
          double* q = st.acc[asm_slot(cur, j)];
          q[2 * pm] = a0;
          q[2 * pm + 1] = a1;
        }
        __syncwarp();
        if (L < 24) {
          const double* q = st.acc[asm_slot(ki, j)];
          a0 = q[2 * pm];
          a1 = q[2 * pm + 1];
        }
        cur = ki;
      }
#pragma unroll 4
      for (int ii = i; ii < iend; ++ii) {
        const bool dn = st.dense[ii] != 0;
        const double P = st.t[dn ? pD : pN][ii] * st.w[wc][ii];
        a0 += P * st.t[dn ? q0D : q0N][ii];
        a1 += P * st.t[dn ? q1D : q1N][ii];
      }
      i = iend;
    }
  }
  __syncwarp();
  if (L < 24) {
    if (cur >= 0) {
      double* q = st.acc[asm_slot(cur, j)];
      q[2 * pm] = a0;
      q[2 * pm + 1] = a1;
    }
  } else if (cm < 6) {
    st.acc[27][cm] = a0;
  }
  __syncwarp();
}
// acc (28 x 6, summed over `nseg` stage tables in order) -> the row's outputs;
// threads [0, nthr) of the caller take part
__device__ __forceinline__ void asm_write(const AsmStage* stages, int nseg, int tid, int nthr, const Grid& g, int N,
                                          int r, const int32_t* rows, const int32_t* node_row, double* blk,
                                          int32_t* cols, int soa, double4* crhs, double4* cdiag) {
  for (int t = tid; t < 28 * 6; t += nthr) {
    const int s = t / 6, m = t % 6;
    double v = stages[0].acc[s][m];
    for (int w = 1; w < nseg; ++w) v += stages[w].acc[s][m];
    if (s < 27) {
      blk[soa ? (int64_t(s) * 6 + m) * N + r : int64_t(r) * 27 * 6 + t] = v;
    } else {
      double* out = reinterpret_cast<double*>(m < 3 ? &crhs[r] : &cdiag[r]);
      out[m % 3] = v;
      if (m % 3 == 0) out[3] = 0.0;
    }
  }
  if (tid < 27) {
    const int dx = tid % 3 - 1, dy = (tid / 3) % 3 - 1, dz = tid / 9 - 1;
    int x, y, z;
    g.idx3(rows[r], x, y, z);
    const int col = g.in_grid(x + dx, y + dy, z + dz) ? node_row[g.lin(x + dx, y + dy, z + dz)] : -1;
    cols[soa ? int64_t(tid) * N + r : int64_t(r) * 27 + tid] = col;
  }
}
__global__ void __launch_bounds__(kAsmWarps * 32, 2) k_assemble_rows(
    Grid g, int N, const int32_t* rows, const int32_t* node_row, const int32_t* row_ptr, const int32_t* ent_con,
    const uint8_t* ent_k, const double* ent_w, const double* c_w, const double* c_g, const double* c_b,
    const int32_t* c_kind, double* blk, int32_t* cols, int soa, double4* crhs, double4* cdiag) {
  extern __shared__ double4 asm_smem[];
  AsmStage* stages = reinterpret_cast<AsmStage*>(asm_smem);
  __shared__ int grp[kAsmWarps][2];
  const int warp = threadIdx.x >> 5, L = threadIdx.x & 31;
  AsmStage& st = stages[warp];
  const AsmIn in{ent_con, ent_k, ent_w, c_w, c_g, c_b, c_kind};
  for (int k = L; k < 32; k += 32) {  // constant columns
    st.t[kTone][k] = 1.0;
    st.t[kTzero][k] = 0.0;
    st.w[8][k] = 1.0;
  }
  // rows b, b + G, b + 2G, ... in groups of kAsmWarps
  for (int g0 = blockIdx.x; g0 < N; g0 += gridDim.x * kAsmWarps) {
    __syncthreads();
    if (threadIdx.x < kAsmWarps) {
      const int r = g0 + int(threadIdx.x) * gridDim.x;
      grp[threadIdx.x][0] = r < N ? row_ptr[r] : 0;
      grp[threadIdx.x][1] = r < N ? row_ptr[r + 1] : 0;
    }
    __syncthreads();
    // long rows of the group: every warp one segment
    for (int q = 0; q < kAsmWarps; ++q) {
      const int r = g0 + q * gridDim.x;
      const int e0 = grp[q][0], e1 = grp[q][1];
      if (r >= N || e1 - e0 <= kAsmLong) continue;  // block-uniform
      const int seglen = (e1 - e0 + kAsmWarps - 1) / kAsmWarps;
      asm_segment(in, st, min(e1, e0 + warp * seglen), min(e1, e0 + (warp + 1) * seglen));
      __syncthreads();
      asm_write(stages, kAsmWarps, threadIdx.x, blockDim.x, g, N, r, rows, node_row, blk, cols, soa, crhs, cdiag);
      __syncthreads();
    }
    // short rows: warp q sums row q of the group alone
    const int r = g0 + warp * gridDim.x;
    const int e0 = grp[warp][0], e1 = grp[warp][1];
    if (r < N && e1 - e0 <= kAsmLong) {
      asm_segment(in, st, e0, e1);
      asm_write(&st, 1, L, 32, g, N, r, rows, node_row, blk, cols, soa, crhs, cdiag);
    }
  }
}

// ConstraintCache (solver.hpp:66-70): constraint part of the rhs and of the
// Jacobi diagonal.  Rows with at most kCacheWarpRow incidences accumulate in
// the reference's order (solver.cpp:196-226) on one thread; longer rows (the
// coarse levels) are summed by a warp with a fixed shuffle tree.
WF_D void cache_term(int c, double a, const int32_t* c_kind, const double* c_g, const double* c_b, V3& rhs,
                     V3& diag) {
  const V3 g{c_g[4 * c], c_g[4 * c + 1], c_g[4 * c + 2]};
  const double coef = c_g[4 * c + 3];
  const double s = coef * a * a;
  if (c_kind[c] == WFK_DENSE_PLANE) {
    diag.x += s * (g.x * g.x);
    diag.y += s * (g.y * g.y);
    diag.z += s * (g.z * g.z);
    rhs -= (coef * a * c_b[c]) * g;
  } else {
    diag.x += s * 1.0;
    diag.y += s * 1.0;
    diag.z += s * 1.0;
    rhs += (coef * a) * g;
  }
}

__global__ void k_constraint_cache(int N, const int32_t* row_ptr, const int32_t* ent_con, const double* ent_w,
                                   const int32_t* c_kind, const double* c_g, const double* c_b, double4* crhs,
                                   double4* cdiag) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    if (row_ptr[r + 1] - row_ptr[r] > kCacheWarpRow) continue;
    V3 rhs{0, 0, 0}, diag{0, 0, 0};
    for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) cache_term(ent_con[e], ent_w[e], c_kind, c_g, c_b, rhs, diag);
    crhs[r] = make_double4(rhs.x, rhs.y, rhs.z, 0.0);
    cdiag[r] = make_double4(diag.x, diag.y, diag.z, 0.0);
  }
}

__global__ void k_constraint_cache_warp(int N, const int32_t* row_ptr, const int32_t* ent_con, const double* ent_w,
                                        const int32_t* c_kind, const double* c_g, const double* c_b, double4* crhs,
                                        double4* cdiag) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < N; r += warps) {
    if (row_ptr[r + 1] - row_ptr[r] <= kCacheWarpRow) continue;
    V3 rhs{0, 0, 0}, diag{0, 0, 0};
    for (int e = row_ptr[r] + lane; e < row_ptr[r + 1]; e += 32)
      cache_term(ent_con[e], ent_w[e], c_kind, c_g, c_b, rhs, diag);
    rhs.x = warp_sum(rhs.x);
    rhs.y = warp_sum(rhs.y);
    rhs.z = warp_sum(rhs.z);
    diag.x = warp_sum(diag.x);
    diag.y = warp_sum(diag.y);
    diag.z = warp_sum(diag.z);
    if (lane == 0) {
      crhs[r] = make_double4(rhs.x, rhs.y, rhs.z, 0.0);
      cdiag[r] = make_double4(diag.x, diag.y, diag.z, 0.0);
    }
  }
}

// ============================================================================
// hierarchy (solver.cpp:455-534)
// ============================================================================

// coarse field from the fine one (solver.cpp:470-483), every coarse point
__global__ void k_coarse_init(Grid fine, Grid coarse, const double* f_def, const double* f_eul, double* c_def,
                              double* c_eul, uint8_t* c_act) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < coarse.n();
       i += int64_t(gridDim.x) * blockDim.x) {
    const V3 xc = coarse.canonical(int(i));
    V3 xq = xc;
    double q[3] = {xq.x, xq.y, xq.z};
    for (int k = 0; k < 3; ++k) q[k] = clampd(q[k], fine.org(k), fine.org(k) + fine.voxel * (fine.dim(k) - 1));
    xq = V3{q[0], q[1], q[2]};
    st3(c_def, i, fine.interpolate(f_def, xq) + (xc - xq));
    int nearest[3];
    for (int k = 0; k < 3; ++k)
      nearest[k] = clampi(int(llround((q[k] - fine.org(k)) / fine.voxel)), 0, fine.dim(k) - 1);
    st3(c_eul, i, ld3(f_eul, fine.lin(nearest[0], nearest[1], nearest[2])));
    c_act[i] = 0;
  }
}

// coarse activity: all 8 coarse anchors of every active fine node (solver.cpp:485-490)
__global__ void k_coarse_activity(Grid fine, Grid coarse, const uint8_t* f_act, uint8_t* c_act, int32_t* err) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < fine.n(); i += int64_t(gridDim.x) * blockDim.x) {
    if (!f_act[i]) continue;
    const V3 x = fine.canonical(int(i));
    if (!coarse.contains(x)) {
      atomicOr(err, 2);
      continue;
    }
    int idx[8];
    double w[8];
    coarse.anchors(x, idx, w);
    for (int k = 0; k < 8; ++k) c_act[idx[k]] = 1;
  }
}

// re-anchor every constraint on a coarse lattice (solver.cpp:492-499)
__global__ void k_reanchor(int64_t C, Grid coarse, const double* canonical, int32_t* c_node, double* c_w,
                           uint8_t* c_act, int32_t* err) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < C; c += int64_t(gridDim.x) * blockDim.x) {
    const V3 x = ld3(canonical, c);
    if (!coarse.contains(x)) {
      atomicOr(err, 2);
      for (int k = 0; k < 8; ++k) {
        c_node[8 * c + k] = 0;
        c_w[8 * c + k] = 0;
      }
      continue;
    }
    int idx[8];
    double w[8];
    coarse.anchors(x, idx, w);
    for (int k = 0; k < 8; ++k) {
      c_node[8 * c + k] = idx[k];
      c_w[8 * c + k] = w[k];
      if (w[k] > 0) c_act[idx[k]] = 1;
    }
  }
}

// prolongation coarse -> fine over active fine nodes (solver.cpp:518-529)
// prev <- cur, and flag |= bit if any element differed
__global__ void k_mask_update(int64_t n, const uint8_t* cur, uint8_t* prev, int32_t* flag, int32_t bit) {
  bool diff = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint8_t v = cur[i];
    if (prev[i] != v) {
      diff = true;
      prev[i] = v;
    }
  }
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) atomicOr(flag, bit);
}

__global__ void k_prolong(Grid fine, Grid coarse, const uint8_t* f_act, double* f_def, double* f_eul,
                          const double* c_def, const double* c_eul) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < fine.n(); i += int64_t(gridDim.x) * blockDim.x) {
    if (!f_act[i]) continue;
    const V3 x = fine.canonical(int(i));
    st3(f_def, i, coarse.interpolate(c_def, x));
    const double q[3] = {x.x, x.y, x.z};
    int nearest[3];
    for (int k = 0; k < 3; ++k)
      nearest[k] = clampi(int(llround((q[k] - coarse.org(k)) / coarse.voxel)), 0, coarse.dim(k) - 1);
    st3(f_eul, i, ld3(c_eul, coarse.lin(nearest[0], nearest[1], nearest[2])));
  }
}

// ============================================================================
// the cooperative flip-flop kernel
// ============================================================================

// Krylov storage of the packed Chronopoulos-Gear PCG (pcg_pk): xyz triples,
// 12 B (fp32) or 24 B (fp64) per row instead of 32-byte padded double4
template <class S>
struct AlignedOf {  // the gathered vector u stays one aligned load: double4 / float4
  using type = double4;
};
template <>
struct AlignedOf<float> {
  using type = float4;
};
template <class S>
struct PackVecs {
  S *r, *p, *s, *d, *dinv, *wpart;  // streamed row by row: packed xyz
  typename AlignedOf<S>::type* u;   // gathered by both matvec passes: aligned, not packed
  // scattered by the constraint pass (one store per incidence): aligned, so
  // each store is one sector
  typename AlignedOf<S>::type* contrib;
};

// the Chronopoulos-Gear PCG of a matrix-free level cut into
// S z-slab ranks inside the persistent kernel (pcg_slab).  Every pointer a
// rank reaches another rank through is an array entry per rank -- on one GPU
// (S virtual ranks = block groups of one cooperative launch) they point into
// one allocation; across GPUs they are peer pointers to the other GPUs'
// buffers.  The rows are cut into tiles of about equal work; a rank owns a
// contiguous range of tiles (a z-slab), and every dot product is summed
// per tile (fixed thread -> row map and block tree) and then over the tiles in
// tile order, so the result does not depend on S or on which block ran a tile.
struct SlabDev {
  int S;                           // ranks; 0 = not partitioned
  int ntiles;                      // tiles
  const int32_t* tile_row;         // ntiles + 1: tile t = rows [tile_row[t], tile_row[t + 1])
  const int32_t* rank_tile;        // S + 1: rank s owns tiles [rank_tile[s], rank_tile[s + 1])
  const int32_t* win_lo;           // S: first row of rank s's u window (own rows + halo)
  const int32_t* win_hi;           // S
  double4* const* uwin;            // S: u window of each rank, rows [win_lo[s], win_hi[s])
  const int32_t* con_ptr;          // S + 1: constraints incident to a rank's rows ...
  const int32_t* con_list;         // ... (a constraint straddling two slabs is in both lists)
  unsigned* const* ctr;            // S: per rank [0] rank arrivals, [32] halo pushes from below,
                                   //    [64] halo pushes from above, [96] reduction arrivals
  unsigned long long* const* part; // S: 2 x ntiles x 8 flag-embedded tile-partial words
  unsigned long long* const* tot;  // S: 2 x 8 flag-embedded totals
};

struct FFArgs {
  Grid g;
  int N;
  int64_t C;
  int mode;  // 0 = flip-flop, 1 = energy only, 2 = rotations only
  int level;
  // params
  double w_d, w_s, w_r, ff_rel_tol, pcg_tol;
  int ff_iters, pcg_max;
  PoseD pose;
  // rows
  const int32_t* rows;
  const int32_t* nbr;
  const uint8_t* frozen;
  // field (node indexed, the volume's AoS layout)
  double* field_def;
  double* field_eul;
  // row state: 32-byte padded 3-vectors, one 256-bit access each
  double4 *t, *x, *rhs, *r, *p, *ap, *dinv, *u, *w;  // ap holds s = A p
  double4 *z, *m0, *m1;  // pipelined PCG: z = A D s, m = D w (double-buffered)
  double4* nbuf;         // pipelined PCG: n = A m of the rows a thread leads
  unsigned long long* sync_ll;  // split-reduction totals (flag-embedded words)
  int meta_rows, meta_cons;     // pipelined matrix-free levels: metadata cached in shared memory
  int asm_smem;                 // pipelined assembled levels: row slots whose B^T B is cached in shared
                                // memory (round-major: a partial last round may stay in global), or 0
  double* state_spill;          // pipelined PCG row state in global memory (too many rows for shared), or null
  const int32_t* perm;          // pipelined matrix-free levels: row order (decreasing incidences), or null
  int pcg_variant;       // 0 pipelined (one reduction, overlapped), 1 Chronopoulos-Gear
  const double4 *crhs, *cdiag;
  double* rot;  // 9 per row
  // assembled B^T B (levels with many incidences per row)
  int assembled;
  int asm_rows_on_lanes;  // rows on lanes (large levels) vs kAsmLanes lanes per row
  const double* blk;     // N x 27 x 6 (xx xy xz yy yz zz)
  const int32_t* cols;   // N x 27
  // constraints
  const int4* c_row;     // 2 per constraint: anchor rows (-1 inactive)
  const double4* c_w;    // 2 per constraint: anchor weights
  const double4* c_g;    // g = R^T n (dense) | R^T (f - t) (sparse), coef
  const int32_t* c_kind;
  const double* target;
  const double* normal;
  const double* conf;
  const int32_t* row_ptr;
  const int4* c_pos;     // 2 per constraint: incidence slot of each corner or -1
  double4* contrib;      // E: a_k u_c per incidence slot (row-sorted)
  const int4* xitems;    // matrix-free extra work items (row, e_begin, e_end)
  int n_xitems;
  const int2* xrange;    // N: first extra item and count of each row
  double4* wpart;        // per-item partial (A v): rows first, then extra items
  // packed-storage Chronopoulos-Gear PCG of large matrix-free levels: fp32
  // (V = 2, WFK_PRECISION_FAST) or fp64 (V = 3) Krylov vectors, packed xyz
  PackVecs<float> fv;
  PackVecs<double> dv;
  int item2;  // Chronopoulos-Gear item pass with two items in flight per thread
  int cluster2;  // launched in 2-CTA clusters: one grid-barrier arrival per cluster
  SlabDev slab;  // V = 4: slab-partitioned CG
  int heavy_deal;  // pipelined matrix-free levels may deal round 0 one heavy row per warp (mf_pos)
  // outputs
  double* partials;  // 4 slots x gridDim
  unsigned* sync_count;  // grid barrier arrival counter (own 128 B line)
  unsigned* sync_gen;    // grid barrier generation (own 128 B line)
  double* sync_total;    // reduction totals published by the last arriver
  wfk_trace_entry* trace;
  int32_t* status;   // [0] trace length, [1] error bits, [2] total pcg iterations
  unsigned long long* dbg;  // per-block phase cycles (WFK_PHASE_TIMING=1), else null
  double* energy_out;
};

struct Red {
  unsigned gen = 0;  // generation of the grid barrier this block has passed
  // slab-partitioned CG: rank barriers, halo epochs and all-reduces this block
  // has passed in the launch (the counters are reset once per launch)
  unsigned sl_gen = 0, sl_epoch = 0, sl_seq = 0;
};

// Diagnostic phase clock: thread 0 of every block accumulates SM cycles per
// phase (enabled with WFK_PHASE_TIMING=1; a null sink compiles to a branch).
__device__ __forceinline__ long long sm_cycles() {
#ifdef __CUDA_ARCH__
  return clock64();
#else
  return 0;
#endif
}
struct PhaseClock {
  unsigned long long* sink;
  unsigned long long acc[16];
  long long t;
  __device__ explicit PhaseClock(unsigned long long* s, unsigned owner = 0)
      : sink((threadIdx.x == owner && s) ? s + 16 * blockIdx.x : nullptr), t(sm_cycles()) {
    for (int k = 0; k < 16; ++k) acc[k] = 0;
  }
  __device__ void lap(int k) {
    if (sink) {
      const long long n = sm_cycles();
      acc[k] += (unsigned long long)(n - t);
      t = n;
    }
  }
  __device__ void count(int k) {
    if (sink) acc[k] += 1;
  }
  __device__ ~PhaseClock() {
    if (sink)
      for (int k = 0; k < 16; ++k)
        if (acc[k]) sink[k] += acc[k];
  }
};

// Padded 3-vectors are accessed as one 32-byte-aligned unit: CUDA's double4
// is only 16-byte aligned (two 128-bit accesses, two L2 sector requests);
// through this type the compiler emits single 256-bit LDG/STG.E.ENL2.256.
struct __align__(32) D4 {
  double x, y, z, w;
};
WF_D V3 ld4(const double4* p, int64_t i) {
  const D4 v = reinterpret_cast<const D4*>(p)[i];
  return {v.x, v.y, v.z};
}
WF_D void st4(double4* p, int64_t i, V3 v) { reinterpret_cast<D4*>(p)[i] = D4{v.x, v.y, v.z, 0.0}; }
WF_D double4 ld4w(const double4* p, int64_t i) {
  const D4 v = reinterpret_cast<const D4*>(p)[i];
  return make_double4(v.x, v.y, v.z, v.w);
}
WF_D void st4w(double4* p, int64_t i, double4 v) { reinterpret_cast<D4*>(p)[i] = D4{v.x, v.y, v.z, v.w}; }

// ---- grid synchronisation of the persistent kernel -------------------------
// One arrival counter and one generation word (separate 128 B lines).  A block
// arrives with a single acq_rel atomic from thread 0 after a block barrier; the
// others poll the counter until it reaches G (gen + 1), and the last arrival
// raises the generation word (monotonically, red.max) for grid_reduce.
//
// grid_reduce fuses that barrier with a deterministic sum: every block
// publishes its partials before arriving, and ONLY the last arriving block
// reads them (fixed order, so the value does not depend on who is last),
// stores the totals and then releases the generation -- the other blocks read
// one line of totals instead of all G partials.  A partial or total slot is
// never rewritten before every block has passed the barrier that consumed it.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// monotonic release of the generation word: plain-barrier and reduction
// releases can land out of order, the word must never move backwards
__device__ __forceinline__ void atom_max_release_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_u32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// 2-CTA clusters (a.cluster2): the pair meets at a cluster barrier (release /
// acquire at cluster scope) and only cluster rank 0 arrives on the grid
// counter -- its gpu-scope release is cumulative over its partner's writes --
// so the counter sees G / 2 arrivals per generation; both CTAs poll it.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned arrivals_per_gen(const FFArgs& a) { return a.cluster2 ? gridDim.x / 2 : gridDim.x; }

__device__ __forceinline__ void grid_barrier(const FFArgs& a, Red& rs) {
  __syncthreads();
  if (a.cluster2) cluster_sync_all();
  if (threadIdx.x == 0) {
    // the arrival counter only grows (reset at launch): the last arrival of
    // generation g reads A (g + 1) - 1 (A arrivals per generation).  The
    // acq_rel arrival releases the block's writes (ordered before it by the
    // block barrier) and, for the last block, acquires everyone else's.
    const unsigned target = arrivals_per_gen(a) * (rs.gen + 1);
    const unsigned old = (a.cluster2 && cluster_rank() != 0) ? 0u : atom_add_acq_rel_u32(a.sync_count, 1u);
    if ((!a.cluster2 || cluster_rank() == 0) && old == target - 1) {
      atom_max_release_u32(a.sync_gen, rs.gen + 1);
    } else {
      // poll the arrival counter itself: the last arrival's RMW is visible
      // one L2 round trip earlier than the generation word it then writes
      while (int(ld_acquire_u32(a.sync_count) - target) < 0) {
      }
    }
  }
  rs.gen += 1;
  __syncthreads();
}

template <int NV>
__device__ __forceinline__ void grid_reduce(const FFArgs& a, Red& rs, double (&v)[NV], PhaseClock* pc = nullptr) {
  __shared__ double smem[4 * 32];
  __shared__ double bcast[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) smem[k * 32 + warp] = v[k];
  __syncthreads();
  if (pc) pc->lap(6);
  double s[NV];
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) s[k] = warp_sum(lane < nw ? smem[k * 32 + lane] : 0.0);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) a.partials[size_t(k) * gridDim.x + blockIdx.x] = s[k];
  }
  // 2-CTA clusters: the partner's partials are released to rank 0 here
  if (a.cluster2) cluster_sync_all();
  if (warp == 0) {
    unsigned last = 0;
    if (lane == 0 && (!a.cluster2 || cluster_rank() == 0))
      last = atom_add_acq_rel_u32(a.sync_count, 1u) == arrivals_per_gen(a) * (rs.gen + 1) - 1 ? 1u : 0u;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
#pragma unroll
      for (int k = 0; k < NV; ++k) s[k] = sum_partials(a.partials + size_t(k) * gridDim.x, gridDim.x);
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) a.sync_total[k] = s[k];
        atom_max_release_u32(a.sync_gen, rs.gen + 1);
      }
    } else if (lane == 0) {
      // the generation word may still lag (a plain barrier's last arrival
      // raises it after the others have left): wait until it reaches ours
      while (int(ld_acquire_u32(a.sync_gen) - (rs.gen + 1)) < 0) {
      }
    }
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < NV; ++k) bcast[k] = __ldcg(a.sync_total + k);
  }
  rs.gen += 1;
  if (pc) pc->lap(7);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = bcast[k];
  if (pc) pc->lap(13);
}

// Work distribution of the persistent kernel: chunks of 32 consecutive items
// (one per warp, coalesced) interleaved across the blocks, so even a few
// thousand rows spread over every SM instead of the first few blocks.
__device__ __forceinline__ int64_t gtid() {
  return (int64_t((threadIdx.x >> 5) * gridDim.x + blockIdx.x) << 5) + (threadIdx.x & 31);
}
__device__ __forceinline__ int64_t gstride() { return int64_t(gridDim.x) * blockDim.x; }
__device__ __forceinline__ int gwarp() { return (threadIdx.x >> 5) * gridDim.x + blockIdx.x; }
__device__ __forceinline__ int nwarps() { return (blockDim.x >> 5) * gridDim.x; }

WF_D void ld_anchors(const FFArgs& a, int64_t c, int rows[8], double w[8]) {
  const int4 r0 = a.c_row[2 * c], r1 = a.c_row[2 * c + 1];
  const double4 w0 = ld4w(a.c_w, 2 * c), w1 = ld4w(a.c_w, 2 * c + 1);
  rows[0] = r0.x; rows[1] = r0.y; rows[2] = r0.z; rows[3] = r0.w;
  rows[4] = r1.x; rows[5] = r1.y; rows[6] = r1.z; rows[7] = r1.w;
  w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
  w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
}

// E_sparse, E_dense, E_reg partials (solver.cpp:345-383)
__device__ __forceinline__ void energy_partials(const FFArgs& a, double& es, double& ed, double& er, int& bad) {
  es = ed = er = 0;
  for (int64_t c = gtid(); c < a.C; c += gstride()) {
    int rows[8];
    double w[8];
    ld_anchors(a, c, rows, w);
    V3 q{0, 0, 0};
    for (int k = 0; k < 8; ++k) {
      if (w[k] > 0 && rows[k] < 0) bad = 1;
      if (w[k] != 0 && rows[k] >= 0) q += w[k] * ld4(a.t, rows[k]);
    }
    const V3 s = a.pose.apply(q);
    const V3 f = ld3(a.target, c);
    if (a.c_kind[c] == WFK_DENSE_PLANE) {
      const double rr = dot(s - f, ld3(a.normal, c));
      ed += a.conf[c] * rr * rr;
    } else {
      es += a.conf[c] * sqnorm(s - f);
    }
  }
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const M3 ri = ld_m3(a.rot, r);
    const int node = a.rows[r];
    const V3 can_i = a.g.canonical(node);
    const V3 ti = ld4(a.t, r);
    for (int k = 0; k < 6; ++k) {
      const int j = a.nbr[int64_t(k) * a.N + r];
      if (j < 0) continue;
      const V3 can_j = a.g.canonical(a.rows[j]);
      const V3 resid = (ti - ld4(a.t, j)) - mul(ri, can_i - can_j);
      er += sqnorm(resid);
    }
  }
}

__device__ __forceinline__ wfk_energy energy(const FFArgs& a, cg::grid_group& grid, Red& rs, bool& logic_error) {
  double es, ed, er;
  int bad = 0;
  energy_partials(a, es, ed, er, bad);
  double v[4] = {es, ed, er, double(bad)};
  grid_reduce<4>(a, rs, v);
  wfk_energy e;
  e.sparse = v[0];
  e.dense = v[1];
  e.reg = v[2];
  e.total = a.w_s * e.sparse + a.w_d * e.dense + a.w_r * e.reg;
  logic_error = v[3] > 0;
  return e;
}

// matrix-free A*v, pass 1: u_c = coef (g . q_c) g | coef q_c with
// q_c = sum_k a_k v[a_k], and a_k u_c scattered to the incidence slot of each
// anchor row (row-sorted order), so pass 2 sums a contiguous range per row.
template <class Meta = std::nullptr_t>
__device__ __forceinline__ void matvec_constraints(const FFArgs& a, const double4* v, int skip = 0, const Meta* mm = nullptr) {
  const int64_t c0 = gtid() - 32 * skip;
  if (c0 < 0) return;
  int k_round = 0;
  for (int64_t c = c0; c < a.C; c += gstride() - 32 * skip, ++k_round) {
    int rows[8];
    double w[8];
    double4 gc;
    int kind;
    int4 p0, p1;
    bool cached = false;
    if constexpr (!std::is_same<Meta, std::nullptr_t>::value) {
      if (mm && mm->cons) {
        cached = true;
        const int q = k_round * int(blockDim.x) + threadIdx.x;
        const int SC = int(blockDim.x) * ((a.C + (gstride() - 32 * skip) - 1) / (gstride() - 32 * skip));
        const int4 r0 = mm->crow[q], r1 = mm->crow[SC + q];
        const double4 w0 = mm->cw[q], w1 = mm->cw[SC + q];
        rows[0] = r0.x; rows[1] = r0.y; rows[2] = r0.z; rows[3] = r0.w;
        rows[4] = r1.x; rows[5] = r1.y; rows[6] = r1.z; rows[7] = r1.w;
        w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
        w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
        gc = mm->cg[q];
        kind = mm->ckind[q];
        p0 = mm->cpos[q];
        p1 = mm->cpos[SC + q];
      }
    }
    if (!cached) {
      ld_anchors(a, c, rows, w);
      gc = ld4w(a.c_g, c);
      kind = a.c_kind[c];
      p0 = a.c_pos[2 * c];
      p1 = a.c_pos[2 * c + 1];
    }
    V3 q{0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (rows[k] >= 0) q += w[k] * ld4(v, rows[k]);
    V3 u;
    if (kind == WFK_DENSE_PLANE) {
      const V3 g{gc.x, gc.y, gc.z};
      u = (gc.w * dot(g, q)) * g;
    } else {
      u = gc.w * q;
    }
    const int pos[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pos[k] >= 0) st4(a.contrib, pos[k], w[k] * u);
  }
}

__device__ __forceinline__ V3 laplacian(const FFArgs& a, const double4* v, int r, V3 vr, V3 acc) {
  const double w2 = 2.0 * a.w_r;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const int j = a.nbr[int64_t(k) * a.N + r];
    if (j < 0) continue;
    acc += w2 * (vr - ld4(v, j));
  }
  return acc;
}

// Assembled levels: (A v)_r for every row over the 27-slot B^T B stencil,
// delivered once per row to the group leader as sink(r, v_r, (A v)_r).
//  * small levels: a group of kAsmLanes lanes per row, each lane a few of the
//    27 stencil slots (one parallel round of gathers), folding the ARAP
//    Laplacian into the six face slots, then a sub-warp shuffle tree;
//  * large levels (asm_rows_on_lanes): one row per lane over slot-major blocks.
// (Matrix-free levels: row_pass_mf, or item_pass in the Chronopoulos-Gear PCG.)
template <bool ASM, int AL = kAsmLanes, class Sink, class Sl = std::nullptr_t>
__device__ __forceinline__ void row_pass(const FFArgs& a, const double4* v, Sink& sink, int skip = 0,
                                         const Sl* sl = nullptr, const double* smb = nullptr,
                                         const int* smc = nullptr) {
  const int lane = threadIdx.x & 31;
  const double w2 = 2.0 * a.w_r;
  if (gwarp() < skip) return;  // warps reserved for the split reduction
  if (ASM && a.asm_rows_on_lanes) {
    // large assembled levels: rows on lanes, slot loop, coalesced SoA loads
    const int N = a.N;
    for (int r = int(gtid()) - 32 * skip; r < N; r += int(gstride()) - 32 * skip) {
      const V3 vr = ld4(v, r);
      if (a.frozen[r]) {
        sink(r, vr, vr);
        continue;
      }
      V3 acc{0, 0, 0};
#pragma unroll 9
      for (int s = 0; s < 27; ++s) {
        const int col = a.cols[int64_t(s) * N + r];
        if (col < 0) continue;
        const V3 x = ld4(v, col);
        const double* b = a.blk + int64_t(s) * 6 * N + r;
        const double b0 = b[0], b1 = b[N], b2 = b[2 * int64_t(N)], b3 = b[3 * int64_t(N)],
                     b4 = b[4 * int64_t(N)], b5 = b[5 * int64_t(N)];
        acc.x += b0 * x.x + b1 * x.y + b2 * x.z;
        acc.y += b1 * x.x + b3 * x.y + b4 * x.z;
        acc.z += b2 * x.x + b4 * x.y + b5 * x.z;
        if (s == 4 || s == 10 || s == 12 || s == 14 || s == 16 || s == 22) acc += w2 * (vr - x);
      }
      sink(r, vr, acc);
    }
    return;
  }
  if (ASM) {
    constexpr int L = AL, RPW = 32 / L;
    const int sub = lane % L, grp = lane / L;
    for (int base = (gwarp() - skip) * RPW; base < a.N; base += (nwarps() - skip) * RPW) {
      const int r = base + grp;
      const bool live = r < a.N;
      const bool frozen = live && a.frozen[r];
      const V3 vr = live ? ld4(v, r) : V3{0, 0, 0};
      V3 acc{0, 0, 0};
      const double* bb = a.blk + int64_t(r) * 27 * 6;
      const int* cc = a.cols + int64_t(r) * 27;
      if constexpr (!std::is_same<Sl, std::nullptr_t>::value) {
        if (smb && live) {  // the solve's blocks of this warp's rows, cached in shared memory
          const int q = sl->amat_of(r);
          if (q < a.asm_smem) {
            bb = smb + q * 27 * 6;
            cc = smc + q * 27;
          }
        }
      }
      if (live && !frozen) {
        // branch-free over the lane's slots so all of its gathers are in
        // flight at once: an absent column gathers the row itself (always
        // valid) and its terms are masked to zero
        constexpr int NS = (27 + L - 1) / L;
        int colv[NS];
        V3 xs[NS];
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int s = sub + L * i;
          colv[i] = s < 27 ? cc[s] : -1;
        }
#pragma unroll
        for (int i = 0; i < NS; ++i) xs[i] = ld4(v, colv[i] < 0 ? r : colv[i]);
#pragma unroll
        for (int i = 0; i < NS; ++i) {
          const int s = sub + L * i;
          if (s >= 27) break;
          const double mk = colv[i] < 0 ? 0.0 : 1.0;
          const V3 x = xs[i];
          const double* b = bb + s * 6;  // xx xy xz yy yz zz
          acc.x += mk * (b[0] * x.x + b[1] * x.y + b[2] * x.z);
          acc.y += mk * (b[1] * x.x + b[3] * x.y + b[4] * x.z);
          acc.z += mk * (b[2] * x.x + b[4] * x.y + b[5] * x.z);
          if (s == 4 || s == 10 || s == 12 || s == 14 || s == 16 || s == 22) acc += (mk * w2) * (vr - x);
        }
      }
#pragma unroll
      for (int o = L / 2; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
        acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
      }
      if (live && sub == 0) sink(r, vr, frozen ? vr : acc);
    }
  }
}

// finish_row (solver.cpp:240-269) + Jacobi diagonal (solver.cpp:289-294)
__device__ __forceinline__ void assemble_rows(const FFArgs& a) {
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const int node = a.rows[r];
    if (a.frozen[r]) {
      a.rhs[r] = a.t[r];
      a.dinv[r] = make_double4(1.0, 1.0, 1.0, 0.0);
      continue;
    }
    V3 rhs = ld4(a.crhs, r);
    V3 diag = ld4(a.cdiag, r);
    const M3 ri = ld_m3(a.rot, r);
    const V3 can_i = a.g.canonical(node);
    const double w2 = 2.0 * a.w_r;
    for (int k = 0; k < 6; ++k) {
      const int j = a.nbr[int64_t(k) * a.N + r];
      if (j < 0) continue;
      const V3 dij = can_i - a.g.canonical(a.rows[j]);
      diag.x += w2 * 1.0;
      diag.y += w2 * 1.0;
      diag.z += w2 * 1.0;
      rhs += a.w_r * mul(add(ri, ld_m3(a.rot, j)), dij);
      if (a.frozen[j]) rhs += w2 * ld4(a.t, j);
    }
    st4(a.rhs, r, rhs);
    st4(a.dinv, r, V3{diag.x > 1e-300 ? 1.0 / diag.x : 1.0, diag.y > 1e-300 ? 1.0 / diag.y : 1.0,
                      diag.z > 1e-300 ? 1.0 / diag.z : 1.0});
  }
}

// Matrix-free row pass, load-balanced: every row's contiguous incidence
// contributions are cut into work items of at most kItemLen entries.  Item r
// (r < N) is row r's first item and also carries the ARAP Laplacian, so its
// loads need no item record; rows with more incidences own extra items
// (stored after the first N).  Each item writes its partial (A v) to
// wpart[item]; the update phase adds a row's items in order, and the w.u dot
// is accumulated per item (it is linear), so no row waits on a long list.
WF_D V3 ldf3(const float* p, int64_t i) { return {double(p[3 * i]), double(p[3 * i + 1]), double(p[3 * i + 2])}; }
WF_D void stf3(float* p, int64_t i, V3 v) {
  p[3 * i] = float(v.x);
  p[3 * i + 1] = float(v.y);
  p[3 * i + 2] = float(v.z);
}
WF_D V3 rnd3(V3 v) { return {double(float(v.x)), double(float(v.y)), double(float(v.z))}; }
// storage-generic access for the two-in-flight item pass: fp64 padded 32-byte
// vectors (double4) or fp32 packed xyz (float)
WF_D V3 ldv(const double4* p, int64_t i) { return ld4(p, i); }
WF_D V3 ldv(const float* p, int64_t i) { return ldf3(p, i); }
WF_D V3 ldv(const double* p, int64_t i) { return {p[3 * i], p[3 * i + 1], p[3 * i + 2]}; }
WF_D void stv(double4* p, int64_t i, V3 v) { st4(p, i, v); }
WF_D void stv(float* p, int64_t i, V3 v) { stf3(p, i, v); }
WF_D void stv(double* p, int64_t i, V3 v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}
WF_D V3 sink_round(const double4*, V3 v) { return v; }
WF_D V3 sink_round(const float*, V3 v) { return rnd3(v); }
WF_D V3 sink_round(const double*, V3 v) { return v; }
WF_D V3 ldv(const float4* p, int64_t i) {
  const float4 f = p[i];
  return {double(f.x), double(f.y), double(f.z)};
}
WF_D void stv(float4* p, int64_t i, V3 v) { p[i] = make_float4(float(v.x), float(v.y), float(v.z), 0.f); }
WF_D V3 sink_round(const float4*, V3 v) { return rnd3(v); }
template <class Sink>
__device__ __forceinline__ void item_pass(const FFArgs& a, const double4* v, Sink& sink) {
  const double w2 = 2.0 * a.w_r;
  const int total = a.N + a.n_xitems;
  for (int i = int(gtid()); i < total; i += int(gstride())) {
    int r, e0, e1;
    bool first;
    if (i < a.N) {
      r = i;
      e0 = a.row_ptr[r];
      e1 = min(a.row_ptr[r + 1], e0 + kItemLen);
      first = true;
    } else {
      const int4 it = a.xitems[i - a.N];
      r = it.x;
      e0 = it.y;
      e1 = it.z;
      first = false;
    }
    const V3 vr = ld4(v, r);
    V3 acc{0, 0, 0};
    if (first && a.frozen[r]) {
      acc = vr;  // frozen rows: A = I (solver.cpp:241-246); they carry no incidences
    } else {
#pragma unroll 4
      for (int e = e0; e < e1; ++e) acc += ld4(a.contrib, e);
      if (first) {
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          const int j = a.nbr[int64_t(k) * a.N + r];
          if (j >= 0) acc += w2 * (vr - ld4(v, j));
        }
      }
    }
    st4(a.wpart, i, acc);
    sink(r, vr, acc);
  }
}

// (A v)_r of one row from its items (fixed order)
WF_D V3 row_from_items(const FFArgs& a, int r) {
  V3 acc = ld4(a.wpart, r);
  const int2 xr = a.xrange[r];
  for (int i = 0; i < xr.y; ++i) acc += ld4(a.wpart, a.N + xr.x + i);
  return acc;
}

// ---- WFK_PRECISION_FAST: the Chronopoulos-Gear PCG with fp32 vectors --------
// Only for matrix-free levels too large for shared memory, which are
// HBM-bound (configs[4]: 3.6 M rows, ~580 B per row per iteration in fp64 with
// 32-byte padded vectors).  Storage of r, u, p, s = A p, the solution
// increment d = x - x0, D^-1, the constraint contributions and the item
// partials is fp32 packed xyz (12 B); every multiply / add, the three dot
// products and the initial residual r0 = b - A x0 stay fp64, and x = x0 + d
// is formed in fp64 at the end, so the rounding is relative to the update,
// not to the absolute positions.
// matvec pass 1 (see matvec_constraints) on a packed vector
template <class VT, class S>
__device__ __forceinline__ void matvec_constraints_pk(const FFArgs& a, const VT* v, S* contrib) {
  for (int64_t c = gtid(); c < a.C; c += gstride()) {
    int rows[8];
    double w[8];
    ld_anchors(a, c, rows, w);
    const double4 gc = ld4w(a.c_g, c);
    V3 q{0, 0, 0};
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (rows[k] >= 0) q += w[k] * ldv(v, rows[k]);
    V3 u;
    if (a.c_kind[c] == WFK_DENSE_PLANE) {
      const V3 g{gc.x, gc.y, gc.z};
      u = (gc.w * dot(g, q)) * g;
    } else {
      u = gc.w * q;
    }
    const int4 p0 = a.c_pos[2 * c], p1 = a.c_pos[2 * c + 1];
    const int pos[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (pos[k] >= 0) stv(contrib, pos[k], w[k] * u);
  }
}
// matvec pass 2 (see item_pass) on an fp32 vector, two items in flight per
// thread: at ~47 items per thread (3.6 M rows) the pass is a chain of
// dependent loads (item -> neighbour table -> gathers), so every load of both
// items is issued before any of their arithmetic.
template <class VT, class CT, class WT, class Sink>
__device__ __forceinline__ void item_pass2(const FFArgs& a, const VT* v, CT* contrib, WT* wpart, Sink& sink) {
  const double w2 = 2.0 * a.w_r;
  const int total = a.N + a.n_xitems;
  const int st = int(gstride());
  for (int i0 = int(gtid()); i0 < total; i0 += 2 * st) {
    int r[2], e0[2], e1[2], nb[2][6];
    bool live[2], first[2], frz[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = i0 + h * st;
      live[h] = i < total;
      first[h] = live[h] && i < a.N;
      r[h] = 0;
      e0[h] = e1[h] = 0;
      frz[h] = false;
#pragma unroll
      for (int k = 0; k < 6; ++k) nb[h][k] = -1;
      if (!live[h]) continue;
      if (first[h]) {
        r[h] = i;
        e0[h] = a.row_ptr[i];
        e1[h] = min(a.row_ptr[i + 1], e0[h] + kItemLen);
        frz[h] = a.frozen[i];
#pragma unroll
        for (int k = 0; k < 6; ++k) nb[h][k] = a.nbr[int64_t(k) * a.N + i];
      } else {
        const int4 it = a.xitems[i - a.N];
        r[h] = it.x;
        e0[h] = it.y;
        e1[h] = it.z;
      }
    }
    // item_pass's order: the contributions in incidence order, then the six
    // Laplacian terms in face order (bit-identical fp64 results); the two
    // items' loads are interleaved step by step
    V3 vr[2], acc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      vr[h] = live[h] ? ldv(v, r[h]) : V3{0, 0, 0};
      acc[h] = V3{0, 0, 0};
      if (live[h] && !(first[h] && frz[h]))
        for (int e = e0[h]; e < e1[h]; ++e) acc[h] += ldv(contrib, e);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (first[h] && !frz[h] && nb[h][k] >= 0) acc[h] += w2 * (vr[h] - ldv(v, nb[h][k]));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!live[h]) continue;
      if (first[h] && frz[h]) acc[h] = vr[h];  // frozen rows: A = I (solver.cpp:241-246)
      stv(wpart, i0 + h * st, acc[h]);
      sink(r[h], vr[h], sink_round(v, acc[h]));
    }
  }
}
template <class S>
WF_D V3 row_from_items_pk(const FFArgs& a, const S* wpart, int r) {
  V3 acc = ldv(wpart, r);
  const int2 xr = a.xrange[r];
  for (int i = 0; i < xr.y; ++i) acc += ldv(wpart, a.N + xr.x + i);
  return acc;
}
template <class S>
WF_D V3 rnd_s(V3 v) {
  if constexpr (std::is_same<S, float>::value)
    return rnd3(v);
  else
    return v;
}
template <class S>
__device__ __forceinline__ const PackVecs<S>& pack_of(const FFArgs& a) {
  if constexpr (std::is_same<S, float>::value)
    return a.fv;
  else
    return a.dv;
}
template <class S>
__device__ void pcg_pk(const FFArgs& a, Red& rs, int& iters, double& relres) {
  const PackVecs<S>& pv = pack_of<S>(a);
  iters = 0;
  relres = 0;
  PhaseClock pc(a.dbg);
  auto none = [](int, V3, V3) {};
  // r0 = b - A x0 in fp64 (the fp64 matvec of x0), then rounded into storage
  double acc_rr = 0, acc_bb = 0;
  matvec_constraints(a, a.x);
  grid_barrier(a, rs);
  item_pass(a, a.x, none);
  grid_barrier(a, rs);
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const V3 b = ld4(a.rhs, r);
    const V3 rr = rnd_s<S>(b - row_from_items(a, r));
    const V3 d = rnd_s<S>(ld4(a.dinv, r));
    stv(pv.r, r, rr);
    stv(pv.dinv, r, d);
    stv(pv.u, r, cmul(d, rr));
    stv(pv.p, r, V3{0, 0, 0});
    stv(pv.s, r, V3{0, 0, 0});
    stv(pv.d, r, V3{0, 0, 0});
    acc_rr += dot(rr, rr);
    acc_bb += sqnorm(b);
  }
  grid_barrier(a, rs);
  // w0 = A u0
  double v4[4] = {0, 0, acc_rr, acc_bb};
  matvec_constraints_pk(a, pv.u, pv.contrib);
  grid_barrier(a, rs);
  auto w_sink = [&](int, V3 ur, V3 wpart) { v4[1] += dot(wpart, ur); };
  item_pass2(a, pv.u, pv.contrib, pv.wpart, w_sink);
  for (int r = int(gtid()); r < a.N; r += int(gstride())) v4[0] += dot(ldv(pv.r, r), ldv(pv.u, r));
  grid_reduce<4>(a, rs, v4);
  double gamma = v4[0], delta = v4[1];
  double r_norm = sqrt(v4[2]);
  const double b_norm = sqrt(v4[3]);
  if (b_norm == 0) {
    for (int r = int(gtid()); r < a.N; r += int(gstride())) st4(a.x, r, V3{0, 0, 0});
    grid_barrier(a, rs);
    return;
  }
  relres = r_norm / b_norm;
  const double stop = fmax(a.pcg_tol * r_norm, 1e-13 * b_norm);
  double gamma_prev = 0, alpha_prev = 0;
  pc.lap(12);
  for (int it = 0; it < a.pcg_max && r_norm > stop; ++it) {
    const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
    const double pap = it == 0 ? delta : delta - beta * gamma / alpha_prev;
    if (pap <= 0) break;  // solver.cpp:327
    const double alpha = gamma / pap;
    double v3[3] = {0, 0, 0};
    // one row per thread in flight here: two (as in item_pass_f32) spill at
    // 512 threads and measured slower (U 238 K vs 205 K cycles per level-0 iteration)
    for (int r = int(gtid()); r < a.N; r += int(gstride())) {
      const V3 w = row_from_items_pk(a, static_cast<const S*>(pv.wpart), r);
      const V3 p = rnd_s<S>(ldv(pv.u, r) + beta * ldv(pv.p, r));
      const V3 sv = rnd_s<S>(w + beta * ldv(pv.s, r));
      const V3 d = ldv(pv.d, r) + alpha * p;
      const V3 rr = rnd_s<S>(ldv(pv.r, r) - alpha * sv);
      const V3 u = rnd_s<S>(cmul(ldv(pv.dinv, r), rr));
      stv(pv.p, r, p);
      stv(pv.s, r, sv);
      stv(pv.d, r, d);
      stv(pv.r, r, rr);
      stv(pv.u, r, u);
      v3[0] += dot(rr, u);
      v3[2] += dot(rr, rr);
    }
    pc.lap(4);
    grid_barrier(a, rs);
    pc.lap(5);
    matvec_constraints_pk(a, pv.u, pv.contrib);
    pc.lap(0);
    grid_barrier(a, rs);
    pc.lap(1);
    auto w_sink2 = [&](int, V3 ur, V3 wpart) { v3[1] += dot(wpart, ur); };
    item_pass2(a, pv.u, pv.contrib, pv.wpart, w_sink2);
    pc.lap(2);
    grid_reduce<3>(a, rs, v3, &pc);
    pc.lap(3);
    pc.count(15);
    gamma_prev = gamma;
    alpha_prev = alpha;
    gamma = v3[0];
    delta = v3[1];
    r_norm = sqrt(v3[2]);
    relres = r_norm / b_norm;
    iters = it + 1;
  }
  // x = x0 + d in fp64 (a.x still holds x0 = t)
  for (int r = int(gtid()); r < a.N; r += int(gstride())) st4(a.x, r, ld4(a.x, r) + ldv(pv.d, r));
  grid_barrier(a, rs);
}

// pcg_solve (solver.cpp:282-343) in the Chronopoulos-Gear arrangement: the
// same Krylov iterates (p = u + beta p, x += alpha p, r -= alpha A p with
// u = D^-1 r, alpha = r.u / p.Ap, beta = r.u / r.u_prev), but s = A p and
// w = A u are carried as vectors, so p.Ap = w.u - beta r.u / alpha_prev and
// every iteration needs ONE grid reduction {r.u, w.u, r.r}:
//   U  w from its items, p, s, x, r, u update (own rows)  -> barrier
//   A  constraint pass of A u (matrix-free levels only)    -> barrier
//   B  item pass (matrix-free) | row pass (assembled)      -> reduction
// The stopping rule, breakdown test and iteration count are the reference's.
// ---- slab-partitioned CG (V = 4) ---------------------------------------------
// pcg_pk<double> with the rows cut into S ranks.  Per iteration a rank
//   U: updates the rows of its tiles; writes u into its own window and pushes
//      the rows a neighbour's window covers into that neighbour's window;
//      writes the tile partials (r.u, r.r) into every rank's partial array;
//   signals "pushed" to both neighbours and waits for its own blocks and for
//      both neighbours' pushes (no grid barrier);
//   A: the constraint pass over the constraints incident to its rows (spread
//      over all of the rank's threads), writing only its own rows' incidence
//      slots (straddling constraints are evaluated by both ranks, identically);
//   rank barrier;
//   B: the item pass over its tiles' items (u of halo rows from its window);
//      tile partials (w.u) into every rank's array;
//   all-reduce: every block arrives on every rank's counter; each rank's first
//      block sums the tile partials in tile order and publishes the totals.
// Scopes are gpu (one GPU); a multi-GPU build uses the same code at sys scope.
struct SlabRank {
  int s, S, G, b0, nb;  // rank, ranks, blocks, first block, blocks of the rank
  int t0, t1;           // own tiles
  int lo, hi, wlo;      // own rows, window start
  double4* uw;          // own window
};
__device__ __forceinline__ int slab_bstart(int s, int S, int G) { return int((int64_t(s) * G) / S); }
__device__ __forceinline__ SlabRank slab_rank(const FFArgs& a) {
  SlabRank k;
  k.S = a.slab.S;
  k.G = gridDim.x;
  int s = int((int64_t(blockIdx.x) * k.S) / k.G);
  while (s + 1 < k.S && slab_bstart(s + 1, k.S, k.G) <= int(blockIdx.x)) ++s;
  while (s > 0 && slab_bstart(s, k.S, k.G) > int(blockIdx.x)) --s;
  k.s = s;
  k.b0 = slab_bstart(s, k.S, k.G);
  k.nb = slab_bstart(s + 1, k.S, k.G) - k.b0;
  k.t0 = a.slab.rank_tile[s];
  k.t1 = a.slab.rank_tile[s + 1];
  k.lo = a.slab.tile_row[k.t0];
  k.hi = a.slab.tile_row[k.t1];
  k.wlo = a.slab.win_lo[s];
  k.uw = a.slab.uwin[s];
  return k;
}
__device__ __forceinline__ void red_add_release_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void slab_wait_ge(const unsigned* p, unsigned target) {
  while (int(ld_acquire_u32(p) - target) < 0) {
  }
}
// u of row r as rank k sees it: its own rows and halo rows, all in its window
WF_D V3 slab_u(const SlabRank& k, int r) { return ld4(k.uw, r - k.wlo); }
// store u of an own row: own window, and every neighbour window covering it
__device__ __forceinline__ void slab_put_u(const FFArgs& a, const SlabRank& k, int r, V3 u) {
  st4(k.uw, r - k.wlo, u);
  if (k.s > 0 && r < a.slab.win_hi[k.s - 1]) st4(a.slab.uwin[k.s - 1], r - a.slab.win_lo[k.s - 1], u);
  if (k.s + 1 < k.S && r >= a.slab.win_lo[k.s + 1]) st4(a.slab.uwin[k.s + 1], r - a.slab.win_lo[k.s + 1], u);
}
// this block's arrival at its rank, and (after u pushes) at both neighbours
__device__ __forceinline__ void slab_sync(const FFArgs& a, const SlabRank& k, unsigned& gen, bool halo,
                                          unsigned& epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (halo) {
      if (k.s > 0) red_add_release_u32(a.slab.ctr[k.s - 1] + 64, 1u);
      if (k.s + 1 < k.S) red_add_release_u32(a.slab.ctr[k.s + 1] + 32, 1u);
    }
    red_add_release_u32(a.slab.ctr[k.s], 1u);
    slab_wait_ge(a.slab.ctr[k.s], unsigned(k.nb) * (gen + 1));
    if (halo) {
      if (k.s > 0) {
        const int nbl = k.b0 - slab_bstart(k.s - 1, k.S, k.G);
        slab_wait_ge(a.slab.ctr[k.s] + 32, unsigned(nbl) * (epoch + 1));
      }
      if (k.s + 1 < k.S) {
        const int nbu = slab_bstart(k.s + 2, k.S, k.G) - slab_bstart(k.s + 1, k.S, k.G);
        slab_wait_ge(a.slab.ctr[k.s] + 64, unsigned(nbu) * (epoch + 1));
      }
    }
  }
  gen += 1;
  if (halo) epoch += 1;
  __syncthreads();
}
// Tile partials: after each tile every warp reduces its lanes' sums (fixed
// butterfly) into a shared slot; after a batch of tiles one block barrier,
// then the warps' sums of each tile are added in warp order (fixed) and
// written as words 2j, 2j + 1 of the tile into every rank's partial array
// (tag seq + 1).  No block barrier between the tiles of a batch.
constexpr int kSlabBatch = 16;
struct SlabTileSm {
  double v[kSlabBatch][32][4];
};
template <int NV>
__device__ __forceinline__ void slab_tile_stash(SlabTileSm& sm, int tl, double (&v)[NV]) {
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const double w = warp_sum(v[j]);
    if ((threadIdx.x & 31) == 0) sm.v[tl][threadIdx.x >> 5][j] = w;
  }
}
template <int NV>
__device__ __forceinline__ void slab_tile_flush(const FFArgs& a, const SlabRank& k, SlabTileSm& sm, int n, int t_first,
                                                const int (&slot)[NV], unsigned seq) {
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int idx = threadIdx.x; idx < n * NV; idx += blockDim.x) {
    const int tl = idx / NV, j = idx % NV;
    double v = 0;
    for (int w = 0; w < nw; ++w) v += sm.v[tl][w][j];
    const int t = t_first + tl * k.nb;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const size_t off = (size_t(seq & 1) * a.slab.ntiles + size_t(t)) * 8 + 2 * slot[j];
    const unsigned long long w0 = (unsigned long long)unsigned(bits) << 32 | (seq + 1u);
    const unsigned long long w1 = (bits >> 32) << 32 | (seq + 1u);
    for (int d = 0; d < k.S; ++d) {
      st_relaxed_u64(a.slab.part[d] + off, w0);
      st_relaxed_u64(a.slab.part[d] + off + 1, w1);
    }
  }
  __syncthreads();
}
// runs f(t, r0, r1, v) over this block's tiles with per-tile partials v[NV]
template <int NV, class F>
__device__ __forceinline__ void slab_for_tiles(const FFArgs& a, const SlabRank& k, SlabTileSm& sm,
                                               const int (&slot)[NV], unsigned seq, F f) {
  int tl = 0, t_first = k.t0 + (int(blockIdx.x) - k.b0);
  for (int t = t_first; t < k.t1; t += k.nb) {
    const int r0 = a.slab.tile_row[t], r1 = a.slab.tile_row[t + 1];
    double v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = 0;
    f(r0, r1, v);
    slab_tile_stash<NV>(sm, tl, v);
    if (++tl == kSlabBatch) {
      slab_tile_flush<NV>(a, k, sm, tl, t_first, slot, seq);
      t_first += kSlabBatch * k.nb;
      tl = 0;
    }
  }
  if (tl) slab_tile_flush<NV>(a, k, sm, tl, t_first, slot, seq);
}
// all-reduce of NV values over every tile, tile order
template <int NV>
__device__ __forceinline__ void slab_allreduce(const FFArgs& a, const SlabRank& k, double (&v)[NV], unsigned seq) {
  __shared__ double smem[4 * 32];
  __shared__ double bc[4];
  __syncthreads();  // every tile word of this block is written
  if (threadIdx.x == 0)
    for (int d = 0; d < k.S; ++d) red_add_release_u32(a.slab.ctr[d] + 96, 1u);
  if (int(blockIdx.x) == k.b0) {
    // the rank's first block: every block's tiles in, then the fixed-order sum
    // (thread i: tiles i, i + blockDim, ... in order; then the block tree)
    if (threadIdx.x == 0) slab_wait_ge(a.slab.ctr[k.s] + 96, unsigned(k.G) * (seq + 1));
    __syncthreads();
    const unsigned long long* pw = a.slab.part[k.s] + size_t(seq & 1) * a.slab.ntiles * 8;
    double t[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) t[j] = 0;
    for (int tile = threadIdx.x; tile < a.slab.ntiles; tile += blockDim.x) {
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const unsigned long long lo_w = ld_relaxed_u64(pw + size_t(tile) * 8 + 2 * j);
        const unsigned long long hi_w = ld_relaxed_u64(pw + size_t(tile) * 8 + 2 * j + 1);
        t[j] += __longlong_as_double((long long)((hi_w >> 32) << 32 | (lo_w >> 32)));
      }
    }
    block_sum<NV>(t, smem);
    if (threadIdx.x < 2 * NV) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(t[threadIdx.x >> 1]);
      const unsigned half = (threadIdx.x & 1) ? unsigned(bits >> 32) : unsigned(bits);
      st_relaxed_u64(a.slab.tot[k.s] + size_t(seq & 1) * 8 + threadIdx.x, (unsigned long long)half << 32 | (seq + 1u));
    }
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned half = 0;
    if (lane < 2 * NV) {
      const unsigned long long* w = a.slab.tot[k.s] + size_t(seq & 1) * 8 + lane;
      unsigned long long x;
      do {
        x = ld_relaxed_u64(w);
      } while (unsigned(x) != seq + 1u);
      half = unsigned(x >> 32);
    }
    const unsigned hi = __shfl_down_sync(0xffffffffu, half, 1);
    if (lane < 2 * NV && !(lane & 1)) bc[lane >> 1] = __longlong_as_double((long long)((unsigned long long)hi << 32 | half));
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) v[j] = bc[j];
}
// constraint pass of rank k over its constraint list on u (window) or on a
// complete global vector (x0: xg), writing only its own rows' incidence slots
__device__ __forceinline__ void slab_cons(const FFArgs& a, const SlabRank& k, const double4* xg, double4* contrib) {
  const int c0 = a.slab.con_ptr[k.s], c1 = a.slab.con_ptr[k.s + 1];
  const int t0 = (int(blockIdx.x) - k.b0) * blockDim.x + threadIdx.x, nt = k.nb * blockDim.x;
  for (int i = c0 + t0; i < c1; i += nt) {
    const int64_t c = a.slab.con_list[i];
    int rows[8];
    double w[8];
    ld_anchors(a, c, rows, w);
    const double4 gc = ld4w(a.c_g, c);
    V3 q{0, 0, 0};
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (rows[j] >= 0) q += w[j] * (xg ? ld4(xg, rows[j]) : slab_u(k, rows[j]));
    V3 u;
    if (a.c_kind[c] == WFK_DENSE_PLANE) {
      const V3 g{gc.x, gc.y, gc.z};
      u = (gc.w * dot(g, q)) * g;
    } else {
      u = gc.w * q;
    }
    const int4 p0 = a.c_pos[2 * c], p1 = a.c_pos[2 * c + 1];
    const int pos[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (pos[j] >= 0 && rows[j] >= k.lo && rows[j] < k.hi) st4(contrib, pos[j], w[j] * u);
  }
}
// item pass over one tile's items: its rows' first items, then their extra
// items (contiguous); item_pass's arithmetic and order, two items per thread
// in flight (item_pass2)
template <class Sink>
__device__ __forceinline__ void slab_items(const FFArgs& a, const SlabRank& k, int r0, int r1, const double4* xg,
                                           const double4* contrib, double* wpart, Sink& sink) {
  if (r1 <= r0) return;
  const int x0 = a.xrange[r0].x, x1 = a.xrange[r1 - 1].x + a.xrange[r1 - 1].y;
  const int nfirst = r1 - r0, total = nfirst + (x1 - x0);
  const double w2 = 2.0 * a.w_r;
  const int st = blockDim.x;
  auto uof = [&](int r) { return xg ? ld4(xg, r) : slab_u(k, r); };
  for (int j0 = threadIdx.x; j0 < total; j0 += 2 * st) {
    int r[2], e0[2], e1[2], item[2], nb[2][6];
    bool live[2], first[2], frz[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + h * st;
      live[h] = j < total;
      first[h] = live[h] && j < nfirst;
      r[h] = r0;
      e0[h] = e1[h] = 0;
      item[h] = 0;
      frz[h] = false;
#pragma unroll
      for (int f = 0; f < 6; ++f) nb[h][f] = -1;
      if (!live[h]) continue;
      if (first[h]) {
        r[h] = r0 + j;
        item[h] = r[h];
        e0[h] = a.row_ptr[r[h]];
        e1[h] = min(a.row_ptr[r[h] + 1], e0[h] + kItemLen);
        frz[h] = a.frozen[r[h]];
#pragma unroll
        for (int f = 0; f < 6; ++f) nb[h][f] = a.nbr[int64_t(f) * a.N + r[h]];
      } else {
        item[h] = a.N + x0 + (j - nfirst);
        const int4 it = a.xitems[x0 + (j - nfirst)];
        r[h] = it.x;
        e0[h] = it.y;
        e1[h] = it.z;
      }
    }
    V3 vr[2], acc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      vr[h] = live[h] ? uof(r[h]) : V3{0, 0, 0};
      acc[h] = V3{0, 0, 0};
      if (live[h] && !(first[h] && frz[h]))
        for (int e = e0[h]; e < e1[h]; ++e) acc[h] += ld4(contrib, e);
    }
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (first[h] && !frz[h] && nb[h][f] >= 0) acc[h] += w2 * (vr[h] - uof(nb[h][f]));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!live[h]) continue;
      if (first[h] && frz[h]) acc[h] = vr[h];  // frozen rows: A = I (solver.cpp:241-246)
      stv(wpart, item[h], acc[h]);
      sink(r[h], vr[h], acc[h]);
    }
  }
}
__device__ void pcg_slab(const FFArgs& a, Red& rs, int& iters, double& relres) {
  const PackVecs<double>& pv = a.dv;
  const SlabRank k = slab_rank(a);
  unsigned& gen = rs.sl_gen;
  unsigned& epoch = rs.sl_epoch;
  unsigned& seq = rs.sl_seq;
  iters = 0;
  relres = 0;
  PhaseClock pc(a.dbg);
  auto none = [](int, V3, V3) {};
  __shared__ SlabTileSm tsm;
  // r0 = b - A x0 (x0 = t, complete on every rank); u0 = D r0; tile partials
  // r.u (slot 0), r.r (2), b.b (3) now, w.u (1) after the matvec of u0
  slab_cons(a, k, a.x, pv.contrib);
  slab_sync(a, k, gen, false, epoch);
  for (int t = k.t0 + (int(blockIdx.x) - k.b0); t < k.t1; t += k.nb) {
    slab_items(a, k, a.slab.tile_row[t], a.slab.tile_row[t + 1], a.x, pv.contrib, pv.wpart, none);
  }
  __syncthreads();
  {
    const int slots[3] = {0, 2, 3};
    slab_for_tiles<3>(a, k, tsm, slots, seq, [&](int r0, int r1, double (&v)[3]) {
      for (int r = r0 + int(threadIdx.x); r < r1; r += blockDim.x) {
        const V3 b = ld4(a.rhs, r);
        const V3 rr = b - row_from_items_pk(a, static_cast<const double*>(pv.wpart), r);
        const V3 d = ld4(a.dinv, r);
        const V3 u = cmul(d, rr);
        stv(pv.r, r, rr);
        stv(pv.dinv, r, d);
        slab_put_u(a, k, r, u);
        stv(pv.p, r, V3{0, 0, 0});
        stv(pv.s, r, V3{0, 0, 0});
        stv(pv.d, r, V3{0, 0, 0});
        v[0] += dot(rr, u);
        v[1] += dot(rr, rr);
        v[2] += sqnorm(b);
      }
    });
  }
  slab_sync(a, k, gen, true, epoch);
  // w0 = A u0
  slab_cons(a, k, nullptr, pv.contrib);
  slab_sync(a, k, gen, false, epoch);
  {
    const int slots[1] = {1};
    slab_for_tiles<1>(a, k, tsm, slots, seq, [&](int r0, int r1, double (&v)[1]) {
      auto w_sink = [&](int, V3 ur, V3 wpart) { v[0] += dot(wpart, ur); };
      slab_items(a, k, r0, r1, nullptr, pv.contrib, pv.wpart, w_sink);
    });
  }
  double v4[4];
  slab_allreduce<4>(a, k, v4, seq++);
  double gamma = v4[0], delta = v4[1];
  double r_norm = sqrt(v4[2]);
  const double b_norm = sqrt(v4[3]);
  if (b_norm == 0) {
    for (int r = k.lo + (int(blockIdx.x) - k.b0) * int(blockDim.x) + int(threadIdx.x); r < k.hi;
         r += k.nb * int(blockDim.x))
      st4(a.x, r, V3{0, 0, 0});
    grid_barrier(a, rs);
    return;
  }
  relres = r_norm / b_norm;
  const double stop = fmax(a.pcg_tol * r_norm, 1e-13 * b_norm);
  double gamma_prev = 0, alpha_prev = 0;
  pc.lap(12);
  for (int it = 0; it < a.pcg_max && r_norm > stop; ++it) {
    const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
    const double pap = it == 0 ? delta : delta - beta * gamma / alpha_prev;
    if (pap <= 0) break;  // solver.cpp:327
    const double alpha = gamma / pap;
    {
      const int slots[2] = {0, 2};
      slab_for_tiles<2>(a, k, tsm, slots, seq, [&](int r0, int r1, double (&v)[2]) {
        for (int r = r0 + int(threadIdx.x); r < r1; r += blockDim.x) {
          const V3 w = row_from_items_pk(a, static_cast<const double*>(pv.wpart), r);
          const V3 p = slab_u(k, r) + beta * ldv(pv.p, r);
          const V3 sv = w + beta * ldv(pv.s, r);
          const V3 d = ldv(pv.d, r) + alpha * p;
          const V3 rr = ldv(pv.r, r) - alpha * sv;
          const V3 u = cmul(ldv(pv.dinv, r), rr);
          stv(pv.p, r, p);
          stv(pv.s, r, sv);
          stv(pv.d, r, d);
          stv(pv.r, r, rr);
          v[0] += dot(rr, u);
          v[1] += dot(rr, rr);
          slab_put_u(a, k, r, u);
        }
      });
    }
    pc.lap(4);
    slab_sync(a, k, gen, true, epoch);
    pc.lap(5);
    slab_cons(a, k, nullptr, pv.contrib);
    pc.lap(0);
    slab_sync(a, k, gen, false, epoch);
    pc.lap(1);
    {
      const int slots[1] = {1};
      slab_for_tiles<1>(a, k, tsm, slots, seq, [&](int r0, int r1, double (&v)[1]) {
        auto w_sink2 = [&](int, V3 ur, V3 wpart) { v[0] += dot(wpart, ur); };
        slab_items(a, k, r0, r1, nullptr, pv.contrib, pv.wpart, w_sink2);
      });
    }
    pc.lap(2);
    double v3[3];
    slab_allreduce<3>(a, k, v3, seq++);
    pc.lap(3);
    pc.count(15);
    gamma_prev = gamma;
    alpha_prev = alpha;
    gamma = v3[0];
    delta = v3[1];
    r_norm = sqrt(v3[2]);
    relres = r_norm / b_norm;
    iters = it + 1;
  }
  // x = x0 + d of the rank's rows, then every rank's rows are in x
  for (int r = k.lo + (int(blockIdx.x) - k.b0) * int(blockDim.x) + int(threadIdx.x); r < k.hi;
       r += k.nb * int(blockDim.x))
    st4(a.x, r, ld4(a.x, r) + ldv(pv.d, r));
  grid_barrier(a, rs);
}

template <bool ASM>
__device__ void pcg(const FFArgs& a, cg::grid_group& grid, Red& rs, int& iters, double& relres) {
  iters = 0;
  relres = 0;
  PhaseClock pc(a.dbg);
  auto none = [](int, V3, V3) {};
  // r0 = b - A x0, u0 = D^-1 r0 (solver.cpp:305-310)
  double acc_rr = 0, acc_bb = 0;
  auto init_row = [&](int r, V3 ax) {
    const V3 b = ld4(a.rhs, r);
    const V3 rr = b - ax;
    st4(a.r, r, rr);
    st4(a.u, r, cmul(ld4(a.dinv, r), rr));
    a.p[r] = make_double4(0, 0, 0, 0);
    a.ap[r] = make_double4(0, 0, 0, 0);
    acc_rr += dot(rr, rr);
    acc_bb += sqnorm(b);
  };
  if (ASM) {
    auto init_sink = [&](int r, V3, V3 ax) { init_row(r, ax); };
    row_pass<true>(a, a.x, init_sink);
  } else {
    matvec_constraints(a, a.x);
    grid_barrier(a, rs);
    item_pass(a, a.x, none);
    grid_barrier(a, rs);
    for (int r = int(gtid()); r < a.N; r += int(gstride())) init_row(r, row_from_items(a, r));
  }
  grid_barrier(a, rs);
  // w0 = A u0
  double v4[4] = {0, 0, acc_rr, acc_bb};
  if (ASM) {
    auto w_sink = [&](int r, V3 ur, V3 wr) {
      st4(a.w, r, wr);
      v4[0] += dot(ld4(a.r, r), ur);
      v4[1] += dot(wr, ur);
    };
    row_pass<true>(a, a.u, w_sink);
  } else {
    matvec_constraints(a, a.u);
    grid_barrier(a, rs);
    auto w_sink = [&](int, V3 ur, V3 wpart) { v4[1] += dot(wpart, ur); };
    item_pass(a, a.u, w_sink);
    for (int r = int(gtid()); r < a.N; r += int(gstride())) v4[0] += dot(ld4(a.r, r), ld4(a.u, r));
  }
  grid_reduce<4>(a, rs, v4);
  double gamma = v4[0], delta = v4[1];
  double r_norm = sqrt(v4[2]);
  const double b_norm = sqrt(v4[3]);
  if (b_norm == 0) {
    for (int r = int(gtid()); r < a.N; r += int(gstride())) st4(a.x, r, V3{0, 0, 0});
    grid_barrier(a, rs);
    return;
  }
  relres = r_norm / b_norm;
  const double stop = fmax(a.pcg_tol * r_norm, 1e-13 * b_norm);
  double gamma_prev = 0, alpha_prev = 0;
  pc.lap(12);
  for (int it = 0; it < a.pcg_max && r_norm > stop; ++it) {
    const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
    const double pap = it == 0 ? delta : delta - beta * gamma / alpha_prev;
    if (pap <= 0) break;  // solver.cpp:327
    const double alpha = gamma / pap;
    double v3[3] = {0, 0, 0};
    for (int r = int(gtid()); r < a.N; r += int(gstride())) {
      const V3 w = ASM ? ld4(a.w, r) : row_from_items(a, r);
      const double4 u4 = ld4w(a.u, r), p4 = ld4w(a.p, r), s4 = ld4w(a.ap, r), x4 = ld4w(a.x, r), r4 = ld4w(a.r, r),
                    d4 = ld4w(a.dinv, r);
      const V3 p = V3{u4.x, u4.y, u4.z} + beta * V3{p4.x, p4.y, p4.z};
      const V3 sv = w + beta * V3{s4.x, s4.y, s4.z};
      const V3 x = V3{x4.x, x4.y, x4.z} + alpha * p;
      const V3 rr = V3{r4.x, r4.y, r4.z} - alpha * sv;
      const V3 u = cmul(V3{d4.x, d4.y, d4.z}, rr);
      st4(a.p, r, p);
      st4(a.ap, r, sv);
      st4(a.x, r, x);
      st4(a.r, r, rr);
      st4(a.u, r, u);
      v3[0] += dot(rr, u);
      v3[2] += dot(rr, rr);
    }
    pc.lap(4);
    grid_barrier(a, rs);
    pc.lap(5);
    if (ASM) {
      auto w_sink2 = [&](int r, V3 ur, V3 wr) {
        st4(a.w, r, wr);
        v3[1] += dot(wr, ur);
      };
      row_pass<true>(a, a.u, w_sink2);
    } else {
      matvec_constraints(a, a.u);
      pc.lap(0);
      grid_barrier(a, rs);
      pc.lap(1);
      auto w_sink2 = [&](int, V3 ur, V3 wpart) { v3[1] += dot(wpart, ur); };
      if (a.item2)
        item_pass2(a, static_cast<const double4*>(a.u), a.contrib, a.wpart, w_sink2);
      else
        item_pass(a, a.u, w_sink2);
    }
    pc.lap(2);
    grid_reduce<3>(a, rs, v3, &pc);
    pc.lap(3);
    pc.count(15);
    gamma_prev = gamma;
    alpha_prev = alpha;
    gamma = v3[0];
    delta = v3[1];
    r_norm = sqrt(v3[2]);
    relres = r_norm / b_norm;
    iters = it + 1;
  }
}

// Round k of warp gw (of nw): rounds are dealt to the warps in order, or --
// when the rows are sorted by decreasing incidence count -- in snake order
// (0..nw-1, nw-1..0, ...), so every warp gets a heavy and a light share.
__device__ __forceinline__ int mf_round(int k, int gw, int nw, bool snake) {
  return k * nw + ((snake && (k & 1)) ? nw - 1 - gw : gw);
}
// Position (in the row order) of row-in-round grp of round k of warp gw.  With
// the decreasing-incidence order (perm) the rounds are dealt in snake order.
// When the level's heaviest row is very heavy (`hybrid`: more than kHeavyDeal
// incidences -- late in the configs[2] sequence the sparse term concentrates
// incidences on a few rows), round 0 is dealt differently: every warp's first
// row is one of the nw heaviest rows (warp gw takes position gw) and its other
// RPW - 1 rows are consecutive positions after those; dealing round 0's RPW
// heaviest rows to warp 0 held every block at the barrier (that warp's row
// pass 21 K cycles against 9 K on average).  The heaviest kHeavyRows rows are
// then summed by their whole warp (row_pass_mf).  Without perm: RPW
// consecutive rows per warp and round.
__device__ __forceinline__ int mf_pos(int k, int grp, int gw, int nw, int RPW, bool sorted, bool hybrid) {
  if (hybrid && k == 0) return grp == 0 ? gw : nw + gw * (RPW - 1) + (grp - 1);
  return mf_round(k, gw, nw, sorted) * RPW + grp;
}
constexpr int kHeavyDeal = 96;   // heaviest-row incidences from which round 0 is dealt one heavy row per warp
constexpr int kHeavyRows = 1024; // that many of the heaviest rows (all in round 0, row 0 of a warp, for any
                                 // block shape) are summed by their whole warp when above kHeavyRow
constexpr int kHeavyRow = 32;   // ... incidences

// Matrix-free row pass with kMfLanes lanes per row: the row's contiguous
// incidence contributions and its six face neighbours are strided over the
// lanes, a sub-warp shuffle tree sums them (fixed order), and the group
// leader receives (A v)_r -- so a row is complete inside one warp and its
// update can follow without another grid barrier.
template <bool HY = false, class Sink, class Meta = std::nullptr_t, class Sl = std::nullptr_t>
__device__ __forceinline__ void row_pass_mf(const FFArgs& a, const double4* v, Sink& sink, int skip = 0,
                                            const Meta* mm = nullptr, const Sl* sl = nullptr) {
  constexpr bool hybrid = HY;  // a separate instantiation: the common case keeps its code
  constexpr int L = kMfLanes, RPW = 32 / L;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L, grp = lane / L;
  const double w2 = 2.0 * a.w_r;
  if (gwarp() < skip) return;
  const int gw = gwarp() - skip, nw = nwarps() - skip;
  for (int k = 0;; ++k) {
    const bool sorted = a.perm != nullptr;
    const int pos = mf_pos(k, grp, gw, nw, RPW, sorted, hybrid);
    // rounds only grow with k: the warp's round start (hybrid round 0 is not
    // contiguous: every position of round k is >= k nw RPW)
    if ((HY ? k * nw * RPW : pos - grp) >= a.N) break;
    const bool live = pos < a.N;
    const int q = int(threadIdx.x >> 5) * (sl ? sl->K : 0) * RPW + k * RPW + grp;  // row slot
    int r = pos, e0 = 0, e1 = 0, nb[6] = {-1, -1, -1, -1, -1, -1};
    bool frozen = false;
    bool cached = false;
    if constexpr (!std::is_same<Meta, std::nullptr_t>::value) {
      if (mm && mm->rows) {
        cached = true;
        if (live) {
          const int4 m0 = mm->rm[q], m1 = mm->rn[q];
          e0 = m0.x;
          e1 = m0.y;
          frozen = m0.z != 0;
          nb[0] = m0.w; nb[1] = m1.x; nb[2] = m1.y; nb[3] = m1.z; nb[4] = m1.w;
          nb[5] = mm->rn5[q];
          r = mm->rid[q];
        }
      }
    }
    if (!cached && live) {
      if (a.perm) r = a.perm[pos];
      frozen = a.frozen[r];
      e0 = a.row_ptr[r];
      e1 = a.row_ptr[r + 1];
#pragma unroll
      for (int k2 = sub; k2 < 6; k2 += L) nb[k2] = a.nbr[int64_t(k2) * a.N + r];
    }
    const V3 vr = live ? ld4(v, r) : V3{0, 0, 0};
    V3 acc{0, 0, 0};
    // round 0's first row (one of the heaviest): its contributions summed by
    // all 32 lanes (butterfly tree) when it has more than kHeavyRow of them
    bool heavy = false;
    V3 hsum{0, 0, 0};
    if constexpr (HY) {
    if (k == 0 && gw < kHeavyRows) {
      const int he0 = __shfl_sync(0xffffffffu, e0, 0), he1 = __shfl_sync(0xffffffffu, e1, 0);
      const int hl = __shfl_sync(0xffffffffu, (live && !frozen) ? 1 : 0, 0);
      if (hl && he1 - he0 > kHeavyRow) {  // warp-uniform
        for (int e = he0 + lane; e < he1; e += 32) hsum += ld4(a.contrib, e);
        hsum.x = warp_sum(hsum.x);
        hsum.y = warp_sum(hsum.y);
        hsum.z = warp_sum(hsum.z);
        heavy = grp == 0;
      }
    }
    }
    if (live && !frozen) {
      if (heavy) {
        if (sub == 0) acc = hsum;
      } else {
        // the row's contributions in incidence order, eight loads in flight
        // before their (sequential, order-preserving) adds
        int e = e0 + sub;
        for (; e + 7 * L < e1; e += 8 * L) {
          V3 t[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = ld4(a.contrib, e + i * L);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc += t[i];
        }
        for (; e < e1; e += L) acc += ld4(a.contrib, e);
      }
#pragma unroll
      for (int k2 = sub; k2 < 6; k2 += L) {
        const int j = nb[k2];
        if (j >= 0) acc += w2 * (vr - ld4(v, j));
      }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    }
    if (live && sub == 0) sink(r, q, vr, frozen ? vr : acc);
  }
}

// ---- split reduction --------------------------------------------------------
// The pipelined iteration needs its dot products only after the next matvec,
// so the reduction is split off the barrier: every block publishes its block
// partials and passes a plain grid barrier; then global warp 0 (block 0,
// warp 0, which the PCG passes leave without rows) sums the partials in fixed
// block order and publishes the totals as flag-embedded words {32-bit half,
// 32-bit tag} (single-copy atomic 64-bit stores, so a reader that sees the tag
// sees the value), while every other warp proceeds with the matvec.  Blocks
// poll the totals only when the update needs them.  Partials and totals are
// double-buffered by the reduction sequence number, which a block can only
// reuse two reductions later -- after every block has consumed the older one.
constexpr int kSplitNV = 3;
__device__ __forceinline__ double* split_partials(const FFArgs& a, unsigned seq) {
  return a.partials + size_t(seq & 1) * kSplitNV * gridDim.x;
}
__device__ __forceinline__ unsigned long long* split_totals(const FFArgs& a, unsigned seq) {
  return a.sync_ll + (seq & 1) * 8;
}
// block sum of v -> partials[seq], then a grid barrier (publishes all writes)
__device__ __forceinline__ void split_arrive(const FFArgs& a, Red& rs, double (&v)[kSplitNV], unsigned seq) {
  __shared__ double smem[kSplitNV * 32];
  block_sum<kSplitNV>(v, smem);
  if (threadIdx.x < kSplitNV) split_partials(a, seq)[threadIdx.x * gridDim.x + blockIdx.x] = v[threadIdx.x];
  grid_barrier(a, rs);
}
// global warp 0 only, after split_arrive's barrier
__device__ __forceinline__ void split_total(const FFArgs& a, unsigned seq) {
  const int lane = threadIdx.x & 31;
  const double* part = split_partials(a, seq);
  double t[kSplitNV];
#pragma unroll
  for (int k = 0; k < kSplitNV; ++k) t[k] = 0;
  // fixed order: lane l sums blocks l, l + 32, ... then a fixed shuffle tree
  // one batch of loads for up to 160 blocks (B200: 148), then any remainder
  constexpr int J = 5;
  double x[kSplitNV][J];
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int k = 0; k < kSplitNV; ++k) {
      const int b = lane + 32 * j;
      x[k][j] = b < int(gridDim.x) ? __ldcg(part + k * gridDim.x + b) : 0.0;
    }
#pragma unroll
  for (int j = 0; j < J; ++j)
#pragma unroll
    for (int k = 0; k < kSplitNV; ++k) t[k] += x[k][j];
  for (int b = lane + 32 * J; b < int(gridDim.x); b += 32)
#pragma unroll
    for (int k = 0; k < kSplitNV; ++k) t[k] += __ldcg(part + k * gridDim.x + b);
#pragma unroll
  for (int k = 0; k < kSplitNV; ++k) t[k] = warp_sum(t[k]);
  if (lane < 2 * kSplitNV) {
    double tv = t[0];
#pragma unroll
    for (int k = 1; k < kSplitNV; ++k)
      if ((lane >> 1) == k) tv = t[k];
    const unsigned long long bits = (unsigned long long)__double_as_longlong(tv);
    const unsigned half = (lane & 1) ? unsigned(bits >> 32) : unsigned(bits);
    st_relaxed_u64(split_totals(a, seq) + lane, (unsigned long long)half << 32 | (seq + 1u));
  }
}
// every block: wait for the totals of reduction seq
__device__ __forceinline__ void split_wait(const FFArgs& a, unsigned seq, double (&v)[kSplitNV]) {
  __shared__ double bc[kSplitNV];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    unsigned half = 0;
    if (lane < 2 * kSplitNV) {
      const unsigned long long* w = split_totals(a, seq) + lane;
      unsigned long long x;
      do {
        x = ld_relaxed_u64(w);
      } while (unsigned(x) != seq + 1u);
      half = unsigned(x >> 32);
    }
    const unsigned hi = __shfl_down_sync(0xffffffffu, half, 1);
    if (lane < 2 * kSplitNV && !(lane & 1))
      bc[lane >> 1] = __longlong_as_double((long long)((unsigned long long)hi << 32 | half));
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kSplitNV; ++k) v[k] = bc[k];
}

// The rows a warp received from row_pass / row_pass_mf (L lanes per row: RPW
// rows per round, rounds nw apart), revisited with every lane busy: lane l
// takes row l % RPW of round l / RPW, 32 / RPW rounds per step.  The matvec
// results were stored by lanes of the same warp, so a __syncwarp orders them.
template <int L, class F>
__device__ __forceinline__ void for_warp_rows(int N, int skip, int K, const int32_t* perm, const int* rid, F f,
                                              bool hybrid = false) {
  constexpr int RPW = 32 / L, RPS = 32 / RPW;
  if (gwarp() < skip) return;
  __syncwarp();
  const int lane = threadIdx.x & 31;
  const int gw = gwarp() - skip, nw = nwarps() - skip;
  for (int k = lane / RPW;; k += RPS) {
    const int pos = mf_pos(k, lane % RPW, gw, nw, RPW, perm != nullptr, hybrid);
    if (!hybrid && pos >= N) break;  // positions grow with k
    if (hybrid) {                     // hybrid round 0 is not contiguous
      if (k * nw * RPW >= N) break;
      if (pos >= N) continue;
    }
    const int q = int(threadIdx.x >> 5) * K * RPW + k * RPW + lane % RPW;
    f(rid ? rid[q] : perm ? perm[pos] : pos, q);
  }
}

// Shared-memory row slots of the pipelined PCG.  The rows a warp receives
// from the row pass (L lanes per row: RPW rows per round, rounds nw warps
// apart) are always the same, so their Krylov state lives in the block's
// shared memory for the whole solve: slot (warp-in-block, round, row-in-round),
// stored component-major (vector, component, slot): consecutive lanes hit
// consecutive 8-byte words, 24 bytes per 3-vector.
enum { kSx, kSr, kSw, kSp, kSs, kSz, kSd, kSn, kSlotVecs };
// NSM (compile time): kSlotVecs -- the row state lives in shared memory and
// is addressed through the shared window; kSlotsSpill -- levels too large for
// shared memory keep it in a global spill area (this block's part, component
// arrays G x S apart), addressed through a generic pointer.  Specialising the
// shared case lets the compiler use 32-bit shared addressing in the hot loops.
constexpr int kSlotsSpill = -1;
template <int NSM>
struct SlotsT {
  double4* sm;    // shared memory, or the spill area (kSlotsSpill)
  size_t stride;  // S in shared memory, G x S in the spill area
  int S;          // slots per block = warps per block x K x RPW
  int K;          // rounds per warp
  int RPW, gw, nw;
  __device__ __forceinline__ int of(int r) const {
    return int(threadIdx.x >> 5) * K * RPW + ((r / RPW - gw) / nw) * RPW + r % RPW;
  }
  // round-major slot of the cached B^T B (assembled levels): the first rounds
  // first, so a partial last round is what stays in global memory
  __device__ __forceinline__ int amat_of(int r) const {
    return ((r / RPW - gw) / nw) * int(blockDim.x >> 5) * RPW + int(threadIdx.x >> 5) * RPW + r % RPW;
  }
  // component-major: (vector, component, slot) -- 24 bytes per 3-vector
  __device__ __forceinline__ double4 get(int v, int q) const {
    const double* b = reinterpret_cast<const double*>(sm) + size_t(3 * v) * stride + q;
    return make_double4(b[0], b[stride], b[2 * stride], 0.0);
  }
  __device__ __forceinline__ void put(int v, int q, double4 x) const {
    double* b = reinterpret_cast<double*>(sm) + size_t(3 * v) * stride + q;
    b[0] = x.x;
    b[stride] = x.y;
    b[2 * stride] = x.z;
  }
};
__host__ __device__ constexpr int pipe_rpw(bool asm_level, bool rows_on_lanes, int asm_lanes = kAsmLanes) {
  return rows_on_lanes ? 32 : 32 / (asm_level ? asm_lanes : kMfLanes);
}
// Shared-memory layout of one pipelined solve (host and device compute it
// alike): the row-state slots; on matrix-free levels optionally each row
// slot's metadata {e0, e1, frozen, 6 neighbours} (36 B) and each constraint
// slot's anchors, weights, g, incidence slots and kind (164 B), which are
// fixed for the whole solve and so cost one gather chain per iteration less.
struct PipeLayout {
  int K, S;      // rounds per warp, row slots per block
  int KC, SC;    // constraint rounds per thread, constraint slots per block
  size_t rmeta, cmeta, amat, total;  // byte offsets / size
};
__host__ __device__ inline PipeLayout pipe_layout(int N, int64_t C, int rpw, int G, int tpb, int skip, bool rows,
                                                  bool cons, int amat_slots = 0, int state_vecs = kSlotVecs) {
  PipeLayout l;
  const int wpb = tpb / 32;
  const int nw = G * wpb - skip;
  l.K = (N + nw * rpw - 1) / (nw * rpw);
  l.S = wpb * l.K * rpw;
  const int64_t nt = int64_t(G) * tpb - 32 * skip;
  l.KC = cons ? int((C + nt - 1) / nt) : 0;
  l.SC = tpb * l.KC;
  // row state in shared memory (state_vecs of the kSlotVecs vectors; the rest spill)
  size_t off = size_t(state_vecs) * l.S * 3 * sizeof(double);
  l.rmeta = off;
  if (rows) off += size_t(l.S) * (2 * sizeof(int4) + 2 * sizeof(int));
  off = (off + 31) / 32 * 32;
  l.cmeta = off;
  if (cons) off += size_t(l.SC) * (4 * sizeof(int4) + 3 * sizeof(double4) + sizeof(int));
  off = (off + 31) / 32 * 32;
  l.amat = off;  // assembled levels: 27 x 6 block values + 27 columns per cached row slot
  off += size_t(amat_slots) * 27 * (6 * sizeof(double) + sizeof(int));
  l.total = off;
  return l;
}
// SMEM views of the cached metadata
struct MfMeta {
  const int4* rm;   // S: e0, e1, frozen, nbr0
  const int4* rn;   // S: nbr1..nbr4
  const int* rn5;   // S: nbr5
  const int* rid;   // S: row id of the slot
  const int4* crow; // 2 SC
  const int4* cpos; // 2 SC
  const double4* cw;  // 2 SC
  const double4* cg;  // SC
  const int* ckind;   // SC
  bool rows, cons;
};
__device__ inline MfMeta mf_meta(char* base, const PipeLayout& l, bool rows, bool cons) {
  MfMeta m;
  m.rows = rows;
  m.cons = cons;
  char* r = base + l.rmeta;
  m.rm = reinterpret_cast<const int4*>(r);
  m.rn = reinterpret_cast<const int4*>(r + size_t(l.S) * sizeof(int4));
  m.rn5 = reinterpret_cast<const int*>(r + size_t(l.S) * 2 * sizeof(int4));
  m.rid = reinterpret_cast<const int*>(r + size_t(l.S) * (2 * sizeof(int4) + sizeof(int)));
  char* c = base + l.cmeta;
  const size_t SC = size_t(l.SC);
  m.cw = reinterpret_cast<const double4*>(c);
  m.cg = reinterpret_cast<const double4*>(c + 2 * SC * sizeof(double4));
  m.crow = reinterpret_cast<const int4*>(c + 3 * SC * sizeof(double4));
  m.cpos = reinterpret_cast<const int4*>(c + 3 * SC * sizeof(double4) + 2 * SC * sizeof(int4));
  m.ckind = reinterpret_cast<const int*>(c + 3 * SC * sizeof(double4) + 4 * SC * sizeof(int4));
  return m;
}
constexpr int kPipeSkip = 1;  // global warp 0 sums the split reductions
constexpr int kCgMinRows = 500000;  // spilled levels from this size run the Chronopoulos-Gear PCG
// ... and from this size when they carry fewer than 4 constraint incidences
// per row (256^3 level 0: 214 K rows, 2.3 per row, frame-1 solve 13.57 ->
// 13.21 ms; 512^3 level 2: 205 K rows, 12.6 per row, stays pipelined: 119.9
// vs 121.0 ms with CG)
constexpr int kCgMinRowsSparse = 200000;
// WFK_SLABS: matrix-free levels from this size are slab-partitioned; smaller
// levels (latency-bound, a few thousand rows per SM) run the unpartitioned
// fused PCG, replicated on every rank of a multi-GPU solve the way dist.cu
// replicates assembly.  WFK_SLAB_MIN_ROWS overrides (tests: 0 = every level).
constexpr int kSlabMinRows = 100000;
constexpr int kFastBlock = 512;      // threads per block of the WFK_PRECISION_FAST CG kernel
constexpr size_t kPipeSmemMax = 220 * 1024;  // dynamic shared memory for the row slots

// pcg_solve (solver.cpp:282-343) as pipelined Jacobi-PCG (Ghysels & Vanroose
// 2014): the same Krylov iterates as the reference's PCG in exact arithmetic,
// with w = A u, s = A p and z = A D s carried by recurrences, so the one grid
// reduction {r.u, w.u, r.r} of an iteration is not needed until after the
// next matvec n = A m (m = D w).  Per iteration:
//   assembled:    row pass n = A m | totals (global warp 0)
//                 update own rows  -> partials + barrier         (1 barrier)
//   matrix-free:  constraint pass of A m | totals -> barrier
//                 row pass n = A m, update own rows -> partials + barrier
// The update: z = n + beta z, s = w + beta s, p = u + beta p, x += alpha p,
// r -= alpha s, w -= alpha z, u = D r, m' = D w (into the other m buffer, as
// slower blocks may still gather the current one).  alpha and beta are the
// reference's: alpha = r.u / p.Ap with p.Ap = w.u - beta r.u / alpha_prev.
// Only m (gathered by neighbours) lives in global memory; x, r, w, p, s, z,
// D^-1 and n stay in the shared-memory slots of the warp that owns the row.
// Stopping rule, breakdown test and iteration count are the reference's.
template <bool ASM, int NSM, int AL = kAsmLanes>
__device__ __forceinline__ void pcg_pipe(const FFArgs& a, Red& rs, int& iters, double& relres) {
  extern __shared__ double4 dyn_smem[];
  iters = 0;
  relres = 0;
  PhaseClock pc(a.dbg);
  constexpr int kSkip = kPipeSkip;
  const bool comm = gwarp() == 0;
  constexpr int LM = ASM ? AL : kMfLanes;
  const bool rows_on_lanes = ASM && a.asm_rows_on_lanes;
  // round 0 dealt one heavy row per warp when the level's heaviest row is very heavy (mf_pos)
  bool hybrid = false;
  if (!ASM && a.perm && a.N > 0 && a.heavy_deal) {
    const int r0 = a.perm[0];
    hybrid = a.row_ptr[r0 + 1] - a.row_ptr[r0] > kHeavyDeal;
  }
  SlotsT<NSM> sl;
  sl.sm = dyn_smem;
  sl.RPW = pipe_rpw(ASM, rows_on_lanes, AL);
  const bool amat = ASM && a.asm_smem > 0 && !rows_on_lanes;
  const PipeLayout lay = pipe_layout(a.N, a.C, sl.RPW, gridDim.x, blockDim.x, kSkip, !ASM && a.meta_rows,
                                     !ASM && a.meta_cons, amat ? a.asm_smem : 0, a.state_spill ? 0 : kSlotVecs);
  sl.K = lay.K;
  sl.S = lay.S;
  sl.stride = size_t(lay.S);
  if (NSM == kSlotsSpill && a.state_spill) {  // the block's slots in the global spill area
    sl.sm = reinterpret_cast<double4*>(a.state_spill + size_t(blockIdx.x) * lay.S);
    sl.stride = size_t(lay.S) * gridDim.x;
  }
  sl.gw = gwarp() - kSkip;
  sl.nw = nwarps() - kSkip;
  const MfMeta mm = mf_meta(reinterpret_cast<char*>(dyn_smem), lay, !ASM && a.meta_rows, !ASM && a.meta_cons);
  const MfMeta* mmp = ASM ? nullptr : &mm;
  double* smb = amat ? reinterpret_cast<double*>(reinterpret_cast<char*>(dyn_smem) + lay.amat) : nullptr;
  int* smc = amat ? reinterpret_cast<int*>(reinterpret_cast<char*>(dyn_smem) + lay.amat + size_t(a.asm_smem) * 27 * 48)
                  : nullptr;
  if (amat && gwarp() >= kSkip) {
    // this warp's rows of B^T B into shared memory (fixed for the whole solve)
    const int lane = threadIdx.x & 31;
    for (int idx = 0; idx < sl.K * sl.RPW; ++idx) {
      const int r = (sl.gw + (idx / sl.RPW) * sl.nw) * sl.RPW + idx % sl.RPW;
      if (r >= a.N) break;
      const int q = sl.amat_of(r);
      if (q >= a.asm_smem) continue;  // beyond the cached slots: read from global in the row pass
      for (int t = lane; t < 27 * 6; t += 32) smb[q * 27 * 6 + t] = a.blk[int64_t(r) * 27 * 6 + t];
      if (lane < 27) smc[q * 27 + lane] = a.cols[int64_t(r) * 27 + lane];
    }
    __syncwarp();
  }
  // sinks receive (row, slot, v_r, (A v)_r)
  auto matvec = [&](const double4* v, auto& sink4) {
    if (ASM) {
      auto sink3 = [&](int r, V3 vr, V3 av) { sink4(r, sl.of(r), vr, av); };
      if (amat)
        row_pass<true, AL>(a, v, sink3, kSkip, &sl, smb, smc);
      else
        row_pass<true, AL>(a, v, sink3, kSkip);
    } else {
      matvec_constraints(a, v, kSkip, mmp);
      grid_barrier(a, rs);
      if (hybrid)
        row_pass_mf<true>(a, v, sink4, kSkip, mmp, &sl);
      else
        row_pass_mf<false>(a, v, sink4, kSkip, mmp, &sl);
    }
  };
  const int* rid_sm = (!ASM && mm.rows) ? mm.rid : nullptr;
  auto each_row = [&](auto f) {  // f(row, slot)
    if (rows_on_lanes)
      for_warp_rows<1>(a.N, kSkip, sl.K, nullptr, nullptr, f);
    else
      for_warp_rows<LM>(a.N, kSkip, sl.K, ASM ? nullptr : a.perm, rid_sm, f, hybrid);
  };
  if (!ASM && (mm.rows || mm.cons)) {
    // the solve's fixed row / constraint metadata into shared memory
    if (mm.rows)
      for_warp_rows<LM>(a.N, kSkip, sl.K, a.perm, nullptr, [&](int r, int q) {
        const_cast<int*>(mm.rid)[q] = r;
        int nb[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) nb[k] = a.nbr[int64_t(k) * a.N + r];
        const_cast<int4*>(mm.rm)[q] = make_int4(a.row_ptr[r], a.row_ptr[r + 1], a.frozen[r], nb[0]);
        const_cast<int4*>(mm.rn)[q] = make_int4(nb[1], nb[2], nb[3], nb[4]);
        const_cast<int*>(mm.rn5)[q] = nb[5];
      }, hybrid);
    if (mm.cons) {
      const int64_t c0 = gtid() - 32 * kSkip;
      if (c0 >= 0)
        for (int64_t c = c0, k = 0; c < a.C; c += gstride() - 32 * kSkip, ++k) {
          const int q = int(k) * blockDim.x + threadIdx.x;
          const int SC = lay.SC;
          const_cast<int4*>(mm.crow)[q] = a.c_row[2 * c];
          const_cast<int4*>(mm.crow)[SC + q] = a.c_row[2 * c + 1];
          const_cast<double4*>(mm.cw)[q] = a.c_w[2 * c];
          const_cast<double4*>(mm.cw)[SC + q] = a.c_w[2 * c + 1];
          const_cast<int4*>(mm.cpos)[q] = a.c_pos[2 * c];
          const_cast<int4*>(mm.cpos)[SC + q] = a.c_pos[2 * c + 1];
          const_cast<double4*>(mm.cg)[q] = a.c_g[c];
          const_cast<int*>(mm.ckind)[q] = a.c_kind[c];
        }
    }
    __syncthreads();
  }
  // r0 = b - A x0, u0 = D^-1 r0 (solver.cpp:305-310)
  double acc_rr = 0, acc_bb = 0;
  auto init_sink = [&](int r, int q, V3 xr, V3 ax) {
    const V3 b = ld4(a.rhs, r);
    const V3 rr = b - ax;
    const double4 d4 = ld4w(a.dinv, r);
    st4(a.u, r, cmul(V3{d4.x, d4.y, d4.z}, rr));
    const double4 zero = make_double4(0, 0, 0, 0);
    sl.put(kSx, q, make_double4(xr.x, xr.y, xr.z, 0.0));
    sl.put(kSr, q, make_double4(rr.x, rr.y, rr.z, 0.0));
    sl.put(kSp, q, zero);
    sl.put(kSs, q, zero);
    sl.put(kSz, q, zero);
    sl.put(kSd, q, d4);
    acc_rr += dot(rr, rr);
    acc_bb += sqnorm(b);
  };
  matvec(a.x, init_sink);
  grid_barrier(a, rs);
  // w0 = A u0, m0 = D w0
  double v4[4] = {0, 0, 0, 0};
  auto w_sink = [&](int r, int q, V3 ur, V3 wr) {
    const double4 d4 = sl.get(kSd, q), r4 = sl.get(kSr, q);
    sl.put(kSw, q, make_double4(wr.x, wr.y, wr.z, 0.0));
    st4(a.m0, r, cmul(V3{d4.x, d4.y, d4.z}, wr));
    v4[0] += dot(V3{r4.x, r4.y, r4.z}, ur);
    v4[1] += dot(wr, ur);
  };
  matvec(a.u, w_sink);
  v4[2] = acc_rr;
  v4[3] = acc_bb;
  grid_reduce<4>(a, rs, v4);
  double gamma = v4[0], delta = v4[1];
  double r_norm = sqrt(v4[2]);
  const double b_norm = sqrt(v4[3]);
  if (b_norm == 0) {
    for (int r = int(gtid()); r < a.N; r += int(gstride())) st4(a.x, r, V3{0, 0, 0});
    grid_barrier(a, rs);
    return;
  }
  relres = r_norm / b_norm;
  const double stop = fmax(a.pcg_tol * r_norm, 1e-13 * b_norm);
  double gamma_prev = 0, alpha_prev = 0;
  unsigned seq = 0;
  bool pending = false;  // totals of reduction seq - 1 not yet read
  pc.lap(12);
  for (int it = 0; it < a.pcg_max; ++it) {
    const double4* mcur = (it & 1) ? a.m1 : a.m0;
    double4* mnext = (it & 1) ? a.m0 : a.m1;
    // n = A m for own rows (into the leader's slot), overlapped with the
    // totals of the previous update
    auto n_sink = [&](int, int q, V3, V3 n) { sl.put(kSn, q, make_double4(n.x, n.y, n.z, 0.0)); };
    if (ASM) {
      if (comm && pending) split_total(a, seq - 1);
      matvec(mcur, n_sink);
    } else {
      matvec_constraints(a, mcur, kSkip, mmp);
      if (comm && pending) split_total(a, seq - 1);
      pc.lap(0);
      grid_barrier(a, rs);
      pc.lap(1);
      if (hybrid)
        row_pass_mf<true>(a, mcur, n_sink, kSkip, mmp, &sl);
      else
        row_pass_mf<false>(a, mcur, n_sink, kSkip, mmp, &sl);
    }
    pc.lap(2);
    if (pending) {
      double v3[3];
      split_wait(a, seq - 1, v3);
      gamma_prev = gamma;
      gamma = v3[0];
      delta = v3[1];
      r_norm = sqrt(v3[2]);
      relres = r_norm / b_norm;
      pending = false;
    }
    pc.lap(6);
    if (!(r_norm > stop)) break;
    const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
    const double pap = it == 0 ? delta : delta - beta * gamma / alpha_prev;
    if (pap <= 0) break;  // solver.cpp:327
    const double alpha = gamma / pap;
    double v3[3] = {0, 0, 0};
    auto upd = [&](int r, int q) {
      const double4 n4 = sl.get(kSn, q), w4 = sl.get(kSw, q), s4 = sl.get(kSs, q), z4 = sl.get(kSz, q),
                    p4 = sl.get(kSp, q), x4 = sl.get(kSx, q), r4 = sl.get(kSr, q), d4 = sl.get(kSd, q);
      const V3 d{d4.x, d4.y, d4.z};
      const V3 w{w4.x, w4.y, w4.z};
      V3 rr{r4.x, r4.y, r4.z};
      const V3 z = V3{n4.x, n4.y, n4.z} + beta * V3{z4.x, z4.y, z4.z};
      const V3 sv = w + beta * V3{s4.x, s4.y, s4.z};
      const V3 p = cmul(d, rr) + beta * V3{p4.x, p4.y, p4.z};
      const V3 x = V3{x4.x, x4.y, x4.z} + alpha * p;
      rr = rr - alpha * sv;
      const V3 wn = w - alpha * z;
      const V3 u = cmul(d, rr);
      sl.put(kSz, q, make_double4(z.x, z.y, z.z, 0.0));
      sl.put(kSs, q, make_double4(sv.x, sv.y, sv.z, 0.0));
      sl.put(kSp, q, make_double4(p.x, p.y, p.z, 0.0));
      sl.put(kSx, q, make_double4(x.x, x.y, x.z, 0.0));
      sl.put(kSr, q, make_double4(rr.x, rr.y, rr.z, 0.0));
      sl.put(kSw, q, make_double4(wn.x, wn.y, wn.z, 0.0));
      st4(mnext, r, cmul(d, wn));
      v3[0] += dot(rr, u);
      v3[1] += dot(wn, u);
      v3[2] += dot(rr, rr);
    };
    each_row(upd);
    pc.lap(4);
    split_arrive(a, rs, v3, seq);
    pc.lap(7);
    pc.count(15);
    alpha_prev = alpha;
    ++seq;
    pending = true;
    iters = it + 1;
  }
  if (pending) {
    // totals of the last update: residual of the returned iterate
    if (comm) split_total(a, seq - 1);
    double v3[3];
    split_wait(a, seq - 1, v3);
    r_norm = sqrt(v3[2]);
    relres = r_norm / b_norm;
  }
  // the solution back to global memory for the write-back phase
  each_row([&](int r, int q) { st4w(a.x, r, sl.get(kSx, q)); });
  grid_barrier(a, rs);
}

// update_rotations (solver.cpp:385-417) for every row; rot[] follows euler.
__device__ __forceinline__ void rotations(const FFArgs& a) {
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const int node = a.rows[r];
    const V3 can_i = a.g.canonical(node);
    const V3 ti = ld4(a.t, r);
    M3 h = m3_zero();
    for (int k = 0; k < 6; ++k) {
      const int j = a.nbr[int64_t(k) * a.N + r];
      if (j < 0) continue;
      const V3 rest = can_i - a.g.canonical(a.rows[j]);
      const V3 cur = ti - ld4(a.t, j);
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) h.a[p][q] += comp(rest, p) * comp(cur, q);
    }
    M3 u, v;
    double sv[3];
    svd3(h, u, sv, v);
    if (sv[1] < 1e-14) continue;
    M3 rm = mul(v, transpose(u));
    if (det(rm) < 0) {
      M3 flip = m3_identity();
      flip.a[2][2] = -1;
      rm = mul(mul(v, flip), transpose(u));
    }
    const V3 e = matrix_to_euler(rm);
    st3(a.field_eul, node, e);
    st_m3(a.rot, r, euler_to_matrix(e));
  }
}

// One instantiation per (PCG variant, level kind): each carries only the PCG
// code it runs, so the register allocation of one variant does not spill
// another's hot loops.
template <int V, bool ASM, int NSM = kSlotVecs, int TPB = kCoopBlock, int AL = kAsmLanes>
__global__ void __launch_bounds__(TPB, 1) k_flip_flop(FFArgs a) {
  cg::grid_group grid = cg::this_grid();
  Red rs;
  // load the row state from the field
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const int node = a.rows[r];
    st4(a.t, r, ld3(a.field_def, node));
    st_m3(a.rot, r, euler_to_matrix(ld3(a.field_eul, node)));
  }
  grid_barrier(a, rs);
  if (a.mode == 2) {
    rotations(a);
    return;
  }
  bool logic = false;
  wfk_energy prev = energy(a, grid, rs, logic);
  if (a.mode == 1 || logic) {
    if (gtid() == 0) {
      a.energy_out[0] = prev.total;
      a.energy_out[1] = prev.sparse;
      a.energy_out[2] = prev.dense;
      a.energy_out[3] = prev.reg;
      a.status[0] = 0;
      if (logic) a.status[1] |= 1;
    }
    return;
  }
  int n_trace = 0;
  int total_pcg = 0;
  if (prev.total != 0) {
    PhaseClock pc(a.dbg);
    for (int it = 0; it < a.ff_iters; ++it) {
      // assemble rhs / diagonal with the current rotations; x0 = t
      assemble_rows(a);
      for (int r = int(gtid()); r < a.N; r += int(gstride())) a.x[r] = a.t[r];
      grid_barrier(a, rs);
      pc.lap(8);
      int iters;
      double relres;
      if (V == 2 || V == 3 || V == 4) {
        if constexpr (!ASM) {
          if constexpr (V == 2)
            pcg_pk<float>(a, rs, iters, relres);
          else if constexpr (V == 3)
            pcg_pk<double>(a, rs, iters, relres);
          else
            pcg_slab(a, rs, iters, relres);
        }
      } else if (V == 1)
        pcg<ASM>(a, grid, rs, iters, relres);
      else
        pcg_pipe<ASM, NSM, AL>(a, rs, iters, relres);
      total_pcg += iters;
      pc.lap(9);
      // write back non-frozen rows (solver.cpp:436-437)
      for (int r = int(gtid()); r < a.N; r += int(gstride())) {
        if (a.frozen[r]) continue;
        const V3 xr = ld4(a.x, r);
        st4(a.t, r, xr);
        st3(a.field_def, a.rows[r], xr);
      }
      grid_barrier(a, rs);
      rotations(a);
      grid_barrier(a, rs);
      pc.lap(10);
      bool dummy;
      const wfk_energy e = energy(a, grid, rs, dummy);
      pc.lap(11);
      const bool anomaly = e.total > prev.total + 1e-9 * prev.total;
      if (gtid() == 0) {
        wfk_trace_entry& t = a.trace[n_trace];
        t.level = a.level;
        t.iteration = it;
        t.energy = e;
        t.pcg_iterations = iters;
        t.anomaly = anomaly ? 1 : 0;
        t.pcg_residual = relres;
      }
      ++n_trace;
      const double rel = (prev.total - e.total) / fmax(prev.total, 1e-300);
      prev = e;
      if (rel >= 0 && rel < a.ff_rel_tol) break;
    }
  }
  if (gtid() == 0) {
    a.status[0] = n_trace;
    a.status[2] = total_pcg;
    a.energy_out[0] = prev.total;
    a.energy_out[1] = prev.sparse;
    a.energy_out[2] = prev.dense;
    a.energy_out[3] = prev.reg;
  }
}

// ============================================================================
// assembled-system PCG (pcg_solve on an explicit NormalEquations)
// ============================================================================
struct AsmArgs {
  int N;
  const double* blocks;  // N x 27 x 9
  const int32_t* cols;   // N x 27
  const double* rhs;
  double *x, *r, *p, *ap, *dinv;
  double tol;
  int max_iters;
  int mode;  // 0 = pcg, 1 = multiply x -> ap
  double* partials;
  int32_t* status;
  double* relres_out;
};

__device__ __forceinline__ V3 asm_row(const AsmArgs& a, const double* v, int r) {
  V3 acc{0, 0, 0};
  for (int s = 0; s < 27; ++s) {
    const int c = a.cols[27 * int64_t(r) + s];
    if (c >= 0) acc += mul(ld_m3(a.blocks, 27 * int64_t(r) + s), ld3(v, c));
  }
  return acc;
}

template <int NV>
__device__ void grid_reduce_asm(const AsmArgs& a, cg::grid_group& grid, int& region, double (&v)[NV]) {
  __shared__ double smem[4 * 32];
  block_sum<NV>(v, smem);
  double* base = a.partials + size_t(region) * 4 * gridDim.x;
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) base[size_t(k) * gridDim.x + blockIdx.x] = v[k];
  grid.sync();
  for (int k = 0; k < NV; ++k) v[k] = sum_partials(base + size_t(k) * gridDim.x, gridDim.x);
  region ^= 1;
}

__global__ void __launch_bounds__(kCoopBlock, 1) k_pcg_assembled(AsmArgs a) {
  cg::grid_group grid = cg::this_grid();
  int region = 0;
  if (a.mode == 1) {
    for (int r = int(gtid()); r < a.N; r += int(gstride())) st3(a.ap, r, asm_row(a, a.x, r));
    return;
  }
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const M3 d = ld_m3(a.blocks, 27 * int64_t(r) + kCenter);
    st3(a.dinv, r, V3{d.a[0][0] > 1e-300 ? 1.0 / d.a[0][0] : 1.0, d.a[1][1] > 1e-300 ? 1.0 / d.a[1][1] : 1.0,
                      d.a[2][2] > 1e-300 ? 1.0 / d.a[2][2] : 1.0});
  }
  double v3[3] = {0, 0, 0};
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const V3 b = ld3(a.rhs, r);
    const V3 rr = b - asm_row(a, a.x, r);
    const V3 dv{1, 1, 1};
    (void)dv;
    st3(a.r, r, rr);
  }
  grid.sync();
  for (int r = int(gtid()); r < a.N; r += int(gstride())) {
    const V3 rr = ld3(a.r, r);
    const V3 z = cmul(ld3(a.dinv, r), rr);
    st3(a.p, r, z);
    v3[0] += dot(rr, z);
    v3[1] += dot(rr, rr);
    v3[2] += sqnorm(ld3(a.rhs, r));
  }
  grid_reduce_asm<3>(a, grid, region, v3);
  double rz = v3[0];
  double r_norm = sqrt(v3[1]);
  const double b_norm = sqrt(v3[2]);
  int iters = 0;
  double relres = 0;
  if (b_norm == 0) {
    for (int r = int(gtid()); r < a.N; r += int(gstride())) st3(a.x, r, V3{0, 0, 0});
  } else {
    relres = r_norm / b_norm;
    const double stop = fmax(a.tol * r_norm, 1e-13 * b_norm);
    for (int it = 0; it < a.max_iters && r_norm > stop; ++it) {
      double v1[1] = {0};
      for (int r = int(gtid()); r < a.N; r += int(gstride())) {
        const V3 apr = asm_row(a, a.p, r);
        st3(a.ap, r, apr);
        v1[0] += dot(ld3(a.p, r), apr);
      }
      grid_reduce_asm<1>(a, grid, region, v1);
      const double pap = v1[0];
      if (pap <= 0) break;
      const double alpha = rz / pap;
      double v2[2] = {0, 0};
      for (int r = int(gtid()); r < a.N; r += int(gstride())) {
        st3(a.x, r, ld3(a.x, r) + alpha * ld3(a.p, r));
        const V3 rr = ld3(a.r, r) - alpha * ld3(a.ap, r);
        st3(a.r, r, rr);
        const V3 z = cmul(ld3(a.dinv, r), rr);
        v2[0] += dot(rr, z);
        v2[1] += dot(rr, rr);
      }
      grid_reduce_asm<2>(a, grid, region, v2);
      const double beta = v2[0] / rz;
      rz = v2[0];
      for (int r = int(gtid()); r < a.N; r += int(gstride())) {
        const V3 z = cmul(ld3(a.dinv, r), ld3(a.r, r));
        st3(a.p, r, z + beta * ld3(a.p, r));
      }
      grid.sync();
      r_norm = sqrt(v2[1]);
      relres = r_norm / b_norm;
      iters = it + 1;
    }
  }
  if (gtid() == 0) {
    a.status[0] = iters;
    a.relres_out[0] = relres;
  }
}

// ============================================================================
// NormalEquations materialisation (test-facing build_normal_equations)
// ============================================================================
// build_normal_equations' blocks, cols and rhs (solver.cpp:113-275) with one
// warp per row: lane s < 27 owns stencil slot s and accumulates its 3x3 block
// in registers in the reference's order (incidences, then corners, then the
// ARAP terms); lane 0 builds the rhs.
__global__ void k_ne_assemble_warp(Grid g, int r0, int r1, const int32_t* rows, const int32_t* node_row,
                                   const int32_t* nbr, int N, const uint8_t* frozen, const int32_t* row_ptr,
                                   const int32_t* ent_con, const double* ent_w, const int32_t* c_node,
                                   const double* c_w, const int32_t* c_kind, const double* c_g, const double* rot,
                                   const double4* t, const double4* crhs, double w_r, double* blocks, int32_t* cols,
                                   double* rhs) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = r0 + warp; r < r1; r += nwarps) {
    const int node = rows[r];
    int x, y, z;
    g.idx3(node, x, y, z);
    double b[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) b[q] = 0.0;
    if (lane < 27) {
      const int dx = lane % 3 - 1, dy = (lane / 3) % 3 - 1, dz = lane / 9 - 1;
      cols[27 * int64_t(r) + lane] = g.in_grid(x + dx, y + dy, z + dz) ? node_row[g.lin(x + dx, y + dy, z + dz)] : -1;
    }
    if (frozen[r]) {
      if (lane == kCenter) b[0] = b[4] = b[8] = 1.0;
      if (lane == 0) st3(rhs, r, V3{t[r].x, t[r].y, t[r].z});
    } else {
      for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
        const int c = ent_con[e];
        const double ai = ent_w[e];
        const double coef = c_g[4 * c + 3];
        const double gg[3] = {c_g[4 * c], c_g[4 * c + 1], c_g[4 * c + 2]};
        const bool dense = c_kind[c] == WFK_DENSE_PLANE;
        for (int k = 0; k < 8; ++k) {
          int a, bb, cz;
          g.idx3(c_node[8 * c + k], a, bb, cz);
          if (stencil_slot(a - x, bb - y, cz - z) != lane) continue;
          const double sc = coef * ai * c_w[8 * c + k];
          if (dense) {
            for (int i = 0; i < 3; ++i)
              for (int j = 0; j < 3; ++j) b[i * 3 + j] += sc * (gg[i] * gg[j]);
          } else {
            for (int i = 0; i < 3; ++i)
              for (int j = 0; j < 3; ++j) b[i * 3 + j] += sc * (i == j ? 1.0 : 0.0);
          }
        }
      }
      const double w2 = 2.0 * w_r;
      V3 rv{crhs[r].x, crhs[r].y, crhs[r].z};
      const M3 ri = ld_m3(rot, r);
      const V3 can_i = g.canonical(node);
      for (int k = 0; k < 6; ++k) {
        const int j = nbr[int64_t(k) * N + r];
        if (j < 0) continue;
        if (lane == kCenter)
          for (int i = 0; i < 3; ++i) b[i * 4] += w2 * 1.0;
        if (lane == 0) {
          const V3 dij = can_i - g.canonical(rows[j]);
          rv += w_r * mul(add(ri, ld_m3(rot, j)), dij);
          if (frozen[j]) rv += w2 * V3{t[j].x, t[j].y, t[j].z};
        }
        if (!frozen[j] && lane == stencil_slot(kFace[k][0], kFace[k][1], kFace[k][2]))
          for (int i = 0; i < 3; ++i) b[i * 4] -= w2 * 1.0;
      }
      if (lane == 0) st3(rhs, r, rv);
    }
    if (lane < 27) {
      double* B = blocks + (int64_t(r) * 27 + lane) * 9;
#pragma unroll
      for (int q = 0; q < 9; ++q) B[q] = b[q];
    }
  }
}

__global__ void k_load_rows(int N, const int32_t* rows, const double* f_def, const double* f_eul, double4* t,
                            double* rot) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const V3 v = ld3(f_def, rows[r]);
    t[r] = make_double4(v.x, v.y, v.z, 0.0);
    st_m3(rot, r, euler_to_matrix(ld3(f_eul, rows[r])));
  }
}

// ============================================================================
// host orchestration
// ============================================================================

static void sync_check(wfk_ctx* c) { WFK_CUDA(cudaStreamSynchronize(c->stream)); }

// Compacts the level's active mask into rows (ascending), builds node_row,
// neighbours and the union-find labels.
static void level_rows(wfk_ctx* c, Level& L) {
  const int64_t n = L.g.n();
  cudaStream_t s = c->stream;
  // Level 0 mirrors the volume's active mask, which no solve changes: its rows,
  // neighbour table and component labels are reused until the mask changes
  // (compute_active_set / expand_grid / an ACTIVE upload bump active_gen).
  // Coarse levels: reused while build_hierarchy finds their activity mask
  // unchanged (it compares against the mask the rows were built from).
  const bool level0 = &L == &c->lv[0];
  const bool cached = level0 ? (L.rows_gen == c->vol.active_gen && L.rows_gen != 0) : (L.mask_same && L.rows_valid);
  if (cached) {
    if (L.N > 0) WFK_CUDA(cudaMemsetAsync(L.comp_flag.p, 0, size_t(L.N), s));
    return;
  }
  L.rows_valid = false;
  L.rows.ensure(size_t(n));
  L.node_row.ensure(size_t(n));
  int32_t* d_count = c->ivec.ensure(16);
  size_t tmp = 0;
  thrust::counting_iterator<int32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmp, it, L.active, L.rows.p, d_count, int(n), s);
  c->temp.ensure(tmp);
  WFK_CUDA(cub::DeviceSelect::Flagged(c->temp.p, tmp, it, L.active, L.rows.p, d_count, int(n), s));
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, d_count, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemsetAsync(L.node_row.p, 0xff, size_t(n) * sizeof(int32_t), s));
  sync_check(c);
  L.N = c->h_pinned[0];
  const int N = L.N;
  const size_t Nc = size_t(N > 0 ? N : 1);
  L.nbr.ensure(6 * Nc);
  L.uf.ensure(Nc);
  L.frozen.ensure(Nc);
  L.comp_flag.ensure(Nc);
  for (DevBuf<double4>* b : {&L.t, &L.x, &L.rhs, &L.r, &L.p, &L.ap, &L.dinv, &L.u, &L.w, &L.crhs, &L.cdiag, &L.z})
    b->ensure(Nc);
  L.mbuf.ensure(2 * Nc);
  L.nbuf.ensure(Nc);
  L.rot.ensure(9 * Nc);
  L.row_ptr.ensure(Nc + 1);
  L.cnt.ensure(Nc + 1);
  L.rows_gen = 0;
  if (N == 0) {
    L.rows_gen = level0 ? c->vol.active_gen : 0;
    L.rows_valid = true;
    return;
  }
  k_scatter_node_row<<<grid_for(N), kBlock, 0, s>>>(L.rows, N, L.node_row);
  k_row_neighbours<<<grid_for(N), kBlock, 0, s>>>(L.g, L.rows, N, L.node_row, L.nbr, L.uf);
  k_union<<<grid_for(N), kBlock, 0, s>>>(L.nbr, N, L.uf);
  k_uf_compress<<<grid_for(N), kBlock, 0, s>>>(N, L.uf, L.comp_flag);
  count_launch(c, 4);
  WFK_CUDA(cudaGetLastError());
  L.rows_gen = level0 ? c->vol.active_gen : 0;
  L.rows_valid = true;
}

// Prepares the level's constraints (anchors in c_node/c_w) for the solve:
// rows, frozen rows, incidence transpose and the constraint cache.
// Prepares the level's constraints (anchors in c_node/c_w) for the solve:
// rows, frozen rows, incidence transpose and the constraint cache.  No host
// synchronisation: the incidence count E stays on the device (row_ptr[N]) and
// every launch is sized by the bound 8C.
static void trace_mark(const char* n);
static void level_constraints(wfk_ctx* c, Level& L, const PoseD& pose, const wfk_solver_params& p) {
  cudaStream_t s = c->stream;
  const int64_t C = L.C;
  const int N = L.N;
  const size_t Cc = size_t(C > 0 ? C : 1);
  const int64_t E8 = 8 * C;  // bound on the incidence count
  L.c_row.ensure(8 * Cc);
  L.c_g.ensure(4 * Cc);
  L.c_b.ensure(Cc);
  L.c_u.ensure(3 * Cc);
  L.c_kind.ensure(Cc);
  L.key_in.ensure(8 * Cc);
  L.key_out.ensure(8 * Cc);
  L.val_in.ensure(8 * Cc);
  L.val_out.ensure(8 * Cc);
  L.ent_con.ensure(8 * Cc);
  L.ent_w.ensure(8 * Cc);
  L.ent_k.ensure(8 * Cc);
  L.c_pos.ensure(8 * Cc);
  L.items_built = false;
  if (C > 0) {
    k_con_prepare<<<grid_for(8 * C), kBlock, 0, s>>>(C, c->cons.kind, c->cons.target, c->cons.normal, c->cons.conf,
                                                 L.c_node, L.c_w, L.node_row, L.uf, pose, p.w_d, p.w_s, N, L.c_row,
                                                 L.c_g, L.c_b, L.c_kind, L.comp_flag, L.key_in, L.val_in);
    count_launch(c);
  }
  // E upper bound for the host-side decisions; the kernels use row_ptr[N]
  L.E = E8;
  if (N == 0) {
    WFK_CUDA(cudaMemsetAsync(L.row_ptr.p, 0, sizeof(int32_t), s));
    return;
  }
  trace_mark(" prep");
  k_frozen<<<grid_for(N), kBlock, 0, s>>>(N, L.uf, L.comp_flag, L.frozen);
  count_launch(c);
  if (C > 0) {
    // incidences sorted by (row, cell order); rows' ranges from the sorted keys
    int bits = 1;
    while ((int64_t(1) << bits) <= int64_t(N) * 8) ++bits;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, L.key_in.p, L.key_out.p, L.val_in.p, L.val_out.p, int(E8), 0, bits,
                                    s);
    c->temp.ensure(tmp);
    WFK_CUDA(cub::DeviceRadixSort::SortPairs(c->temp.p, tmp, L.key_in.p, L.key_out.p, L.val_in.p, L.val_out.p,
                                             int(E8), 0, bits, s));
    k_row_ptr_from_keys<<<grid_for(E8 + 1), kBlock, 0, s>>>(E8, L.key_out, N, L.row_ptr);
    WFK_CUDA(cudaMemsetAsync(L.c_pos.p, 0xff, size_t(E8) * sizeof(int32_t), s));
    k_entries<<<grid_for(E8), kBlock, 0, s>>>(L.row_ptr + N, L.val_out, L.c_w, L.ent_con, L.ent_k, L.ent_w,
                                              L.c_pos);
    count_launch(c, 3);
  } else {
    WFK_CUDA(cudaMemsetAsync(L.row_ptr.p, 0, size_t(N + 1) * sizeof(int32_t), s));
  }
  trace_mark(" sort");
  // Rows carrying many constraint incidences (coarse levels, where every
  // constraint of the frame lands on a few thousand nodes) get their B^T B
  // assembled once per solve, so the PCG row pass is a fixed 27-block stencil;
  // the same pass produces their constraint cache.
  L.assembled = E8 > int64_t(kAssembleRatio) * N;
  L.n_xitems = 0;
  if (!L.assembled) {
    L.contrib.ensure(size_t(std::max<int64_t>(E8, 1)));
    // row order of the pipelined row pass: decreasing incidence count (stable)
    L.perm.ensure(size_t(N));
    L.perm_key.ensure(2 * size_t(N));
    L.perm_val.ensure(size_t(N));
    k_row_count_keys<<<grid_for(N), kBlock, 0, s>>>(N, L.row_ptr, L.perm_key.p, L.perm_val.p);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, L.perm_key.p, L.perm_key.p + N, L.perm_val.p, L.perm.p,
                                              N, 0, 16, s);
    c->temp.ensure(tmp);
    WFK_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->temp.p, tmp, L.perm_key.p, L.perm_key.p + N,
                                                       L.perm_val.p, L.perm.p, N, 0, 16, s));
    count_launch(c, 2);
    k_constraint_cache<<<grid_for(N), kBlock, 0, s>>>(N, L.row_ptr, L.ent_con, L.ent_w, L.c_kind, L.c_g, L.c_b,
                                                      L.crhs, L.cdiag);
    count_launch(c);
    if (E8 > int64_t(kCacheWarpRow) * 2) {
      k_constraint_cache_warp<<<std::min(grid_for(int64_t(N) * 32), c->num_sms * 16), kBlock, 0, s>>>(
          N, L.row_ptr, L.ent_con, L.ent_w, L.c_kind, L.c_g, L.c_b, L.crhs, L.cdiag);
      count_launch(c);
    }
  } else {
    const int soa = N >= kAsmThreadRows ? 1 : 0;  // rows on lanes read slot-major blocks
    L.blk.ensure(size_t(N) * 27 * 6);
    L.cols.ensure(size_t(N) * 27);
    {
      // per device, under a lock (contexts on several devices / threads)
      static std::mutex asm_mu;
      static unsigned long long asm_attr = 0;  // bit d: device d configured
      std::lock_guard<std::mutex> lock(asm_mu);
      if (!(asm_attr & (1ull << (c->device & 63)))) {
        WFK_CUDA(cudaFuncSetAttribute(k_assemble_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kAsmSmem)));
        asm_attr |= 1ull << (c->device & 63);
      }
    }
    k_assemble_rows<<<std::min((N + kAsmWarps - 1) / kAsmWarps, c->num_sms * 2), kAsmWarps * 32, kAsmSmem, s>>>(
        L.g, N, L.rows, L.node_row, L.row_ptr, L.ent_con, L.ent_k, L.ent_w, L.c_w, L.c_g, L.c_b, L.c_kind, L.blk,
        L.cols, soa, L.crhs, L.cdiag);
    count_launch(c);
  }
  WFK_CUDA(cudaGetLastError());
}

// ---- slab plan (WFK_SLABS; see pcg_slab) -------------------------------------
__device__ __forceinline__ int slab_segment_of(const int32_t* bounds, int n, int r) {
  int lo = 0, hi = n - 1;  // last i with bounds[i] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bounds[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// u window of every rank: the rows its own rows' stencil and incident
// constraints reach (initialised to its own range)
__global__ void k_slab_window(int N, int S, const int32_t* rank_lo, const int32_t* nbr, const int32_t* row_ptr,
                              const int32_t* ent_con, const int4* c_row, int32_t* win_lo, int32_t* win_hi) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const int s = slab_segment_of(rank_lo, S, r);
    int lo = r, hi = r;
    for (int f = 0; f < 6; ++f) {
      const int j = nbr[int64_t(f) * N + r];
      if (j >= 0) {
        lo = min(lo, j);
        hi = max(hi, j);
      }
    }
    for (int e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      const int c = ent_con[e];
      const int4 q0 = c_row[2 * c], q1 = c_row[2 * c + 1];
      const int rr[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      for (int k = 0; k < 8; ++k)
        if (rr[k] >= 0) {
          lo = min(lo, rr[k]);
          hi = max(hi, rr[k]);
        }
    }
    atomicMin(&win_lo[s], lo);
    atomicMax(&win_hi[s], hi + 1);
  }
}
// per-row work weight of the block split, in units of one 32-byte access: the
// update and the row's first item (~12) plus one per incidence contribution
__global__ void k_slab_weight(int N, const int32_t* row_ptr, int32_t* w) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    w[r] = 12 + (row_ptr[r + 1] - row_ptr[r]);
}
// Tile t starts at the first row whose inclusive work prefix exceeds
// t W / ntiles (host and device share the rule: wfk_slab_plan, k_slab_tiles).
__host__ __device__ inline int slab_tile_bound(int t, int ntiles, int N, const int32_t* incl) {
  if (t <= 0 || N == 0) return 0;
  if (t >= ntiles) return N;
  const int64_t target = int64_t(t) * incl[N - 1] / ntiles;
  int lo = 0, hi = N;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (incl[mid] > target) hi = mid; else lo = mid + 1;
  }
  return lo;
}
__global__ void k_slab_tiles(int N, int ntiles, const int32_t* incl, int32_t* tile_row) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= ntiles) tile_row[t] = slab_tile_bound(t, ntiles, N, incl);
}
// constraints incident to each rank's rows: count (fill == nullptr) or list
__global__ void k_slab_cons(int64_t C, int S, const int32_t* rank_lo, const int4* c_row, const int4* c_pos,
                            int32_t* cnt, const int32_t* off, int32_t* fill) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < C; c += int64_t(gridDim.x) * blockDim.x) {
    const int4 q0 = c_row[2 * c], q1 = c_row[2 * c + 1], p0 = c_pos[2 * c], p1 = c_pos[2 * c + 1];
    const int rr[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    const int pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    int seen[8];
    int ns = 0;
    for (int k = 0; k < 8; ++k) {
      if (rr[k] < 0 || pp[k] < 0) continue;
      const int s = slab_segment_of(rank_lo, S, rr[k]);
      bool dup = false;
      for (int i = 0; i < ns; ++i) dup |= seen[i] == s;
      if (dup) continue;
      seen[ns++] = s;
      const int slot = atomicAdd(&cnt[s], 1);
      if (fill) fill[off[s] + slot] = int32_t(c);
    }
  }
}

// Work items of the balanced matrix-free item pass (Chronopoulos-Gear PCG
// only; built on first use per prepared level).
static void level_items(wfk_ctx* c, Level& L) {
  if (L.items_built || L.assembled || L.N == 0) return;
  cudaStream_t s = c->stream;
  const int N = L.N;
  L.xptr.ensure(size_t(N) + 1);
  L.xrange.ensure(size_t(N) + 1);
  int32_t* n_extra = L.cnt.p;  // per-row extra item counts
  k_item_count<<<grid_for(N), kBlock, 0, s>>>(N, L.row_ptr, n_extra);
  WFK_CUDA(cudaMemsetAsync(n_extra + N, 0, sizeof(int32_t), s));
  size_t tmp4 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp4, n_extra, L.xptr.p, N + 1, s);
  c->temp.ensure(tmp4);
  WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tmp4, n_extra, L.xptr.p, N + 1, s));
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 5, L.xptr.p + N, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  L.n_xitems = c->h_pinned[5];
  L.xitems.ensure(size_t(L.n_xitems) + 1);
  L.wpart.ensure(size_t(N) + size_t(L.n_xitems) + 1);
  k_item_write<<<grid_for(N), kBlock, 0, s>>>(N, L.row_ptr, L.xptr, L.xitems, L.xrange);
  count_launch(c, 3);
  L.items_built = true;
}

// Slab plan of a prepared matrix-free level for S ranks over G blocks (see
// pcg_slab): rank row ranges, u windows (checked to reach only the adjacent
// ranks), per-rank constraint lists and the reduction state; fills a.slab.
// Host side of the slab plan, shared with wfk_slab_plan (tests): the tile
// count -- one tile per block per blockDim rows, between 1 and 8 per block,
// from N and G only -- and the rank split: rank s owns tiles
// [s ntiles / S, (s + 1) ntiles / S) (tiles carry about equal work).
int slab_tile_count(int N, int G, int tpb) {
  const int64_t per_block = int64_t(N) / (int64_t(G) * tpb);
  return G * int(std::max<int64_t>(1, std::min<int64_t>(8, per_block)));
}
void slab_split(int ntiles, int S, int32_t* rank_tile) {
  for (int k = 0; k <= S; ++k) rank_tile[k] = int32_t((int64_t(k) * ntiles) / S);
}
int slab_tile_bound_host(int t, int ntiles, int N, const int32_t* incl) { return slab_tile_bound(t, ntiles, N, incl); }

static void slab_plan(wfk_ctx* c, Level& L, int S, int G, FFArgs& a) {
  cudaStream_t s = c->stream;
  const int N = L.N;
  // tiles of about equal work (12 units per row + 1 per incidence), their
  // count from N and G only; ranks take equal numbers of consecutive tiles
  const int ntiles = slab_tile_count(N, G, kFastBlock);
  S = std::max(1, std::min(S, G));
  int32_t* wgt = L.sl_blk.ensure(2 * size_t(std::max(N, 1)) + size_t(ntiles) + 1);
  int32_t* incl = wgt + std::max(N, 1);
  int32_t* d_trow = incl + std::max(N, 1);
  if (N > 0) {
    k_slab_weight<<<grid_for(N), kBlock, 0, s>>>(N, L.row_ptr, wgt);
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, wgt, incl, N, s);
    c->temp.ensure(tmp);
    WFK_CUDA(cub::DeviceScan::InclusiveSum(c->temp.p, tmp, wgt, incl, N, s));
  }
  k_slab_tiles<<<(ntiles + 1 + kBlock - 1) / kBlock, kBlock, 0, s>>>(N, ntiles, incl, d_trow);
  count_launch(c, 3);
  std::vector<int32_t> trow(size_t(ntiles) + 1);
  WFK_CUDA(cudaMemcpyAsync(trow.data(), d_trow, trow.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  std::vector<int32_t> rt(size_t(S) + 1, 0);  // rank tile bounds
  slab_split(ntiles, S, rt.data());
  std::vector<int32_t> lo(size_t(S) + 1);
  for (int k = 0; k <= S; ++k) lo[size_t(k)] = trow[size_t(rt[size_t(k)])];
  // device index area: rank_tile (S+1) | rank_lo (S+1) | win_lo (S) | win_hi (S) | con_ptr (S+1) | cnt (S) | list
  const size_t o_lo = size_t(S) + 1, o_wlo = o_lo + S + 1, o_whi = o_wlo + S, o_cptr = o_whi + S,
               o_cnt = o_cptr + S + 1, o_list = o_cnt + S;
  const size_t Cb = size_t(S) * size_t(std::max<int64_t>(L.C, 1));  // bound on the list entries
  int32_t* idx = L.sl_idx.ensure(o_list + 2 * Cb);
  int32_t* d_rt = idx;
  int32_t* d_lo = idx + o_lo;
  int32_t* d_wlo = idx + o_wlo;
  int32_t* d_whi = idx + o_whi;
  int32_t* d_cptr = idx + o_cptr;
  int32_t* d_cnt = idx + o_cnt;
  int32_t* d_list = idx + o_list;
  int32_t* d_sorted = d_list + Cb;
  std::vector<int32_t> init(o_list, 0);
  for (int k = 0; k <= S; ++k) {
    init[size_t(k)] = rt[size_t(k)];
    init[o_lo + size_t(k)] = lo[size_t(k)];
  }
  for (int k = 0; k < S; ++k) {
    init[o_wlo + size_t(k)] = lo[size_t(k)];
    init[o_whi + size_t(k)] = lo[size_t(k) + 1];
  }
  WFK_CUDA(cudaMemcpyAsync(idx, init.data(), init.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (N > 0)
    k_slab_window<<<grid_for(N), kBlock, 0, s>>>(N, S, d_lo, L.nbr, L.row_ptr, L.ent_con,
                                                 reinterpret_cast<const int4*>(L.c_row.p), d_wlo, d_whi);
  if (L.C > 0)
    k_slab_cons<<<grid_for(L.C), kBlock, 0, s>>>(L.C, S, d_lo, reinterpret_cast<const int4*>(L.c_row.p),
                                                 reinterpret_cast<const int4*>(L.c_pos.p), d_cnt, nullptr, nullptr);
  std::vector<int32_t> back(o_list);
  WFK_CUDA(cudaMemcpyAsync(back.data(), idx, back.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  std::vector<int32_t> wlo(back.begin() + o_wlo, back.begin() + o_wlo + S);
  std::vector<int32_t> whi(back.begin() + o_whi, back.begin() + o_whi + S);
  for (int k = 0; k < S; ++k) {
    if ((k > 0 && wlo[size_t(k)] < lo[size_t(k) - 1]) || (k + 2 <= S && whi[size_t(k)] > lo[size_t(k) + 2]))
      throw Error(WFK_E_INVALID_ARG, "slab partition: a slab is thinner than the stencil / constraint halo");
  }
  std::vector<int32_t> cptr(size_t(S) + 1, 0);
  for (int k = 0; k < S; ++k) cptr[size_t(k) + 1] = cptr[size_t(k)] + back[o_cnt + size_t(k)];
  WFK_CUDA(cudaMemcpyAsync(d_cptr, cptr.data(), cptr.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemsetAsync(d_cnt, 0, size_t(S) * sizeof(int32_t), s));
  if (L.C > 0) {
    k_slab_cons<<<grid_for(L.C), kBlock, 0, s>>>(L.C, S, d_lo, reinterpret_cast<const int4*>(L.c_row.p),
                                                 reinterpret_cast<const int4*>(L.c_pos.p), d_cnt, d_cptr, d_list);
    // each rank's list in constraint order (the atomics filled it unordered):
    // the constraint pass then reads its constraint records in order
    const int nl = cptr[size_t(S)];
    size_t tmp = 0;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp, d_list, d_sorted, nl, S, d_cptr, d_cptr + 1, 0, 32, s);
    c->temp.ensure(tmp);
    WFK_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(c->temp.p, tmp, d_list, d_sorted, nl, S, d_cptr, d_cptr + 1,
                                                     0, 32, s));
    count_launch(c, 3);
  }
  // u windows, counters (128 words per rank), tile partials (2 x ntiles x 8)
  // and totals (2 x 8) per rank
  std::vector<size_t> woff(size_t(S) + 1, 0);
  for (int k = 0; k < S; ++k) woff[size_t(k) + 1] = woff[size_t(k)] + size_t(whi[size_t(k)] - wlo[size_t(k)]);
  double4* win = L.sl_win.ensure(std::max<size_t>(woff[size_t(S)], 1));
  unsigned* ctr = L.sl_ctr.ensure(size_t(S) * 128);
  const size_t red_per_rank = size_t(2) * ntiles * 8 + 16;
  unsigned long long* red = L.sl_red.ensure(size_t(S) * red_per_rank);
  WFK_CUDA(cudaMemsetAsync(ctr, 0, size_t(S) * 128 * sizeof(unsigned), s));
  WFK_CUDA(cudaMemsetAsync(red, 0, size_t(S) * red_per_rank * sizeof(unsigned long long), s));
  // pointer tables (the peer pointers of a multi-GPU run)
  std::vector<unsigned long long> ptr(size_t(4) * S);
  for (int k = 0; k < S; ++k) {
    ptr[size_t(k)] = reinterpret_cast<unsigned long long>(win + woff[size_t(k)]);
    ptr[size_t(S + k)] = reinterpret_cast<unsigned long long>(ctr + size_t(k) * 128);
    ptr[size_t(2 * S + k)] = reinterpret_cast<unsigned long long>(red + size_t(k) * red_per_rank);
    ptr[size_t(3 * S + k)] = reinterpret_cast<unsigned long long>(red + size_t(k) * red_per_rank + size_t(2) * ntiles * 8);
  }
  unsigned long long* d_ptr = L.sl_ptr.ensure(ptr.size());
  WFK_CUDA(cudaMemcpyAsync(d_ptr, ptr.data(), ptr.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  sync_check(c);  // the host vectors above go out of scope
  a.slab.S = S;
  a.slab.ntiles = ntiles;
  a.slab.tile_row = d_trow;
  a.slab.rank_tile = d_rt;
  a.slab.win_lo = d_wlo;
  a.slab.win_hi = d_whi;
  a.slab.uwin = reinterpret_cast<double4* const*>(d_ptr);
  a.slab.ctr = reinterpret_cast<unsigned* const*>(d_ptr + S);
  a.slab.part = reinterpret_cast<unsigned long long* const*>(d_ptr + 2 * S);
  a.slab.tot = reinterpret_cast<unsigned long long* const*>(d_ptr + 3 * S);
  a.slab.con_ptr = d_cptr;
  a.slab.con_list = L.C > 0 ? d_sorted : d_list;
}

PoseD pose_dev(const wfk_pose* p) {
  PoseD q;
  for (int i = 0; i < 9; ++i) q.r.a[i / 3][i % 3] = p ? p->rotation[i] : (i % 4 == 0 ? 1.0 : 0.0);
  q.t = p ? V3{p->translation[0], p->translation[1], p->translation[2]} : V3{0, 0, 0};
  return q;
}

static int coop_blocks(wfk_ctx* c) {
  if (c->coop_blocks == 0) {
    int per_sm = 0;
    WFK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_flip_flop<0, false>, kCoopBlock, 0));
    int per_sm2 = 0;
    WFK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_pcg_assembled, kCoopBlock, 0));
    per_sm = std::min(per_sm, per_sm2);
    if (per_sm < 1) throw Error(WFK_E_CUDA, "cooperative kernel does not fit on an SM");
    // one persistent block per SM: fewest partials and barrier arrivals
    c->coop_blocks = std::min(c->num_sms, kMaxCoopBlocks);
  }
  return c->coop_blocks;
}

// Runs the cooperative kernel on a prepared level.  mode 0 = flip-flop,
// 1 = energy, 2 = rotations.  Returns trace entries appended to `out`.
static void run_level(wfk_ctx* c, Level& L, const PoseD& pose, const wfk_solver_params& p, int mode, int level_tag,
                      std::vector<wfk_trace_entry>* out, wfk_energy* e_out) {
  cudaStream_t s = c->stream;
  const int G = coop_blocks(c);  // one persistent block per SM (fewer blocks measured slower on every level)

  FFArgs a;
  a.g = L.g;
  a.N = L.N;
  a.C = L.C;
  a.mode = mode;
  a.level = level_tag;
  a.w_d = p.w_d;
  a.w_s = p.w_s;
  a.w_r = p.w_r;
  a.ff_rel_tol = p.flip_flop_rel_tol;
  a.pcg_tol = p.pcg_tol;
  a.ff_iters = p.flip_flop_iters;
  a.pcg_max = p.pcg_max_iters;
  a.pose = pose;
  a.rows = L.rows;
  a.nbr = L.nbr;
  a.frozen = L.frozen;
  a.field_def = L.deformed;
  a.field_eul = L.euler;
  a.t = L.t;
  a.x = L.x;
  a.rhs = L.rhs;
  a.r = L.r;
  a.p = L.p;
  a.u = L.u;
  a.w = L.w;
  a.z = L.z;
  a.m0 = L.mbuf.p;
  a.m1 = L.mbuf.p + std::max(L.N, 1);
  a.nbuf = L.nbuf.p;
  // read per call so tests can force the Chronopoulos-Gear variant
  const char* pcg_env = getenv("WFK_PCG");
  a.pcg_variant = (pcg_env && std::string(pcg_env) == "cg") ? 1 : 0;
  // WFK_SLABS=S (per call): matrix-free levels of >= kSlabMinRows rows run
  // the slab-partitioned CG with S ranks (pcg_slab; S = 1 is the same kernel
  // unpartitioned)
  const char* slab_env = getenv("WFK_SLABS");
  const int slabs = slab_env ? atoi(slab_env) : 0;
  const char* slab_min_env = getenv("WFK_SLAB_MIN_ROWS");
  const int64_t slab_min = slab_min_env ? atoll(slab_min_env) : kSlabMinRows;
  const bool slab = slabs >= 1 && !L.assembled && L.N > 0 && int64_t(L.N) >= slab_min && mode == 0 &&
                    c->precision != WFK_PRECISION_FAST;
  a.slab = SlabDev{};
  if (slab) a.pcg_variant = 1;
  a.assembled = L.assembled ? 1 : 0;
  a.asm_rows_on_lanes = L.N >= kAsmThreadRows ? 1 : 0;
  a.blk = L.blk;
  a.cols = L.cols;
  a.ap = L.ap;
  a.dinv = L.dinv;
  a.rot = L.rot;
  a.crhs = L.crhs;
  a.cdiag = L.cdiag;
  a.c_row = reinterpret_cast<const int4*>(L.c_row.p);
  a.c_w = reinterpret_cast<const double4*>(L.c_w.p);
  a.c_g = reinterpret_cast<const double4*>(L.c_g.p);
  a.c_kind = L.c_kind;
  a.target = c->cons.target;
  a.normal = c->cons.normal;
  a.conf = c->cons.conf;
  a.row_ptr = L.row_ptr;
  a.c_pos = reinterpret_cast<const int4*>(L.c_pos.p);
  a.contrib = L.contrib;
  a.xitems = L.xitems;
  a.n_xitems = L.n_xitems;
  a.xrange = L.xrange;
  a.wpart = L.wpart;
  a.partials = c->partials.ensure(size_t(8) * G);
  // barrier state: count, generation, totals, split totals on separate 128 B lines
  unsigned* sync = reinterpret_cast<unsigned*>(c->sync_words.ensure(128));
  WFK_CUDA(cudaMemsetAsync(sync, 0, 4 * 128, s));
  a.sync_count = sync;
  a.sync_gen = sync + 32;
  a.sync_total = reinterpret_cast<double*>(sync + 64);
  a.sync_ll = reinterpret_cast<unsigned long long*>(sync + 96);
  a.trace = c->trace.ensure(size_t(std::max(p.flip_flop_iters, 1)));
  int32_t* status = c->ivec.ensure(16) + 4;
  double* eout = c->eout.ensure(8);
  a.status = status;
  a.energy_out = eout;
  static const bool phase_timing = getenv("WFK_PHASE_TIMING") != nullptr;
  a.dbg = nullptr;
  if (phase_timing) {
    a.dbg = reinterpret_cast<unsigned long long*>(c->lvec.ensure(size_t(16) * G));
    WFK_CUDA(cudaMemsetAsync(a.dbg, 0, size_t(16) * G * sizeof(unsigned long long), s));
  }
  WFK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int32_t), s));
  if (L.N == 0 && L.C == 0 && mode != 2) {
    // nothing to solve: energy is exactly zero
    if (e_out) *e_out = wfk_energy{0, 0, 0, 0};
    return;
  }
  // pipelined PCG keeps the row state in shared memory; levels too large for
  // it use the Chronopoulos-Gear variant (state in global memory)
  size_t smem = 0;
  int nsm = kSlotVecs;  // kSlotVecs: row state in shared memory; 0: spilled (pipelined PCG)
  int tpb = kCoopBlock;  // threads per block of the launch
  int asm_lanes = kAsmLanes;  // lanes per row of a pipelined assembled level (8 or 4)
  a.meta_rows = a.meta_cons = 0;
  a.asm_smem = 0;
  a.state_spill = nullptr;
  // Levels far too large for shared memory (the row state would spill to
  // global) are HBM-bound, not latency-bound: there the Chronopoulos-Gear PCG,
  // which streams fewer vectors per iteration, beats the pipelined one
  // (512^3 frame-1 solve 138 vs 173 ms; at 256^3, 215 K rows, the pipelined
  // spill variant still wins, 13.7 vs 14.5 ms).  WFK_PCG=pipe forces pipelined.
  const char* cg_min_env = getenv("WFK_CG_MIN_ROWS");  // A/B: one plain row threshold
  const bool cg_size = cg_min_env ? int64_t(L.N) >= atoll(cg_min_env)
                                  : (L.N >= kCgMinRows || (L.N >= kCgMinRowsSparse && L.E < 4 * int64_t(L.N)));
  if (a.pcg_variant == 0 && cg_size && !(pcg_env && std::string(pcg_env) == "pipe")) {
    const PipeLayout probe = pipe_layout(L.N, L.C, pipe_rpw(L.assembled, a.asm_rows_on_lanes), G, kCoopBlockShared,
                                         kPipeSkip, false, false);
    if (probe.total > kPipeSmemMax) a.pcg_variant = 1;
  }
  if (a.pcg_variant == 0) {
    // assembled levels: 8 lanes per row.  WFK_ASM_LANES_RT=4 (opt-in) takes 4
    // lanes when that saves a whole round of rows (128^3 level 1: 13.6 K rows,
    // 2 rounds at 8 lanes, 1 at 4; 22.7 -> 22.3 ms/frame), but the reference's
    // acceptance gate through the adapter then failed its energy-descent
    // criterion in 4 of 19 runs (0 of 22 at 8 lanes), so it stays off until
    // that is understood
    if (L.assembled && !a.asm_rows_on_lanes) {
      const int64_t nw = int64_t(G) * (kCoopBlockShared / 32) - kPipeSkip;
      const int64_t r8 = (L.N + nw * 4 - 1) / (nw * 4), r4 = (L.N + nw * 8 - 1) / (nw * 8);
      const char* lanes_env = getenv("WFK_ASM_LANES_RT");
      asm_lanes = (lanes_env && atoi(lanes_env) == 4 && r4 < r8) ? 4 : 8;
    }
    int rpw = pipe_rpw(L.assembled, a.asm_rows_on_lanes, asm_lanes);
    // the row state goes to a global spill area when it does not fit shared memory
    // shared-memory row state runs with kCoopBlockShared threads per block
    // (more registers per thread: no spills); the spill variant with kCoopBlock
    tpb = kCoopBlockShared;
    PipeLayout base = pipe_layout(L.N, L.C, rpw, G, tpb, kPipeSkip, false, false);
    const bool spill = base.total > kPipeSmemMax || getenv("WFK_PIPE_SPILL") != nullptr;  // env (any value): tests force the spill area
    if (spill) {
      asm_lanes = kAsmLanes;  // the spill variant is instantiated with the default lanes
      rpw = pipe_rpw(L.assembled, a.asm_rows_on_lanes, asm_lanes);
      nsm = 0;
      tpb = kCoopBlock;
      base = pipe_layout(L.N, L.C, rpw, G, tpb, kPipeSkip, false, false);
      a.state_spill = L.state_spill.ensure(size_t(kSlotVecs) * 3 * size_t(G) * size_t(base.S));
    }
    auto bytes = [&](bool rows, bool cons) {
      return pipe_layout(L.N, L.C, rpw, G, tpb, kPipeSkip, rows, cons, false, nsm).total;
    };
    static const bool no_meta = getenv("WFK_PIPE_NO_META") != nullptr;
    a.asm_smem = 0;
    static const bool no_asm_smem = getenv("WFK_NO_ASM_SMEM") != nullptr;
    if (L.assembled && !a.asm_rows_on_lanes && !no_meta && !no_asm_smem) {
      // as many row slots' B^T B as fit (the rest of a partial last round is
      // read from global memory)
      const PipeLayout b0 = pipe_layout(L.N, L.C, rpw, G, tpb, kPipeSkip, false, false, 0, nsm);
      const size_t per = size_t(27) * (6 * sizeof(double) + sizeof(int));
      const size_t fit = b0.total < kPipeSmemMax ? (kPipeSmemMax - b0.total) / per : 0;
      a.asm_smem = int(std::min<size_t>(size_t(b0.S), fit));
    }
    static const bool cmeta = getenv("WFK_PIPE_CMETA") != nullptr;
    if (!L.assembled && !no_meta && cmeta && bytes(true, true) <= kPipeSmemMax) {
      a.meta_rows = a.meta_cons = 1;
    } else if (!L.assembled && !no_meta && bytes(true, false) <= kPipeSmemMax) {
      a.meta_rows = 1;
    }
    smem = a.asm_smem ? pipe_layout(L.N, L.C, rpw, G, tpb, kPipeSkip, false, false, a.asm_smem, nsm).total
                      : bytes(a.meta_rows, a.meta_cons);
    if (smem > kPipeSmemMax) {
      a.pcg_variant = 1;
      a.meta_rows = a.meta_cons = 0;
      smem = 0;
      tpb = kCoopBlock;
    }
  }
  static const bool no_perm = getenv("WFK_NO_PERM") != nullptr;
  a.perm = (a.pcg_variant == 0 && !L.assembled && L.N > 0 && !no_perm) ? L.perm.p : nullptr;
  if (a.pcg_variant == 1 && mode == 0) {
    level_items(c, L);  // the Chronopoulos-Gear item pass needs its work items
    a.xitems = L.xitems;
    a.n_xitems = L.n_xitems;
    a.xrange = L.xrange;
    a.wpart = L.wpart;
  }
  void (*kern)(FFArgs) = nullptr;
  const bool asm_k = L.assembled;
  // Matrix-free levels that run the CG variant keep their streamed Krylov
  // vectors packed (pcg_pk): fp64 xyz, 24 B (V = 3), or fp32 xyz, 12 B, with
  // WFK_PRECISION_FAST (V = 2); the gathered u and the scattered constraint
  // contributions stay aligned (double4 / float4), one sector per access.
  // configs[4] level-0 iteration, fp64: padded V = 1 A 58 K, B 264 K,
  // U 379 K cycles -> packed A 58 K, B 203 K, U 309 K (130.6 -> 119.3 ms per
  // frame-1 solve); fast: A 67 K -> 50 K with aligned contributions
  // (108.5 -> 102.8 ms).  WFK_PACK=0 selects the padded fp64 CG.
  const char* pack_env = getenv("WFK_PACK");  // per call: tests switch it
  const bool cg_mf = a.pcg_variant == 1 && !asm_k && L.N > 0 && mode == 0;
  const bool fast = c->precision == WFK_PRECISION_FAST && cg_mf;
  const bool packed64 = !fast && cg_mf && (slab || !(pack_env && pack_env[0] == '0'));
  static const bool item1 = getenv("WFK_ITEM1") != nullptr;  // A/B: one item per thread in flight
  a.heavy_deal = getenv("WFK_NO_HEAVY_DEAL") ? 0 : 1;
  a.item2 = item1 ? 0 : 1;
  a.fv = PackVecs<float>{};
  a.dv = PackVecs<double>{};
  auto bind_pack = [&](auto& pv, auto& r, auto& pp, auto& sv, auto& u, auto& d, auto& di, auto& ct, auto& wp) {
    const size_t n3 = 3 * size_t(L.N);
    pv.r = r.ensure(n3);
    pv.p = pp.ensure(n3);
    pv.s = sv.ensure(n3);
    pv.u = reinterpret_cast<decltype(pv.u)>(u.ensure(4 * size_t(L.N)));
    pv.d = d.ensure(n3);
    pv.dinv = di.ensure(n3);
    pv.contrib = reinterpret_cast<decltype(pv.contrib)>(ct.ensure(4 * size_t(std::max<int64_t>(L.E, 1))));
    pv.wpart = wp.ensure(3 * (size_t(L.N) + size_t(L.n_xitems) + 1));
  };
  if (fast) bind_pack(a.fv, L.f_r, L.f_p, L.f_s, L.f_u, L.f_d, L.f_dinv, L.f_contrib, L.f_wpart);
  if (packed64) bind_pack(a.dv, L.d_r, L.d_p, L.d_s, L.d_u, L.d_d, L.d_dinv, L.d_contrib, L.d_wpart);
  if (slab) {
    slab_plan(c, L, slabs, G, a);
    kern = k_flip_flop<4, false, kSlotVecs, kFastBlock>;
    tpb = kFastBlock;
  } else if (fast || packed64) {
    kern = fast ? k_flip_flop<2, false, kSlotVecs, kFastBlock> : k_flip_flop<3, false, kSlotVecs, kFastBlock>;
    tpb = kFastBlock;
  }
  else if (a.pcg_variant == 1)
    kern = asm_k ? k_flip_flop<1, true> : k_flip_flop<1, false>;
  else if (nsm == kSlotVecs)
    kern = asm_k ? (asm_lanes == 4 ? k_flip_flop<0, true, kSlotVecs, kCoopBlockShared, 4>
                                   : k_flip_flop<0, true, kSlotVecs, kCoopBlockShared>)
                 : k_flip_flop<0, false, kSlotVecs, kCoopBlockShared>;
  else
    kern = asm_k ? k_flip_flop<0, true, kSlotsSpill> : k_flip_flop<0, false, kSlotsSpill>;
  // kernel attributes are per device: set once per device, under a lock
  static std::mutex attr_mu;
  static unsigned long long attr_done = 0;  // bit d: device d configured
  {
  std::lock_guard<std::mutex> attr_lock(attr_mu);
  if (!(attr_done & (1ull << (c->device & 63)))) {
    for (void (*k)(FFArgs) : {k_flip_flop<0, false, kSlotVecs, kCoopBlockShared>,
                              k_flip_flop<0, true, kSlotVecs, kCoopBlockShared>,
                              k_flip_flop<0, true, kSlotVecs, kCoopBlockShared, 4>, k_flip_flop<1, false>,
                              k_flip_flop<1, true>, k_flip_flop<0, false, kSlotsSpill>,
                              k_flip_flop<0, true, kSlotsSpill>})
    {
      WFK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPipeSmemMax)));
      static const int carve = getenv("WFK_CARVEOUT") ? atoi(getenv("WFK_CARVEOUT")) : -1;
      if (carve >= 0) WFK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    }
    attr_done |= 1ull << (c->device & 63);
  }
  }
  void* args[] = {&a};
  Prof& pf = c->prof;
  if (pf.on) WFK_CUDA(cudaEventRecord(pf.ev[0], s));
  static const bool cluster2 = getenv("WFK_CLUSTER2") != nullptr;  // experiment: 2-CTA cluster arrivals
  a.cluster2 = (cluster2 && G % 2 == 0) ? 1 : 0;
  if (a.cluster2) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(G);
    lc.blockDim = dim3(tpb);
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 2;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 2;
    WFK_CUDA(cudaLaunchKernelExC(&lc, (const void*)kern, args));
  } else {
    WFK_CUDA(cudaLaunchCooperativeKernel((void*)kern, dim3(G), dim3(tpb), args, smem, s));
  }
  if (pf.on) WFK_CUDA(cudaEventRecord(pf.ev[1], s));
  count_launch(c);
  int32_t st[4];
  double en[4];
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 8, status, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(reinterpret_cast<double*>(c->h_pinned + 16), eout, 4 * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  // the trace rides along with the status when it fits the pinned area
  wfk_trace_entry* h_trace = reinterpret_cast<wfk_trace_entry*>(c->h_pinned + 256);
  const size_t trace_cap = (4096 - 256 * sizeof(int32_t)) / sizeof(wfk_trace_entry);
  const size_t n_trace_max = size_t(std::max(p.flip_flop_iters, 1));
  const bool trace_inline = out && n_trace_max <= trace_cap;
  if (trace_inline)
    WFK_CUDA(cudaMemcpyAsync(h_trace, a.trace, n_trace_max * sizeof(wfk_trace_entry), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  for (int i = 0; i < 4; ++i) st[i] = c->h_pinned[8 + i];
  for (int i = 0; i < 4; ++i) en[i] = reinterpret_cast<double*>(c->h_pinned + 16)[i];
  if (st[1] & 1) throw Error(WFK_E_LOGIC, "evaluate_energy: constraint anchors an inactive point");
  if (e_out) *e_out = wfk_energy{en[0], en[1], en[2], en[3]};
  c->stats.pcg_iterations += st[2];
  if (phase_timing) {
    std::vector<unsigned long long> d(size_t(16) * G);
    WFK_CUDA(cudaMemcpy(d.data(), a.dbg, d.size() * 8, cudaMemcpyDeviceToHost));
    const double it = double(d[15]) + 1e-9;
    auto stat = [&](int k, double& mean, double& mx) {
      mean = 0;
      mx = 0;
      for (int b = 0; b < G; ++b) {
        const double v = double(d[size_t(b) * 16 + k]) / it;
        mean += v / G;
        mx = std::max(mx, v);
      }
    };
    // pipelined PCG: A constraint pass, Abar its barrier, B row pass, U update,
    // wait = totals poll (incl. intra-block skew), bar = partials + grid barrier
    const char* names_cg[8] = {"A", "Async", "B", "red-", "U", "Usync", "redblk", "redsync"};
    const char* names_pipe[8] = {"A", "Abar", "B", "-", "U", "-", "wait", "bar"};
    const char* const* names = a.pcg_variant == 0 ? names_pipe : names_cg;
    int maxinc = 0;
    if (a.perm && L.N > 0) {  // incidences of the heaviest row (the row order's first)
      int32_t r0 = 0, rp[2] = {0, 0};
      WFK_CUDA(cudaMemcpy(&r0, a.perm, sizeof(int32_t), cudaMemcpyDeviceToHost));
      WFK_CUDA(cudaMemcpy(rp, L.row_ptr.p + r0, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost));
      maxinc = rp[1] - rp[0];
    }
    fprintf(stderr, "[wfk phase] level %d N %d C %lld asm %d maxinc %d iters %.0f | cycles/iter mean/max:", level_tag,
            L.N, (long long)L.C, int(L.assembled), maxinc, it);
    for (int k = 0; k < 8; ++k) {
      double m, x;
      stat(k, m, x);
      fprintf(stderr, " %s %.0f/%.0f", names[k], m, x);
    }
    double m13, x13;
    stat(13, m13, x13);
    fprintf(stderr, " redsum %.0f/%.0f | blk0 Mcyc/launch: assemble %.2f pcg %.2f rot %.2f energy %.2f\n", m13, x13,
            d[8] * 1e-6, d[9] * 1e-6, d[10] * 1e-6, d[11] * 1e-6);
  }
  if (pf.on && mode == 0) {
    float ms = 0;
    WFK_CUDA(cudaEventElapsedTime(&ms, pf.ev[0], pf.ev[1]));
    pf.ff_launches += 1;
    pf.ff_ms += ms;
    pf.pcg_iterations += st[2];
    // algorithmic bytes of this launch.  SURVEY.md 8(d): PCG iteration
    // 160 N + 32 C_d + 20 C_s; rotation fit 28 N; energy 28 N + 44 C;
    // rhs/diagonal 52 N per flip-flop iteration (+ the initial energy).
    const double N = L.N, Cs = double(std::min<int64_t>(c->cons.n_sparse, L.C)), Cd = double(L.C) - Cs;
    const double iters = st[0], pcg = st[2];
    pf.ff_bytes += pcg * (160 * N + 32 * Cd + 20 * Cs) + iters * (52 * N + 28 * N + 28 * N + 44 * (Cd + Cs)) +
                   (28 * N + 44 * (Cd + Cs));
    // the global-memory traffic of this fp64 implementation:
    // pipelined PCG iteration, state in shared memory -- matrix-free 256 N + 768 C
    // (m gathers at 8 anchors + 8 contribution writes per constraint, contribution
    // reads, m_r + 6 neighbour gathers + m write per row), assembled 896 N (27 m
    // gathers + m write per row; + 1404 N when B^T B is not shared-memory resident);
    // Chronopoulos-Gear 365 N + 276 C.  Per flip-flop iteration rhs/diag 153 N,
    // write-back 48 N, rotation fit 201 N, energy 177 N + 232 C.
    double per_it;
    if (a.pcg_variant == 0)
      per_it = L.assembled ? (896 + (a.asm_smem ? 0 : 1404)) * N : 256 * N + 768 * (Cd + Cs);
    else
      per_it = 365 * N + 276 * (Cd + Cs);
    pf.ff_bytes_impl += pcg * per_it + iters * ((153 + 48 + 201 + 177) * N + 232 * (Cd + Cs)) +
                        (177 * N + 232 * (Cd + Cs));
  }
  if (out && st[0] > 0) {
    const size_t k = out->size();
    out->resize(k + size_t(st[0]));
    if (trace_inline) {
      std::copy(h_trace, h_trace + st[0], out->data() + k);
    } else {
      WFK_CUDA(cudaMemcpyAsync(out->data() + k, a.trace, size_t(st[0]) * sizeof(wfk_trace_entry),
                               cudaMemcpyDeviceToHost, s));
      sync_check(c);
    }
  }
}

// level 0 aliases the volume and the uploaded anchors
static void bind_level0(wfk_ctx* c) {
  Level& L = c->lv[0];
  L.g = c->vol.g;
  L.deformed = c->vol.deformed;
  L.euler = c->vol.euler;
  L.active = c->vol.active;
  L.C = c->cons.count;
  const size_t Cc = size_t(std::max<int64_t>(L.C, 1));
  L.c_node.ensure(8 * Cc);
  L.c_w.ensure(8 * Cc);
  if (L.C > 0) {
    WFK_CUDA(cudaMemcpyAsync(L.c_node.p, c->cons.anchor.p, size_t(8 * L.C) * sizeof(int32_t),
                             cudaMemcpyDeviceToDevice, c->stream));
    WFK_CUDA(cudaMemcpyAsync(L.c_w.p, c->cons.weight.p, size_t(8 * L.C) * sizeof(double), cudaMemcpyDeviceToDevice,
                             c->stream));
  }
}

static void require_volume(wfk_ctx* c) {
  if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
}

// build_hierarchy (solver.cpp:455-503): levels 1..L-1 from level 0
static void build_hierarchy(wfk_ctx* c, int levels) {
  if (levels < 1) throw Error(WFK_E_INVALID_ARG, "build_hierarchy: levels must be >= 1");
  if (levels > kMaxLevels) throw Error(WFK_E_INVALID_ARG, "build_hierarchy: too many levels");
  cudaStream_t s = c->stream;
  int32_t* err = c->ivec.ensure(16) + 12;
  WFK_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), s));
  for (int l = 1; l < levels; ++l) {
    Level& F = c->lv[l - 1];
    Level& Cl = c->lv[l];
    Grid cg_ = F.g;
    cg_.nx = (F.g.nx - 1 + 1) / 2 + 1;
    cg_.ny = (F.g.ny - 1 + 1) / 2 + 1;
    cg_.nz = (F.g.nz - 1 + 1) / 2 + 1;
    if (cg_.nx < 2 || cg_.ny < 2 || cg_.nz < 2)
      throw Error(WFK_E_INVALID_ARG, "build_hierarchy: coarsest level below 2^3");
    cg_.voxel = F.g.voxel * 2.0;
    Cl.g = cg_;
    const size_t n = size_t(cg_.n());
    Cl.deformed = Cl.own_deformed.ensure(3 * n);
    Cl.euler = Cl.own_euler.ensure(3 * n);
    Cl.active = Cl.own_active.ensure(n);
    Cl.owns_field = true;
    k_coarse_init<<<grid_for(int64_t(n)), kBlock, 0, s>>>(F.g, cg_, F.deformed, F.euler, Cl.deformed, Cl.euler,
                                                          Cl.active);
    k_coarse_activity<<<grid_for(F.g.n()), kBlock, 0, s>>>(F.g, cg_, F.active, Cl.active, err);
    Cl.C = c->cons.count;
    const size_t Cc = size_t(std::max<int64_t>(Cl.C, 1));
    Cl.c_node.ensure(8 * Cc);
    Cl.c_w.ensure(8 * Cc);
    if (Cl.C > 0)
      k_reanchor<<<grid_for(Cl.C), kBlock, 0, s>>>(Cl.C, cg_, c->cons.canonical, Cl.c_node, Cl.c_w, Cl.active, err);
    // did the activity mask change since the level's rows were built?
    const bool same_grid = Cl.prev_n == n && Cl.prev_dims[0] == cg_.nx && Cl.prev_dims[1] == cg_.ny &&
                           Cl.prev_dims[2] == cg_.nz;
    Cl.prev_active.ensure(n);
    if (!same_grid) WFK_CUDA(cudaMemsetAsync(Cl.prev_active.p, 0xff, n, s));
    k_mask_update<<<grid_for(int64_t(n)), kBlock, 0, s>>>(int64_t(n), Cl.active, Cl.prev_active, err, 1 << (8 + l));
    Cl.prev_n = n;
    Cl.prev_dims[0] = cg_.nx;
    Cl.prev_dims[1] = cg_.ny;
    Cl.prev_dims[2] = cg_.nz;
    count_launch(c, 4);
  }
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 2, err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  if (c->h_pinned[2] & 2) throw Error(WFK_E_OUT_OF_RANGE, "trilinear_anchors: point outside grid");
  for (int l = 1; l < levels; ++l) {
    Level& Cl = c->lv[l];
    Cl.mask_same = !(c->h_pinned[2] & (1 << (8 + l)));
    if (!Cl.mask_same) Cl.rows_valid = false;  // rows were built from an older mask
  }
}

static void prolong(wfk_ctx* c, int l) {
  Level& Cl = c->lv[l];
  Level& F = c->lv[l - 1];
  k_prolong<<<grid_for(F.g.n()), kBlock, 0, c->stream>>>(F.g, Cl.g, F.active, F.deformed, F.euler, Cl.deformed,
                                                         Cl.euler);
  count_launch(c);
}

// WFK_SETUP_TRACE=1: device-timeline breakdown of each coarse-to-fine solve
// (events between the host steps; gaps where the device waits for the host
// are attributed to the step that follows them).
struct SetupTrace {
  bool on = false;
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> name;
  void mark(const char* n) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    name.push_back(n);
  }
  void report() {
    if (!on || ev.size() < 2) return;
    cudaEventSynchronize(ev.back());
    fprintf(stderr, "[wfk setup]");
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
      fprintf(stderr, " %s %.3f", name[i], ms);
    }
    float tot = 0;
    cudaEventElapsedTime(&tot, ev.front(), ev.back());
    fprintf(stderr, " | total %.3f ms\n", tot);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
    name.clear();
  }
};
static SetupTrace* g_trace = nullptr;
static void trace_mark(const char* n) {
  if (g_trace) g_trace->mark(n);
}

void solve_level(wfk_ctx* c, int l, const PoseD& pose, const wfk_solver_params& p, int mode,
                 std::vector<wfk_trace_entry>* trace, wfk_energy* e) {
  Level& L = c->lv[l];
  level_rows(c, L);
  trace_mark(l == 0 ? "L0rows" : l == 1 ? "L1rows" : "L2rows");
  level_constraints(c, L, pose, p);
  trace_mark(l == 0 ? "L0cons" : l == 1 ? "L1cons" : "L2cons");
  run_level(c, L, pose, p, mode, l, trace, e);
  trace_mark(l == 0 ? "L0ff" : l == 1 ? "L1ff" : "L2ff");
}

// --------------------------------------------------------------------------
// entry points used by api.cu
// --------------------------------------------------------------------------
void solver_flip_flop(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, int level_tag,
                      std::vector<wfk_trace_entry>& trace) {
  require_volume(c);
  bind_level0(c);
  Level& L = c->lv[0];
  const PoseD pd = pose_dev(pose);
  level_rows(c, L);
  level_constraints(c, L, pd, p);
  run_level(c, L, pd, p, 0, level_tag, &trace, nullptr);
}

void solver_energy(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, wfk_energy* e) {
  require_volume(c);
  bind_level0(c);
  solve_level(c, 0, pose_dev(pose), p, 1, nullptr, e);
}

void solver_rotations(wfk_ctx* c) {
  require_volume(c);
  bind_level0(c);
  wfk_solver_params p{};
  Level& L = c->lv[0];
  level_rows(c, L);
  if (L.N == 0) return;
  const int64_t Csave = L.C;
  L.C = 0;
  run_level(c, L, pose_dev(nullptr), p, 2, 0, nullptr, nullptr);
  L.C = Csave;
}

// Every level's setup -- rows (level_rows), constraint incidences, frozen
// rows, B^T B / constraint cache (level_constraints) -- depends only on the
// hierarchy (activity, re-anchored constraints) and the frame's constraints,
// never on a coarser level's solution.  So after build_hierarchy the levels'
// setups, chains of small latency-bound kernels, are issued on one stream per
// level and overlap one another; the context stream waits for all of them
// before the first flip-flop launch.  Each level uses its own cub scratch and
// count word while its setup runs (swapped in for the context's); the kernels
// and their inputs are the serial path's, so results are bit-identical
// (WFK_SERIAL_SETUP=1 restores the serial order for A/B runs).
template <class T>
static void swap_buf(DevBuf<T>& a, DevBuf<T>& b) {
  std::swap(a.p, b.p);
  std::swap(a.cap, b.cap);
}
struct SetupScope {
  wfk_ctx* c;
  Level& L;
  cudaStream_t saved;
  SetupScope(wfk_ctx* c_, Level& L_) : c(c_), L(L_), saved(c_->stream) {
    c->stream = L.setup_stream;
    swap_buf(c->temp, L.setup_temp);
    swap_buf(c->ivec, L.setup_ivec);
  }
  ~SetupScope() {
    swap_buf(c->ivec, L.setup_ivec);
    swap_buf(c->temp, L.setup_temp);
    c->stream = saved;
  }
};
static void setup_levels(wfk_ctx* c, int levels, const PoseD& pd, const wfk_solver_params& p) {
  if (!c->setup_ready) WFK_CUDA(cudaEventCreateWithFlags(&c->setup_ready, cudaEventDisableTiming));
  WFK_CUDA(cudaEventRecord(c->setup_ready, c->stream));
  for (int l = levels - 1; l >= 0; --l) {
    Level& L = c->lv[l];
    if (!L.setup_stream) WFK_CUDA(cudaStreamCreateWithFlags(&L.setup_stream, cudaStreamNonBlocking));
    if (!L.setup_done) WFK_CUDA(cudaEventCreateWithFlags(&L.setup_done, cudaEventDisableTiming));
    WFK_CUDA(cudaStreamWaitEvent(L.setup_stream, c->setup_ready, 0));
    {
      SetupScope scope(c, L);
      level_rows(c, L);
      level_constraints(c, L, pd, p);
    }
    WFK_CUDA(cudaEventRecord(L.setup_done, L.setup_stream));
  }
  for (int l = levels - 1; l >= 0; --l) WFK_CUDA(cudaStreamWaitEvent(c->stream, c->lv[l].setup_done, 0));
}

void solver_c2f(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, std::vector<wfk_trace_entry>& trace) {
  require_volume(c);
  bind_level0(c);
  const PoseD pd = pose_dev(pose);
  static const bool tracing = getenv("WFK_SETUP_TRACE") != nullptr;
  SetupTrace tr;
  if (tracing) {
    tr.on = true;
    tr.s = c->stream;
    g_trace = &tr;
    tr.mark("start");
  }
  build_hierarchy(c, p.levels);
  trace_mark("hier");
  static const bool serial_setup = getenv("WFK_SERIAL_SETUP") != nullptr;
  if (!serial_setup) {
    setup_levels(c, p.levels, pd, p);
    trace_mark("setup");
  }
  auto solve = [&](int l) {
    if (serial_setup) {
      solve_level(c, l, pd, p, 0, &trace, nullptr);
    } else {
      run_level(c, c->lv[l], pd, p, 0, l, &trace, nullptr);
      trace_mark(l == 0 ? "L0ff" : l == 1 ? "L1ff" : "L2ff");
    }
  };
  for (int l = p.levels - 1; l >= 1; --l) {
    solve(l);
    prolong(c, l);
    trace_mark("prolong");
  }
  solve(0);
  if (tracing) {
    tr.report();
    g_trace = nullptr;
  }
}

// --------------------------------------------------------------------------
// solve_coarse_to_fine with the PCG partitioned into z-slabs
// (dist.cu).  Every rank holds the same replicated lattice, so the hierarchy,
// rows, constraint cache, normal-equation assembly (k_ne_assemble), the
// write-back, the Procrustes fit and the energy are computed identically on
// every rank; the PCG -- the per-iteration work -- runs on the rank's slab
// with NCCL halo exchanges, and its solution is broadcast back to all ranks.
// flip_flop_solve's control flow (solver.cpp:419-453) is restated on the host.
// slabs > 0: that many slab states on this GPU (single-GPU check); slabs == 0:
// the context's communicator (wfk_dist_init).
// --------------------------------------------------------------------------
__global__ void k_rows_to_x(int N, const double4* t, double* x) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    st3(x, r, V3{t[r].x, t[r].y, t[r].z});
}
__global__ void k_write_back(int N, const int32_t* rows, const uint8_t* frozen, const double* x, double* f_def) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    if (!frozen[r]) st3(f_def, rows[r], ld3(x, r));
}

static void dist_flip_flop(wfk_ctx* c, int l, const PoseD& pose, const wfk_solver_params& p, int slabs,
                           std::vector<wfk_trace_entry>& trace) {
  static const bool dtrace = getenv("WFK_DIST_TRACE") != nullptr;
  auto t_prev = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dtrace) return;
    sync_check(c);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[wfk dist ff] L%d %-10s %.3f ms\n", l, what,
            std::chrono::duration<double, std::milli>(t - t_prev).count());
    t_prev = t;
  };
  Level& L = c->lv[l];
  level_rows(c, L);
  level_constraints(c, L, pose, p);
  lap("setup");
  wfk_energy prev;
  run_level(c, L, pose, p, 1, l, nullptr, &prev);  // evaluate_energy
  lap("energy0");
  if (prev.total == 0) return;
  const int N = L.N;
  cudaStream_t s = c->stream;
  double* blocks = L.ne_blocks.ensure(size_t(std::max(N, 1)) * 27 * 9);
  int32_t* cols = L.ne_cols.ensure(size_t(std::max(N, 1)) * 27);
  double* rhs = L.ne_rhs.ensure(size_t(std::max(N, 1)) * 3);
  double* x = L.ne_x.ensure(size_t(std::max(N, 1)) * 3);
  for (int it = 0; it < p.flip_flop_iters; ++it) {
    wfk_pcg_result pr{0, 0, 0.0};
    if (N > 0) {
      k_load_rows<<<grid_for(N), kBlock, 0, s>>>(N, L.rows, L.deformed, L.euler, L.t, L.rot);
      k_ne_assemble_warp<<<grid_for(int64_t(N) * 32), kBlock, 0, s>>>(
          L.g, 0, N, L.rows, L.node_row, L.nbr, N, L.frozen, L.row_ptr, L.ent_con, L.ent_w, L.c_node, L.c_w,
          L.c_kind, L.c_g, L.rot, L.t, L.crhs, p.w_r, blocks, cols, rhs);
      k_rows_to_x<<<grid_for(N), kBlock, 0, s>>>(N, L.t, x);
      count_launch(c, 3);
      lap("assemble");
      // the row structure is fixed within the solve: plan at the first iteration, then reuse
      dist_pcg_device(c, slabs, N, blocks, cols, rhs, x, p.pcg_tol, p.pcg_max_iters, &L, it == 0, &pr);
      lap("pcg");
      k_write_back<<<grid_for(N), kBlock, 0, s>>>(N, L.rows, L.frozen, x, L.deformed);
      count_launch(c);
    }
    run_level(c, L, pose, p, 2, l, nullptr, nullptr);  // update_rotations
    lap("rotations");
    wfk_trace_entry e{};
    e.level = l;
    e.iteration = it;
    run_level(c, L, pose, p, 1, l, nullptr, &e.energy);
    lap("energy");
    e.pcg_iterations = pr.iterations;
    e.pcg_residual = pr.relative_residual;
    e.anomaly = e.energy.total > prev.total + 1e-9 * prev.total ? 1 : 0;
    trace.push_back(e);
    const double rel = (prev.total - e.energy.total) / std::max(prev.total, 1e-300);
    prev = e.energy;
    if (rel >= 0 && rel < p.flip_flop_rel_tol) break;
  }
}

void solver_c2f_dist(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, int slabs,
                     std::vector<wfk_trace_entry>& trace) {
  require_volume(c);
  bind_level0(c);
  const PoseD pd = pose_dev(pose);
  build_hierarchy(c, p.levels);
  for (int l = p.levels - 1; l >= 1; --l) {
    dist_flip_flop(c, l, pd, p, slabs, trace);
    prolong(c, l);
  }
  dist_flip_flop(c, 0, pd, p, slabs, trace);
  sync_check(c);
}

void solver_hierarchy_info(wfk_ctx* c, int levels, int32_t* dims, int64_t* active) {
  require_volume(c);
  bind_level0(c);
  build_hierarchy(c, levels);
  for (int l = 0; l < levels; ++l) {
    Level& L = c->lv[l];
    if (dims) {
      dims[3 * l] = L.g.nx;
      dims[3 * l + 1] = L.g.ny;
      dims[3 * l + 2] = L.g.nz;
    }
    if (active) {
      level_rows(c, L);
      active[l] = L.N;
    }
  }
}

int solver_build_ne(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params& p, wfk_ne_host* out) {
  require_volume(c);
  bind_level0(c);
  Level& L = c->lv[0];
  const PoseD pd = pose_dev(pose);
  level_rows(c, L);
  level_constraints(c, L, pd, p);
  const int N = L.N;
  if (!out || N == 0) return N;
  cudaStream_t s = c->stream;
  double4* t = L.t;
  k_load_rows<<<grid_for(N), kBlock, 0, s>>>(N, L.rows, L.deformed, L.euler, t, L.rot);
  DevBuf<double> blocks;
  DevBuf<int32_t> cols;
  DevBuf<double> rhs;
  blocks.ensure(size_t(N) * 27 * 9);
  cols.ensure(size_t(N) * 27);
  rhs.ensure(size_t(N) * 3);
  k_ne_assemble_warp<<<grid_for(int64_t(N) * 32), kBlock, 0, s>>>(L.g, 0, N, L.rows, L.node_row, L.nbr, N, L.frozen,
                                                                  L.row_ptr, L.ent_con, L.ent_w, L.c_node, L.c_w,
                                                                  L.c_kind, L.c_g, L.rot, t, L.crhs, p.w_r, blocks,
                                                                  cols, rhs);
  count_launch(c, 2);
  WFK_CUDA(cudaGetLastError());
  if (out->rows) WFK_CUDA(cudaMemcpyAsync(out->rows, L.rows, size_t(N) * 4, cudaMemcpyDeviceToHost, s));
  if (out->node_row)
    WFK_CUDA(cudaMemcpyAsync(out->node_row, L.node_row, size_t(L.g.n()) * 4, cudaMemcpyDeviceToHost, s));
  if (out->blocks)
    WFK_CUDA(cudaMemcpyAsync(out->blocks, blocks, size_t(N) * 27 * 9 * 8, cudaMemcpyDeviceToHost, s));
  if (out->cols) WFK_CUDA(cudaMemcpyAsync(out->cols, cols, size_t(N) * 27 * 4, cudaMemcpyDeviceToHost, s));
  if (out->rhs) WFK_CUDA(cudaMemcpyAsync(out->rhs, rhs, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, s));
  if (out->frozen) WFK_CUDA(cudaMemcpyAsync(out->frozen, L.frozen, size_t(N), cudaMemcpyDeviceToHost, s));
  sync_check(c);
  return N;
}

void solver_pcg_assembled(wfk_ctx* c, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x,
                          double tol, int max_iters, int mode, wfk_pcg_result* res, double* y) {
  cudaStream_t s = c->stream;
  if (N <= 0) {
    if (res) *res = wfk_pcg_result{0, 0, 0.0};
    return;
  }
  DevBuf<double> B, X, R, P, AP, D, RHS;
  DevBuf<int32_t> CL;
  B.ensure(size_t(N) * 27 * 9);
  CL.ensure(size_t(N) * 27);
  X.ensure(size_t(N) * 3);
  R.ensure(size_t(N) * 3);
  P.ensure(size_t(N) * 3);
  AP.ensure(size_t(N) * 3);
  D.ensure(size_t(N) * 3);
  RHS.ensure(size_t(N) * 3);
  WFK_CUDA(cudaMemcpyAsync(B.p, blocks, size_t(N) * 27 * 9 * 8, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(CL.p, cols, size_t(N) * 27 * 4, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(X.p, x, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, s));
  if (rhs) WFK_CUDA(cudaMemcpyAsync(RHS.p, rhs, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, s));
  const int G = coop_blocks(c);
  AsmArgs a;
  a.N = N;
  a.blocks = B;
  a.cols = CL;
  a.rhs = RHS;
  a.x = X;
  a.r = R;
  a.p = P;
  a.ap = AP;
  a.dinv = D;
  a.tol = tol;
  a.max_iters = max_iters;
  a.mode = mode;
  a.partials = c->partials.ensure(size_t(8) * G);
  a.status = c->ivec.ensure(16) + 8;
  a.relres_out = c->dvec.ensure(8);
  void* args[] = {&a};
  WFK_CUDA(cudaLaunchCooperativeKernel((void*)k_pcg_assembled, dim3(G), dim3(kCoopBlock), args, 0, s));
  count_launch(c);
  if (mode == 1) {
    WFK_CUDA(cudaMemcpyAsync(y, AP.p, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, s));
    sync_check(c);
    return;
  }
  WFK_CUDA(cudaMemcpyAsync(x, X.p, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 8, a.status, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(reinterpret_cast<double*>(c->h_pinned + 16), a.relres_out, 8, cudaMemcpyDeviceToHost, s));
  sync_check(c);
  if (res) {
    res->iterations = c->h_pinned[8];
    res->relative_residual = reinterpret_cast<double*>(c->h_pinned + 16)[0];
  }
  c->stats.pcg_iterations += c->h_pinned[8];
}

}  // namespace wfk
