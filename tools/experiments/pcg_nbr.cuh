// EXPERIMENT, NOT BUILT (kept as a measured negative result).
// Replaced the PCG's grid barriers by per-block neighbour flags with
// block-contiguous row ownership; on the 128^3 bench it measured 31.4 ms/frame
// (hybrid: assembled levels only, 26.4) against 25.6 for the barrier-based
// pcg_pipe on the same box: the spatially contiguous partition is far less
// balanced than the snake-dealt global row order, the per-iteration reduction
// still couples every block, and the ownership setup adds ~0.1 ms per level.
// It was included into solver.cu after pcg_pipe (uses its helpers).
// Neighbour-synchronised pipelined Jacobi-PCG (pcg_variant 2) -- included by
// solver.cu after pcg_pipe, whose arithmetic it repeats exactly.
//
// pcg_pipe passes two grid barriers per iteration on the matrix-free level and
// one on assembled levels, each ~1.8 us plus the skew of the slowest block.
// Here every block owns a contiguous range of rows (lattice order, balanced by
// cost) and the constraints anchored at its rows, so the data a block reads in
// an iteration -- m of its rows' stencil neighbours and constraint anchors, and
// the incidence contributions of constraints owned elsewhere -- comes from a
// short interval of neighbouring blocks.  Grid barriers become per-block flags:
//   m flag: the block's m for iteration it is published (after its update),
//   c flag: the block's constraint contributions of iteration it are written,
// and a block waits only for the flags of the blocks it reads from
// (dependency intervals computed once per level solve).  The single reduction
// of an iteration goes through global warp 0 (block 0, warp 0), which polls
// the blocks' flag-embedded partials, sums them in fixed block order and
// publishes the totals; it never joins the worker barriers (named barrier 1).
// Flags and tags only grow within a launch (base = flip-flop iteration x
// (pcg_max + 2)), so no reset is needed between the PCG solves of a launch.
#pragma once

namespace wfk {

constexpr int kNbFlagStride = 32;  // u32 words between two blocks' flags (128 B)
constexpr size_t kNbSmemMax = 220 * 1024;

__device__ __forceinline__ void nb_spin_guard(long long t0) {
  // a dependency that never arrives is a bug; fail the launch instead of hanging the GPU
  if (clock64() - t0 > (1ll << 34)) __trap();
}

struct NbMap {
  int b, P0, nrows;   // block, first row id, rows owned
  int C0, ncons;      // first constraint (in nb_cord), constraints owned
  int wl, nwk;        // worker-warp index, worker warps (block 0 lends warp 0 to the reduction)
  int tw, ntw;        // worker-thread index, worker threads
  bool worker, comm;
};
__device__ __forceinline__ NbMap nb_map(const FFArgs& a) {
  NbMap m;
  m.b = blockIdx.x;
  m.P0 = a.nb_P[m.b];
  m.nrows = a.nb_P[m.b + 1] - m.P0;
  m.C0 = a.nb_CB ? a.nb_CB[m.b] : 0;
  m.ncons = a.nb_CB ? a.nb_CB[m.b + 1] - m.C0 : 0;
  const int w = threadIdx.x >> 5, skipw = m.b == 0 ? 1 : 0;
  m.worker = w >= skipw;
  m.comm = !m.worker;
  m.wl = w - skipw;
  m.nwk = int(blockDim.x >> 5) - skipw;
  m.tw = int(threadIdx.x) - 32 * skipw;
  m.ntw = int(blockDim.x) - 32 * skipw;
  return m;
}
// worker-only block barrier
__device__ __forceinline__ void nb_wsync(const NbMap& m) { asm volatile("bar.sync 1, %0;" ::"r"(m.ntw) : "memory"); }
// round k of worker warp wl: dealt in order, or in snake order for rows sorted by cost
__device__ __forceinline__ int nb_round(int k, const NbMap& m, bool snake) {
  return k * m.nwk + ((snake && (k & 1)) ? m.nwk - 1 - m.wl : m.wl);
}

// shared-memory layout: row-state slots (8 padded vectors), matrix-free row
// metadata, assembled B^T B rows, matrix-free constraint metadata
struct NbLayout {
  int scap, sccap;
  size_t rmeta, amat, cmeta, total;
};
__host__ __device__ inline NbLayout nb_layout(int scap, int sccap, bool mf, bool asm_level) {
  NbLayout l;
  l.scap = scap;
  l.sccap = mf ? sccap : 0;
  size_t off = size_t(kSlotVecs) * scap * sizeof(double4);
  l.rmeta = off;
  if (mf) off += size_t(scap) * (2 * sizeof(int4) + 2 * sizeof(int));
  off = (off + 31) / 32 * 32;
  l.amat = off;
  if (asm_level) off += size_t(scap) * 27 * (6 * sizeof(double) + sizeof(int));
  off = (off + 31) / 32 * 32;
  l.cmeta = off;
  if (mf) off += size_t(l.sccap) * (3 * sizeof(double4) + 4 * sizeof(int4) + sizeof(int));
  l.total = off;
  return l;
}

struct NbSm {
  double4* st;  // kSlotVecs x scap
  int scap, sccap;
  int4 *rm, *rn;
  int *rn5, *rid;
  double* blk;
  int* cols;
  double4 *cw, *cg;
  int4 *crow, *cpos;
  int* ckind;
};
__device__ inline NbSm nb_sm(char* base, const NbLayout& l) {
  NbSm s;
  s.st = reinterpret_cast<double4*>(base);
  s.scap = l.scap;
  s.sccap = l.sccap;
  char* r = base + l.rmeta;
  s.rm = reinterpret_cast<int4*>(r);
  s.rn = reinterpret_cast<int4*>(r + size_t(l.scap) * sizeof(int4));
  s.rn5 = reinterpret_cast<int*>(r + size_t(l.scap) * 2 * sizeof(int4));
  s.rid = reinterpret_cast<int*>(r + size_t(l.scap) * (2 * sizeof(int4) + sizeof(int)));
  s.blk = reinterpret_cast<double*>(base + l.amat);
  s.cols = reinterpret_cast<int*>(base + l.amat + size_t(l.scap) * 27 * 6 * sizeof(double));
  char* c = base + l.cmeta;
  const size_t SC = size_t(l.sccap);
  s.cw = reinterpret_cast<double4*>(c);
  s.cg = reinterpret_cast<double4*>(c + 2 * SC * sizeof(double4));
  s.crow = reinterpret_cast<int4*>(c + 3 * SC * sizeof(double4));
  s.cpos = reinterpret_cast<int4*>(c + 3 * SC * sizeof(double4) + 2 * SC * sizeof(int4));
  s.ckind = reinterpret_cast<int*>(c + 3 * SC * sizeof(double4) + 4 * SC * sizeof(int4));
  return s;
}

// row-state access: shared-memory slot, or the row-indexed global vectors for
// slots beyond the shared capacity
__device__ __forceinline__ double4* nb_gvec(const FFArgs& a, int v) {
  switch (v) {
    case kSx: return a.x;
    case kSr: return a.r;
    case kSw: return a.w;
    case kSp: return a.p;
    case kSs: return a.ap;
    case kSz: return a.z;
    case kSd: return a.dinv;
    default: return a.nbuf;
  }
}
__device__ __forceinline__ double4 nb_get(const FFArgs& a, const NbSm& s, int v, int q, int r) {
  return q < s.scap ? s.st[v * s.scap + q] : ld4w(nb_gvec(a, v), r);
}
__device__ __forceinline__ void nb_put(const FFArgs& a, const NbSm& s, int v, int q, int r, double4 x) {
  if (q < s.scap)
    s.st[v * s.scap + q] = x;
  else
    st4w(nb_gvec(a, v), r, x);
}
__device__ __forceinline__ V3 v3of(double4 d) { return {d.x, d.y, d.z}; }
__device__ __forceinline__ double4 d4of(V3 v) { return make_double4(v.x, v.y, v.z, 0.0); }

// row id of the block's position q
__device__ __forceinline__ int nb_row(const FFArgs& a, const NbMap& m, const NbSm& s, int q, bool mf) {
  if (mf && q < s.scap) return s.rid[q];
  return a.nb_ord ? a.nb_ord[m.P0 + q] : m.P0 + q;
}

// the block's rows as (row, slot) with every lane of the owning warp busy
// (rounds of RPW rows as in the row passes, 32 / RPW rounds per step)
template <int RPW, class F>
__device__ __forceinline__ void nb_each_row(const FFArgs& a, const NbMap& m, const NbSm& s, bool mf, F f) {
  if (!m.worker) return;
  __syncwarp();
  constexpr int RPS = 32 / RPW;
  const int lane = threadIdx.x & 31;
  for (int k = lane / RPW;; k += RPS) {
    const int p0 = nb_round(k, m, mf) * RPW;
    if (p0 >= m.nrows) break;  // rounds grow with k
    const int q = p0 + lane % RPW;
    if (q < m.nrows) f(nb_row(a, m, s, q, mf), q);
  }
}

// matrix-free: constraint pass over the block's constraints
__device__ __forceinline__ void nb_constraints(const FFArgs& a, const NbMap& m, const NbSm& s, const double4* v) {
  if (!m.worker) return;
  for (int j = m.tw; j < m.ncons; j += m.ntw) {
    int rows[8];
    double w[8];
    double4 gc;
    int kind;
    int4 p0, p1;
    if (j < s.sccap) {
      const int4 r0 = s.crow[j], r1 = s.crow[s.sccap + j];
      const double4 w0 = s.cw[j], w1 = s.cw[s.sccap + j];
      rows[0] = r0.x; rows[1] = r0.y; rows[2] = r0.z; rows[3] = r0.w;
      rows[4] = r1.x; rows[5] = r1.y; rows[6] = r1.z; rows[7] = r1.w;
      w[0] = w0.x; w[1] = w0.y; w[2] = w0.z; w[3] = w0.w;
      w[4] = w1.x; w[5] = w1.y; w[6] = w1.z; w[7] = w1.w;
      gc = s.cg[j];
      kind = s.ckind[j];
      p0 = s.cpos[j];
      p1 = s.cpos[s.sccap + j];
    } else {
      const int64_t c = a.nb_cord[m.C0 + j];
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

// matrix-free row pass (kMfLanes lanes per row) over the block's rows, rounds
// in snake order over its worker warps; sink(row, slot, v_r, (A v)_r)
template <class Sink>
__device__ __forceinline__ void nb_row_pass_mf(const FFArgs& a, const NbMap& m, const NbSm& s, const double4* v,
                                               Sink& sink) {
  constexpr int L = kMfLanes, RPW = 32 / L;
  if (!m.worker) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L, grp = lane / L;
  const double w2 = 2.0 * a.w_r;
  for (int k = 0;; ++k) {
    const int p0 = nb_round(k, m, true) * RPW;
    if (p0 >= m.nrows) break;
    const int q = p0 + grp;
    const bool live = q < m.nrows;
    int r = 0, e0 = 0, e1 = 0, nb[6] = {-1, -1, -1, -1, -1, -1};
    bool frozen = false;
    if (live) {
      if (q < s.scap) {
        const int4 m0 = s.rm[q], m1 = s.rn[q];
        e0 = m0.x;
        e1 = m0.y;
        frozen = m0.z != 0;
        nb[0] = m0.w; nb[1] = m1.x; nb[2] = m1.y; nb[3] = m1.z; nb[4] = m1.w;
        nb[5] = s.rn5[q];
        r = s.rid[q];
      } else {
        r = a.nb_ord ? a.nb_ord[m.P0 + q] : m.P0 + q;
        frozen = a.frozen[r];
        e0 = a.row_ptr[r];
        e1 = a.row_ptr[r + 1];
#pragma unroll
        for (int k2 = sub; k2 < 6; k2 += L) nb[k2] = a.nbr[int64_t(k2) * a.N + r];
      }
    }
    const V3 vr = live ? ld4(v, r) : V3{0, 0, 0};
    V3 acc{0, 0, 0};
    if (live && !frozen) {
      for (int e = e0 + sub; e < e1; e += L) acc += ld4(a.contrib, e);
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

// assembled row pass (kAsmLanes lanes per row, 27-slot stencil) over the block's rows
template <class Sink>
__device__ __forceinline__ void nb_row_pass_asm(const FFArgs& a, const NbMap& m, const NbSm& s, const double4* v,
                                                Sink& sink) {
  constexpr int L = kAsmLanes, RPW = 32 / L;
  if (!m.worker) return;
  const int lane = threadIdx.x & 31;
  const int sub = lane % L, grp = lane / L;
  const double w2 = 2.0 * a.w_r;
  for (int k = 0;; ++k) {
    const int p0 = nb_round(k, m, false) * RPW;
    if (p0 >= m.nrows) break;
    const int q = p0 + grp;
    const bool live = q < m.nrows;
    const int r = m.P0 + q;
    const bool frozen = live && a.frozen[r];
    const V3 vr = live ? ld4(v, r) : V3{0, 0, 0};
    V3 acc{0, 0, 0};
    if (live && !frozen) {
      const double* bb = q < s.scap ? s.blk + q * 27 * 6 : a.blk + int64_t(r) * 27 * 6;
      const int* cc = q < s.scap ? s.cols + q * 27 : a.cols + int64_t(r) * 27;
#pragma unroll
      for (int sl = sub; sl < 27; sl += L) {
        const int col = cc[sl];
        if (col < 0) continue;
        const V3 x = ld4(v, col);
        const double* b = bb + sl * 6;  // xx xy xz yy yz zz
        acc.x += b[0] * x.x + b[1] * x.y + b[2] * x.z;
        acc.y += b[1] * x.x + b[3] * x.y + b[4] * x.z;
        acc.z += b[2] * x.x + b[4] * x.y + b[5] * x.z;
        if (sl == 4 || sl == 10 || sl == 12 || sl == 14 || sl == 16 || sl == 22) acc += w2 * (vr - x);
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

// wait until flags[d] >= target for every block d in [lo, hi] (acquire), then worker barrier
__device__ __forceinline__ void nb_wait(const NbMap& m, const unsigned* flags, int lo, int hi, unsigned target) {
  if (m.worker && m.tw <= hi - lo) {
    const unsigned* f = flags + size_t(lo + m.tw) * kNbFlagStride;
    const long long t0 = clock64();
    while (ld_acquire_u32(f) < target) nb_spin_guard(t0);
  }
  nb_wsync(m);
}
// worker barrier (all of the block's writes done), then release the block's flag
__device__ __forceinline__ void nb_signal(const NbMap& m, unsigned* flags, unsigned value) {
  nb_wsync(m);
  if (m.worker && m.tw == 0) st_release_u32(flags + size_t(m.b) * kNbFlagStride, value);
}

// block partials of the workers -> flag-embedded words {32-bit half, tag},
// and (one worker barrier for both) the release of the block's m flag
__device__ __forceinline__ void nb_publish(const FFArgs& a, const NbMap& m, double (&v)[3], unsigned tag,
                                           unsigned* mflag) {
  __shared__ double sm3[3][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) sm3[k][w] = v[k];
  nb_wsync(m);  // every worker's update (m, partials) is done
  if (m.worker && m.tw == 0) st_release_u32(mflag + size_t(m.b) * kNbFlagStride, tag);
  if (m.wl == 0) {  // first worker warp: fixed-order block sum
    const int w0 = int(blockDim.x >> 5) - m.nwk;
    double t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) t[k] = warp_sum(lane < m.nwk ? sm3[k][w0 + lane] : 0.0);
    if (lane < 6) {
      double tv = t[0];
      if ((lane >> 1) == 1) tv = t[1];
      if ((lane >> 1) == 2) tv = t[2];
      const unsigned long long bits = (unsigned long long)__double_as_longlong(tv);
      const unsigned half = (lane & 1) ? unsigned(bits >> 32) : unsigned(bits);
      st_relaxed_u64(a.nb_part + size_t(m.b) * 8 + lane, (unsigned long long)half << 32 | tag);
    }
  }
}

// global warp 0: wait for every block's partials of `tag`, sum them in fixed
// block order, publish the totals (flag-embedded) and return them
__device__ __forceinline__ void nb_comm_total(const FFArgs& a, unsigned tag, double (&out)[3]) {
  const int lane = threadIdx.x & 31;
  double t[3] = {0, 0, 0};
  const long long t0 = clock64();
  // every lane polls all its blocks' words at once (one round trip per poll)
  constexpr int J = 5;  // blocks per lane: up to 160 blocks
  unsigned long long x[J][6];
  unsigned done = 0;  // bit j: block lane + 32 j complete
  unsigned need = 0;
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (lane + 32 * j < int(gridDim.x)) need |= 1u << j;
  while (done != need) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!(need & ~done & (1u << j))) continue;
#pragma unroll
      for (int k = 0; k < 6; ++k) x[j][k] = ld_relaxed_u64(a.nb_part + size_t(lane + 32 * j) * 8 + k);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!(need & ~done & (1u << j))) continue;
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 6; ++k) ok &= unsigned(x[j][k]) == tag;
      if (ok) done |= 1u << j;
    }
    if (done != need) nb_spin_guard(t0);
  }
#pragma unroll
  for (int j = 0; j < J; ++j)
    if (need & (1u << j))
#pragma unroll
      for (int k = 0; k < 3; ++k)
        t[k] += __longlong_as_double((long long)((x[j][2 * k + 1] >> 32) << 32 | (x[j][2 * k] >> 32)));
  for (int b = lane + 32 * J; b < int(gridDim.x); b += 32) {  // beyond 160 blocks: one at a time
    unsigned long long y[6];
    bool ok;
    do {
#pragma unroll
      for (int k = 0; k < 6; ++k) y[k] = ld_relaxed_u64(a.nb_part + size_t(b) * 8 + k);
      ok = true;
#pragma unroll
      for (int k = 0; k < 6; ++k) ok &= unsigned(y[k]) == tag;
      if (!ok) nb_spin_guard(t0);
    } while (!ok);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      t[k] += __longlong_as_double((long long)((y[2 * k + 1] >> 32) << 32 | (y[2 * k] >> 32)));
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) t[k] = warp_sum(t[k]);
  if (lane < 6) {
    double tv = t[0];
    if ((lane >> 1) == 1) tv = t[1];
    if ((lane >> 1) == 2) tv = t[2];
    const unsigned long long bits = (unsigned long long)__double_as_longlong(tv);
    const unsigned half = (lane & 1) ? unsigned(bits >> 32) : unsigned(bits);
    st_relaxed_u64(a.sync_ll + lane, (unsigned long long)half << 32 | tag);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) out[k] = t[k];
}
// workers: wait for the totals of `tag`
__device__ __forceinline__ void nb_totals(const FFArgs& a, const NbMap& m, unsigned tag, double (&v)[3]) {
  __shared__ double bc[3];
  const int lane = threadIdx.x & 31;
  if (m.wl == 0) {
    unsigned half = 0;
    if (lane < 6) {
      const long long t0 = clock64();
      unsigned long long x;
      do {
        x = ld_relaxed_u64(a.sync_ll + lane);
        if (unsigned(x) != tag) nb_spin_guard(t0);
      } while (unsigned(x) != tag);
      half = unsigned(x >> 32);
    }
    const unsigned hi = __shfl_down_sync(0xffffffffu, half, 1);
    if (lane < 6 && !(lane & 1)) bc[lane >> 1] = __longlong_as_double((long long)((unsigned long long)hi << 32 | half));
  }
  nb_wsync(m);
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = bc[k];
}

// pcg_solve (solver.cpp:282-343), pipelined as pcg_pipe, neighbour-synchronised
template <bool ASM>
__device__ void pcg_nbr(const FFArgs& a, Red& rs, int& iters, double& relres, unsigned base) {
  extern __shared__ double4 dyn_smem[];
  iters = 0;
  relres = 0;
  PhaseClock pc(a.dbg, blockIdx.x == 0 ? 32u : 0u);  // block 0's thread 0 is the reduction warp
  constexpr bool MF = !ASM;
  constexpr int RPW = 32 / (ASM ? kAsmLanes : kMfLanes);
  const NbMap m = nb_map(a);
  const NbLayout lay = nb_layout(a.nb_scap, a.nb_sccap, MF, ASM);
  const NbSm s = nb_sm(reinterpret_cast<char*>(dyn_smem), lay);
  // the solve-fixed data into shared memory: row metadata and constraint
  // metadata (matrix-free) or the rows of B^T B (assembled)
  if (MF) {
    nb_each_row<RPW>(a, m, s, false, [&](int, int q) {
      if (q >= s.scap) return;
      const int r = a.nb_ord ? a.nb_ord[m.P0 + q] : m.P0 + q;
      int nb[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) nb[k] = a.nbr[int64_t(k) * a.N + r];
      s.rid[q] = r;
      s.rm[q] = make_int4(a.row_ptr[r], a.row_ptr[r + 1], a.frozen[r], nb[0]);
      s.rn[q] = make_int4(nb[1], nb[2], nb[3], nb[4]);
      s.rn5[q] = nb[5];
    });
    if (m.worker)
      for (int j = m.tw; j < m.ncons && j < s.sccap; j += m.ntw) {
        const int64_t c = a.nb_cord[m.C0 + j];
        s.crow[j] = a.c_row[2 * c];
        s.crow[s.sccap + j] = a.c_row[2 * c + 1];
        s.cw[j] = ld4w(a.c_w, 2 * c);
        s.cw[s.sccap + j] = ld4w(a.c_w, 2 * c + 1);
        s.cpos[j] = a.c_pos[2 * c];
        s.cpos[s.sccap + j] = a.c_pos[2 * c + 1];
        s.cg[j] = ld4w(a.c_g, c);
        s.ckind[j] = a.c_kind[c];
      }
  } else if (m.worker) {
    const int lane = threadIdx.x & 31;
    for (int k = 0;; ++k) {
      const int p0 = nb_round(k, m, false) * RPW;
      if (p0 >= m.nrows) break;
      for (int j = 0; j < RPW; ++j) {
        const int q = p0 + j;
        if (q >= m.nrows || q >= s.scap) break;
        const int r = m.P0 + q;
        for (int t = lane; t < 27 * 6; t += 32) s.blk[q * 27 * 6 + t] = a.blk[int64_t(r) * 27 * 6 + t];
        if (lane < 27) s.cols[q * 27 + lane] = a.cols[int64_t(r) * 27 + lane];
      }
    }
  }
  __syncthreads();
  // sinks receive (row, slot, v_r, (A v)_r)
  auto matvec_all = [&](const double4* v, auto& sink) {
    if (ASM) {
      nb_row_pass_asm(a, m, s, v, sink);
    } else {
      nb_constraints(a, m, s, v);
      grid_barrier(a, rs);
      nb_row_pass_mf(a, m, s, v, sink);
    }
  };
  // r0 = b - A x0, u0 = D^-1 r0 (solver.cpp:305-310)
  double acc_rr = 0, acc_bb = 0;
  auto init_sink = [&](int r, int q, V3 xr, V3 ax) {
    const V3 b = ld4(a.rhs, r);
    const V3 rr = b - ax;
    const double4 d4 = ld4w(a.dinv, r);
    st4(a.u, r, cmul(v3of(d4), rr));
    const double4 zero = make_double4(0, 0, 0, 0);
    nb_put(a, s, kSx, q, r, d4of(xr));
    nb_put(a, s, kSr, q, r, d4of(rr));
    nb_put(a, s, kSp, q, r, zero);
    nb_put(a, s, kSs, q, r, zero);
    nb_put(a, s, kSz, q, r, zero);
    nb_put(a, s, kSd, q, r, d4);
    acc_rr += dot(rr, rr);
    acc_bb += sqnorm(b);
  };
  matvec_all(a.x, init_sink);
  grid_barrier(a, rs);
  // w0 = A u0, m0 = D w0
  double v4[4] = {0, 0, 0, 0};
  auto w_sink = [&](int r, int q, V3 ur, V3 wr) {
    const V3 d = v3of(nb_get(a, s, kSd, q, r)), rq = v3of(nb_get(a, s, kSr, q, r));
    nb_put(a, s, kSw, q, r, d4of(wr));
    st4(a.m0, r, cmul(d, wr));
    v4[0] += dot(rq, ur);
    v4[1] += dot(wr, ur);
  };
  matvec_all(a.u, w_sink);
  v4[2] = acc_rr;
  v4[3] = acc_bb;
  grid_reduce<4>(a, rs, v4);  // also publishes m0 to every block
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
  bool pending = false;  // totals of the last update not yet read
  const int* dep = a.nb_dep;
  const int G = gridDim.x;
  unsigned* mflag = a.nb_flags;
  unsigned* cflag = a.nb_flags + size_t(G) * kNbFlagStride;
  pc.lap(12);
  if (m.comm) {
    // global warp 0: the reductions, mirroring the workers' control flow
    for (int it = 0; it < a.pcg_max; ++it) {
      if (pending) {
        double v3[3];
        nb_comm_total(a, base + unsigned(it), v3);
        gamma_prev = gamma;
        gamma = v3[0];
        delta = v3[1];
        r_norm = sqrt(v3[2]);
        relres = r_norm / b_norm;
        pending = false;
      }
      if (!(r_norm > stop)) break;
      const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
      const double pap = it == 0 ? delta : delta - beta * gamma / alpha_prev;
      if (pap <= 0) break;
      alpha_prev = gamma / pap;
      pending = true;
      iters = it + 1;
    }
    if (pending) {
      double v3[3];
      nb_comm_total(a, base + unsigned(iters), v3);
      r_norm = sqrt(v3[2]);
      relres = r_norm / b_norm;
    }
  } else {
    const int lo_m = dep[m.b], hi_m = dep[G + m.b], lo_c = dep[2 * G + m.b], hi_c = dep[3 * G + m.b];
    for (int it = 0; it < a.pcg_max; ++it) {
      const double4* mcur = (it & 1) ? a.m1 : a.m0;
      double4* mnext = (it & 1) ? a.m0 : a.m1;
      const unsigned tag = base + unsigned(it) + 1u;
      auto n_sink = [&](int r, int q, V3, V3 n) { nb_put(a, s, kSn, q, r, d4of(n)); };
      if (it > 0) nb_wait(m, mflag, lo_m, hi_m, tag - 1u);  // neighbours' m of this iteration
      pc.lap(1);
      if (ASM) {
        nb_row_pass_asm(a, m, s, mcur, n_sink);
      } else {
        nb_constraints(a, m, s, mcur);
        nb_signal(m, cflag, tag);
        pc.lap(0);
        nb_wait(m, cflag, lo_c, hi_c, tag);  // contributions to the block's rows
        pc.lap(5);
        nb_row_pass_mf(a, m, s, mcur, n_sink);
      }
      pc.lap(2);
      if (pending) {
        double v3[3];
        nb_totals(a, m, tag - 1u, v3);
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
      nb_each_row<RPW>(a, m, s, MF, [&](int r, int q) {
        const V3 d = v3of(nb_get(a, s, kSd, q, r));
        const V3 w = v3of(nb_get(a, s, kSw, q, r));
        V3 rr = v3of(nb_get(a, s, kSr, q, r));
        const V3 z = v3of(nb_get(a, s, kSn, q, r)) + beta * v3of(nb_get(a, s, kSz, q, r));
        const V3 sv = w + beta * v3of(nb_get(a, s, kSs, q, r));
        const V3 p = cmul(d, rr) + beta * v3of(nb_get(a, s, kSp, q, r));
        const V3 x = v3of(nb_get(a, s, kSx, q, r)) + alpha * p;
        rr = rr - alpha * sv;
        const V3 wn = w - alpha * z;
        const V3 u = cmul(d, rr);
        nb_put(a, s, kSz, q, r, d4of(z));
        nb_put(a, s, kSs, q, r, d4of(sv));
        nb_put(a, s, kSp, q, r, d4of(p));
        nb_put(a, s, kSx, q, r, d4of(x));
        nb_put(a, s, kSr, q, r, d4of(rr));
        nb_put(a, s, kSw, q, r, d4of(wn));
        st4(mnext, r, cmul(d, wn));
        v3[0] += dot(rr, u);
        v3[1] += dot(wn, u);
        v3[2] += dot(rr, rr);
      });
      pc.lap(4);
      nb_publish(a, m, v3, tag, mflag);  // partials + this block's m of the next iteration
      pc.lap(7);
      pc.count(15);
      alpha_prev = alpha;
      pending = true;
      iters = it + 1;
    }
    if (pending) {
      double v3[3];
      nb_totals(a, m, base + unsigned(iters) + 0u, v3);
      r_norm = sqrt(v3[2]);
      relres = r_norm / b_norm;
    }
  }
  // the solution back to global memory for the write-back phase
  nb_each_row<RPW>(a, m, s, MF, [&](int r, int q) { st4w(a.x, r, nb_get(a, s, kSx, q, r)); });
  grid_barrier(a, rs);
}

// ---------------------------------------------------------------------------
// setup: ownership, row / constraint order, dependency intervals
// ---------------------------------------------------------------------------
// cost of a row: matrix-free incidences + c0, assembled 1
__global__ void k_nb_cost(int N, const int32_t* row_ptr, int c0, int64_t* cost) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x)
    cost[r] = row_ptr ? int64_t(row_ptr[r + 1] - row_ptr[r]) + c0 : 1;
}
// P[b] = first row whose exclusive cost prefix reaches block b's share
// (block 0 lends one of its warps to the reduction: 15/16 of a share)
__global__ void k_nb_partition(int N, int G, int wpb, const int64_t* incl, int32_t* P) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > G) return;
  if (b == 0 || N == 0) {
    P[b] = b == 0 ? 0 : N;
    return;
  }
  if (b == G) {
    P[b] = N;
    return;
  }
  const double total = double(incl[N - 1]);
  const double share = double(b) - 1.0 / wpb;
  const double target = total * share / (double(G) - 1.0 / wpb);
  // first r with exclusive prefix (incl[r] - cost[r] = incl[r - 1]) >= target
  int lo = 0, hi = N;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    const double excl = mid == 0 ? 0.0 : double(incl[mid - 1]);
    if (excl >= target)
      hi = mid;
    else
      lo = mid + 1;
  }
  P[b] = lo;
}
__device__ __forceinline__ int nb_owner_of(const int32_t* P, int G, int r) {
  int lo = 0, hi = G - 1;  // last b with P[b] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (P[mid] <= r)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}
__global__ void k_nb_owner(int N, int G, const int32_t* P, int32_t* owner) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) owner[r] = nb_owner_of(P, G, r);
}
// matrix-free row order: by owner, then decreasing incidences (stable)
__global__ void k_nb_row_keys(int N, const int32_t* owner, const int32_t* row_ptr, int32_t* key, int32_t* val) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    key[r] = owner[r] * 65536 + (65535 - min(row_ptr[r + 1] - row_ptr[r], 65535));
    val[r] = r;
  }
}
// constraint owner: the block of its first anchor row (G: no anchor row)
__global__ void k_nb_cons_keys(int64_t C, int G, const int4* c_row, const int32_t* owner, int32_t* key, int32_t* val) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < C; c += int64_t(gridDim.x) * blockDim.x) {
    const int4 r0 = c_row[2 * c], r1 = c_row[2 * c + 1];
    const int rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    int o = G;
    for (int k = 0; k < 8; ++k)
      if (rr[k] >= 0) {
        o = owner[rr[k]];
        break;
      }
    key[c] = o;
    val[c] = int32_t(c);
  }
}
// Constraint ranges: the owner-sorted list (lattice order of the first anchor
// row, so ranges stay spatially local) cut into G equal parts; constraints
// without an anchor row (key G, sorted last) are not processed.
__global__ void k_nb_cons_ranges(int64_t C, int G, const int32_t* sorted_key, int32_t* CB) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > G) return;
  int64_t lo = 0, hi = C;  // number of constraints with an anchor row
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (sorted_key[mid] >= G)
      hi = mid;
    else
      lo = mid + 1;
  }
  CB[b] = int32_t(lo * b / G);
}
__global__ void k_nb_dep_init(int G, int32_t* dep) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < G; b += gridDim.x * blockDim.x) {
    dep[b] = b;          // lo_m
    dep[G + b] = b;      // hi_m
    dep[2 * G + b] = b;  // lo_c
    dep[3 * G + b] = b;  // hi_c
  }
}
__device__ __forceinline__ void nb_dep_m(int32_t* dep, int G, int b, int o) {
  atomicMin(&dep[b], o);
  atomicMax(&dep[G + b], o);
}
__device__ __forceinline__ void nb_dep_c(int32_t* dep, int G, int b, int o) {
  atomicMin(&dep[2 * G + b], o);
  atomicMax(&dep[3 * G + b], o);
}
// rows: m of the face neighbours (matrix-free) or of the 27 stencil columns (assembled)
__global__ void k_nb_dep_rows(int N, int G, const int32_t* owner, const int32_t* nbr, const int32_t* cols,
                              int32_t* dep) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    const int b = owner[r];
    if (cols) {
      for (int s = 0; s < 27; ++s) {
        const int j = cols[int64_t(r) * 27 + s];
        if (j >= 0) nb_dep_m(dep, G, b, owner[j]);
      }
    } else {
      for (int k = 0; k < 6; ++k) {
        const int j = nbr[int64_t(k) * N + r];
        if (j >= 0) nb_dep_m(dep, G, b, owner[j]);
      }
    }
  }
}
// constraints: the owner reads m at every anchor row; each anchor row's block
// reads the owner's contributions
__global__ void k_nb_dep_cons(int64_t C, int G, const int4* c_row, const int4* c_pos, const int32_t* owner,
                              const int32_t* CB, const int32_t* cord, int32_t* dep) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < C; j += int64_t(gridDim.x) * blockDim.x) {
    if (j >= CB[G]) continue;
    const int o = nb_owner_of(CB, G, int(j));
    const int64_t c = cord[j];
    const int4 r0 = c_row[2 * c], r1 = c_row[2 * c + 1];
    const int4 p0 = c_pos[2 * c], p1 = c_pos[2 * c + 1];
    const int rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const int pp[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
    for (int k = 0; k < 8; ++k) {
      if (rr[k] < 0) continue;
      const int ob = owner[rr[k]];
      nb_dep_m(dep, G, o, ob);
      if (pp[k] >= 0) nb_dep_c(dep, G, ob, o);
    }
  }
}

}  // namespace wfk
