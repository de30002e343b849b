// Slab-partitioned Jacobi-PCG over the normal equations:
// pcg_solve (solver.cpp:282-343) with the rows split into contiguous ranges,
// one per rank.  Rows are in ascending lattice order (solver.cpp:113-161), so
// a contiguous row range is a z-slab of the lattice and the 27-point stencil
// couples it only to the adjacent planes.  Per iteration a rank applies A to
// its own rows, exchanges the halo rows of p with the ranks that own them and
// all-gathers its partial dot products; every rank sums the gathered partials
// in rank order, so the scalars (and hence the iterates) are identical on all
// ranks and independent of the transport.
//
// Two transports run the same kernels:
//   * NCCL (one process per GPU): grouped ncclSend/ncclRecv for the halo,
//     ncclAllGather for the partials, grouped ncclBroadcast for the final x.
//     NCCL is loaded at run time (dlopen "libnccl.so.2"), so libwfk has no
//     link-time dependency and shares torch's NCCL when torch is loaded.
//   * slabs (one process, one GPU, S slab states): the same halo plan executed
//     with device-to-device copies -- the single-GPU test of the partition.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"

namespace wfk {

// ---------------------------------------------------------------------------
// NCCL, resolved at run time
// ---------------------------------------------------------------------------
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) {
    if (!api.h) throw Error(WFK_E_NCCL, "libnccl.so.2 could not be loaded");
    return api;
  }
  tried = true;
  api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) throw Error(WFK_E_NCCL, std::string("dlopen libnccl.so.2: ") + dlerror());
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.h, name));
    if (!fn) throw Error(WFK_E_NCCL, std::string("NCCL symbol missing: ") + name);
  };
  sym(api.GetUniqueId, "ncclGetUniqueId");
  sym(api.CommInitRank, "ncclCommInitRank");
  sym(api.CommDestroy, "ncclCommDestroy");
  sym(api.Send, "ncclSend");
  sym(api.Recv, "ncclRecv");
  sym(api.AllGather, "ncclAllGather");
  sym(api.Broadcast, "ncclBroadcast");
  sym(api.GroupStart, "ncclGroupStart");
  sym(api.GroupEnd, "ncclGroupEnd");
  sym(api.GetErrorString, "ncclGetErrorString");
  return api;
}

#define WFK_NCCL(call)                                                                          \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess) throw ::wfk::Error(WFK_E_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct DistComm {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  ~DistComm() {
    if (comm) nccl().CommDestroy(comm);
  }
};

void dist_forget(wfk_ctx* c);

// drops the communicator AND every captured iteration of this context: the
// graphs hold NCCL nodes bound to the communicator being destroyed
void dist_destroy(wfk_ctx* c) {
  dist_forget(c);
  delete c->dist;
  c->dist = nullptr;
}

// ---------------------------------------------------------------------------
// the partition plan (host; also exported for tests)
// ---------------------------------------------------------------------------
struct Xfer {
  int src, dst, lo, hi;  // rows [lo, hi) owned by src, needed by dst
};
struct DistPlan {
  int world = 1;
  std::vector<int> lo, hi;
  std::vector<Xfer> xfers;
};

// contiguous balanced row ranges; the halo of a range is every row outside it
// that a row inside references (col_min / col_max per row), as ranges
// [min_ref, lo) and [hi, max_ref] split over their owners
static DistPlan make_plan(int N, const int32_t* col_min, const int32_t* col_max, int world) {
  DistPlan p;
  p.world = world;
  for (int k = 0; k < world; ++k) {
    p.lo.push_back(int(int64_t(N) * k / world));
    p.hi.push_back(int(int64_t(N) * (k + 1) / world));
  }
  for (int k = 0; k < world; ++k) {
    int mn = p.lo[k], mx = p.hi[k] - 1;
    for (int r = p.lo[k]; r < p.hi[k]; ++r) {
      if (col_min[r] >= 0) mn = std::min(mn, int(col_min[r]));
      mx = std::max(mx, int(col_max[r]));
    }
    const int need[2][2] = {{mn, p.lo[k]}, {p.hi[k], mx + 1}};
    for (const auto& nd : need)
      for (int j = 0; j < world; ++j) {
        if (j == k) continue;
        const int a = std::max(nd[0], p.lo[j]), b = std::min(nd[1], p.hi[j]);
        if (a < b) p.xfers.push_back({j, k, a, b});
      }
  }
  return p;
}

// ---------------------------------------------------------------------------
// kernels: one slab's rows [lo, hi) of full-length vectors
// ---------------------------------------------------------------------------
constexpr int kDBlock = 256;
constexpr int kDMaxBlocks = 512;
constexpr int kDK = 4;  // partial values per reduction

struct DSlab {
  int lo, hi;
  const double* blocks;  // N x 27 x 9 (row-major 3x3)
  const int32_t* cols;   // N x 27
  const double* rhs;
  double *x, *r, *z, *p, *ap, *dinv;
  double* part;   // kDK x kDMaxBlocks block partials
  double* gath;   // world x kDK gathered slab partials
  double* st;     // scalars: see DS_*
};
enum { DS_RZ, DS_RNORM, DS_BNORM, DS_STOP, DS_ALPHA, DS_BETA, DS_DONE, DS_ITERS, DS_RELRES, DS_N };

__device__ __forceinline__ V3 d_row(const DSlab& a, const double* v, int r) {
  V3 acc{0, 0, 0};
  for (int s = 0; s < 27; ++s) {
    const int c = a.cols[27 * int64_t(r) + s];
    if (c >= 0) acc += mul(ld_m3(a.blocks, 27 * int64_t(r) + s), ld3(v, c));
  }
  return acc;
}

template <int NV>
__device__ void d_block_partials(const DSlab& a, double (&v)[NV]) {
  __shared__ double smem[NV * 32];
  block_sum<NV>(v, smem);
  if (threadIdx.x == 0)
    for (int k = 0; k < NV; ++k) a.part[k * kDMaxBlocks + blockIdx.x] = v[k];
}

// r = b - A x, z = D^-1 r, p = z; partials {r.z, r.r, b.b} (solver.cpp:289-321)
__global__ void __launch_bounds__(kDBlock) k_d_init(DSlab a) {
  double v[3] = {0, 0, 0};
  for (int r = a.lo + blockIdx.x * kDBlock + threadIdx.x; r < a.hi; r += gridDim.x * kDBlock) {
    const M3 d = ld_m3(a.blocks, 27 * int64_t(r) + kCenter);
    const V3 di{d.a[0][0] > 1e-300 ? 1.0 / d.a[0][0] : 1.0, d.a[1][1] > 1e-300 ? 1.0 / d.a[1][1] : 1.0,
                d.a[2][2] > 1e-300 ? 1.0 / d.a[2][2] : 1.0};
    st3(a.dinv, r, di);
    const V3 b = ld3(a.rhs, r);
    const V3 rr = b - d_row(a, a.x, r);
    const V3 z = cmul(di, rr);
    st3(a.r, r, rr);
    st3(a.z, r, z);
    st3(a.p, r, z);
    v[0] += dot(rr, z);
    v[1] += dot(rr, rr);
    v[2] += sqnorm(b);
  }
  d_block_partials<3>(a, v);
}

// Ap for the slab's rows (p's halo rows already exchanged); partial p.Ap
__global__ void __launch_bounds__(kDBlock) k_d_spmv(DSlab a) {
  if (a.st[DS_DONE] != 0) return;
  double v[1] = {0};
  for (int r = a.lo + blockIdx.x * kDBlock + threadIdx.x; r < a.hi; r += gridDim.x * kDBlock) {
    const V3 apr = d_row(a, a.p, r);
    st3(a.ap, r, apr);
    v[0] += dot(ld3(a.p, r), apr);
  }
  d_block_partials<1>(a, v);
}

// x += alpha p, r -= alpha Ap, z = D^-1 r; partials {r.z, r.r}
__global__ void __launch_bounds__(kDBlock) k_d_update(DSlab a) {
  if (a.st[DS_DONE] != 0) return;
  const double alpha = a.st[DS_ALPHA];
  double v[2] = {0, 0};
  for (int r = a.lo + blockIdx.x * kDBlock + threadIdx.x; r < a.hi; r += gridDim.x * kDBlock) {
    st3(a.x, r, ld3(a.x, r) + alpha * ld3(a.p, r));
    const V3 rr = ld3(a.r, r) - alpha * ld3(a.ap, r);
    st3(a.r, r, rr);
    const V3 z = cmul(ld3(a.dinv, r), rr);
    st3(a.z, r, z);
    v[0] += dot(rr, z);
    v[1] += dot(rr, rr);
  }
  d_block_partials<2>(a, v);
}

// p = z + beta p
__global__ void __launch_bounds__(kDBlock) k_d_dir(DSlab a) {
  if (a.st[DS_DONE] != 0) return;
  const double beta = a.st[DS_BETA];
  for (int r = a.lo + blockIdx.x * kDBlock + threadIdx.x; r < a.hi; r += gridDim.x * kDBlock)
    st3(a.p, r, ld3(a.z, r) + beta * ld3(a.p, r));
}

// x = 0 on the slab (b == 0, solver.cpp:299-302)
__global__ void k_d_zero(DSlab a) {
  if (a.st[DS_DONE] != 2) return;
  for (int r = a.lo + blockIdx.x * kDBlock + threadIdx.x; r < a.hi; r += gridDim.x * kDBlock) st3(a.x, r, V3{0, 0, 0});
}

// the slab's partials: block partials summed in a fixed order -> gath[rank]
// (one warp per value: every lane loads its strided share, then a fixed tree)
__global__ void k_d_slab_sum(DSlab a, int nv, int nblocks, int rank) {
  const int k = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (k >= nv) return;
  double v[kDMaxBlocks / 32];
#pragma unroll
  for (int j = 0; j < kDMaxBlocks / 32; ++j) {
    const int b = lane + 32 * j;
    v[j] = b < nblocks ? a.part[k * kDMaxBlocks + b] : 0.0;
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < kDMaxBlocks / 32; ++j) s += v[j];
  s = warp_sum(s);
  if (lane == 0) a.gath[rank * kDK + k] = s;
}

// scalars from the gathered partials, summed in rank order (identical on every rank)
// phase 0: init, 1: after spmv, 2: after update
__global__ void k_d_scalars(DSlab a, int world, int phase, double tol) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t[kDK] = {0, 0, 0, 0};
  for (int q = 0; q < world; ++q)
    for (int k = 0; k < kDK; ++k) t[k] += a.gath[q * kDK + k];
  double* st = a.st;
  if (phase == 0) {
    st[DS_RZ] = t[0];
    st[DS_RNORM] = sqrt(t[1]);
    st[DS_BNORM] = sqrt(t[2]);
    st[DS_ITERS] = 0;
    if (st[DS_BNORM] == 0) {
      st[DS_DONE] = 2;
      st[DS_RELRES] = 0;
      return;
    }
    st[DS_RELRES] = st[DS_RNORM] / st[DS_BNORM];
    st[DS_STOP] = fmax(tol * st[DS_RNORM], 1e-13 * st[DS_BNORM]);
    st[DS_DONE] = st[DS_RNORM] > st[DS_STOP] ? 0 : 1;
  } else if (phase == 1) {
    if (st[DS_DONE] != 0) return;
    if (t[0] <= 0) {  // pap <= 0: break (solver.cpp:327)
      st[DS_DONE] = 1;
      return;
    }
    st[DS_ALPHA] = st[DS_RZ] / t[0];
  } else {
    if (st[DS_DONE] != 0) return;
    st[DS_BETA] = t[0] / st[DS_RZ];
    st[DS_RZ] = t[0];
    st[DS_RNORM] = sqrt(t[1]);
    st[DS_RELRES] = st[DS_RNORM] / st[DS_BNORM];
    st[DS_ITERS] += 1;
    // the loop test of the next iteration (r_norm > stop); the direction
    // update that follows is then skipped, as the reference leaves the loop
    if (!(st[DS_RNORM] > st[DS_STOP])) st[DS_DONE] = 1;
  }
}
// per-row min / max referenced column (for the plan)
__global__ void k_d_col_range(int N, const int32_t* cols, int32_t* mn, int32_t* mx) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < N; r += gridDim.x * blockDim.x) {
    int a = -1, b = -1;
    for (int s = 0; s < 27; ++s) {
      const int c = cols[27 * int64_t(r) + s];
      if (c < 0) continue;
      a = a < 0 ? c : min(a, c);
      b = max(b, c);
    }
    mn[r] = a;
    mx[r] = b;
  }
}

// ---------------------------------------------------------------------------
// driver
// ---------------------------------------------------------------------------
namespace {
struct SlabBufs {
  DevBuf<double> x, r, z, p, ap, dinv, part, gath, st;
};

int slab_blocks(const DSlab& a) {
  return std::max(1, std::min(kDMaxBlocks, (a.hi - a.lo + kDBlock - 1) / kDBlock));
}

// Transport: `mine` are the slab indices this process runs (all of them for the
// slabs transport, its rank for NCCL)
struct Transport {
  virtual ~Transport() = default;
  virtual void exchange(std::vector<DSlab>& s, double* DSlab::*vec, const DistPlan& plan) = 0;
  virtual void allgather(std::vector<DSlab>& s) = 0;
  virtual void final_x(std::vector<DSlab>& s, const DistPlan& plan) = 0;
  virtual const void* id() const { return nullptr; }  // communicator a captured graph binds to
};

struct SlabsTransport : Transport {
  cudaStream_t st;
  int world;
  explicit SlabsTransport(cudaStream_t s, int w) : st(s), world(w) {}
  void exchange(std::vector<DSlab>& s, double* DSlab::*vec, const DistPlan& plan) override {
    for (const Xfer& x : plan.xfers)
      WFK_CUDA(cudaMemcpyAsync(s[size_t(x.dst)].*vec + 3 * int64_t(x.lo), s[size_t(x.src)].*vec + 3 * int64_t(x.lo),
                               size_t(x.hi - x.lo) * 24, cudaMemcpyDeviceToDevice, st));
  }
  void allgather(std::vector<DSlab>& s) override {
    for (int q = 0; q < world; ++q)
      for (int k = 0; k < world; ++k)
        if (k != q)
          WFK_CUDA(cudaMemcpyAsync(s[size_t(k)].gath + q * kDK, s[size_t(q)].gath + q * kDK, kDK * 8,
                                   cudaMemcpyDeviceToDevice, st));
  }
  void final_x(std::vector<DSlab>& s, const DistPlan& plan) override {
    for (int q = 0; q < world; ++q)
      for (int k = 0; k < world; ++k)
        if (k != q)
          WFK_CUDA(cudaMemcpyAsync(s[size_t(k)].x + 3 * int64_t(plan.lo[size_t(q)]),
                                   s[size_t(q)].x + 3 * int64_t(plan.lo[size_t(q)]),
                                   size_t(plan.hi[size_t(q)] - plan.lo[size_t(q)]) * 24, cudaMemcpyDeviceToDevice, st));
  }
};

struct NcclTransport : Transport {
  cudaStream_t st;
  DistComm* d;
  NcclTransport(cudaStream_t s, DistComm* dc) : st(s), d(dc) {}
  const void* id() const override { return d->comm; }
  void exchange(std::vector<DSlab>& s, double* DSlab::*vec, const DistPlan& plan) override {
    NcclApi& n = nccl();
    double* v = s[0].*vec;
    WFK_NCCL(n.GroupStart());
    for (const Xfer& x : plan.xfers) {
      if (x.src == d->rank) WFK_NCCL(n.Send(v + 3 * int64_t(x.lo), size_t(x.hi - x.lo) * 3, ncclDouble, x.dst, d->comm, st));
      if (x.dst == d->rank) WFK_NCCL(n.Recv(v + 3 * int64_t(x.lo), size_t(x.hi - x.lo) * 3, ncclDouble, x.src, d->comm, st));
    }
    WFK_NCCL(n.GroupEnd());
  }
  void allgather(std::vector<DSlab>& s) override {
    WFK_NCCL(nccl().AllGather(s[0].gath + d->rank * kDK, s[0].gath, kDK, ncclDouble, d->comm, st));
  }
  void final_x(std::vector<DSlab>& s, const DistPlan& plan) override {
    NcclApi& n = nccl();
    WFK_NCCL(n.GroupStart());
    for (int q = 0; q < d->world; ++q) {
      double* p = s[0].x + 3 * int64_t(plan.lo[size_t(q)]);
      WFK_NCCL(n.Broadcast(p, p, size_t(plan.hi[size_t(q)] - plan.lo[size_t(q)]) * 3, ncclDouble, q, d->comm, st));
    }
    WFK_NCCL(n.GroupEnd());
  }
};

// the partition plan of a device system (D2H of each row's column range)
DistPlan plan_of(wfk_ctx* c, int N, const int32_t* cols_d, int world) {
  cudaStream_t s = c->stream;
  DevBuf<int32_t> MN, MX;
  MN.ensure(size_t(N));
  MX.ensure(size_t(N));
  k_d_col_range<<<grid_for(N), kBlock, 0, s>>>(N, cols_d, MN.p, MX.p);
  count_launch(c);
  std::vector<int32_t> mn(static_cast<size_t>(N)), mx(static_cast<size_t>(N));
  WFK_CUDA(cudaMemcpyAsync(mn.data(), MN.p, size_t(N) * 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaMemcpyAsync(mx.data(), MX.p, size_t(N) * 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  return make_plan(N, mn.data(), mx.data(), world);
}

// per-solve work state: slab buffers and the CUDA graph of one PCG iteration,
// reused while the system (pointers, size, partition) is unchanged
struct DistWork {
  const wfk_ctx* ctx = nullptr;
  int N = -1, world = 0;
  std::vector<int> ranks;
  const double *B = nullptr, *RHS = nullptr;
  const int32_t* CL = nullptr;
  uint64_t plan_ver = 0;
  const void* transport_id = nullptr;  // the communicator (or null for in-process slabs) the graph captured
  std::vector<std::unique_ptr<SlabBufs>> bufs;
  std::vector<DSlab> sl;
  static constexpr int kBatch = 8;
  cudaGraphExec_t exec = nullptr, exec1 = nullptr;  // kBatch iterations / one iteration
  int kernels_per_iter = 0;
  void reset() {  // the slab buffers stay allocated (they only grow)
    if (exec) cudaGraphExecDestroy(exec);
    if (exec1) cudaGraphExecDestroy(exec1);
    exec = exec1 = nullptr;
    sl.clear();
  }
  ~DistWork() { reset(); }
};

// one partitioned pcg_solve of a device-resident system; `ranks` = the slab
// indices run here; x (device, N x 3) is the initial guess on entry and the
// full solution on return.  One iteration (matvec, all-gathered dots, update,
// direction, halo exchange) is captured once as a CUDA graph -- NCCL calls
// included -- and replayed.
void run_dist_pcg_dev(wfk_ctx* c, int N, int world, const std::vector<int>& ranks, const DistPlan& plan,
                      uint64_t plan_ver, const double* B, const int32_t* CL, const double* RHS, double* x, double tol,
                      int max_iters, wfk_pcg_result* res, Transport& tr, DistWork& w) {
  cudaStream_t s = c->stream;
  const bool reuse = w.exec && w.ctx == c && w.N == N && w.world == world && w.ranks == ranks && w.B == B &&
                     w.CL == CL && w.RHS == RHS && w.plan_ver == plan_ver && w.transport_id == tr.id();
  if (!reuse) {
    w.reset();
    w.transport_id = tr.id();
    w.ctx = c;
    w.N = N;
    w.world = world;
    w.ranks = ranks;
    w.B = B;
    w.CL = CL;
    w.RHS = RHS;
    w.plan_ver = plan_ver;
    while (w.bufs.size() < ranks.size()) w.bufs.push_back(std::make_unique<SlabBufs>());
    for (size_t i = 0; i < ranks.size(); ++i) {
      const int q = ranks[i];
      SlabBufs* b = w.bufs[i].get();
      DSlab a;
      a.lo = plan.lo[size_t(q)];
      a.hi = plan.hi[size_t(q)];
      a.blocks = B;
      a.cols = CL;
      a.rhs = RHS;
      a.x = b->x.ensure(3 * size_t(N));
      a.r = b->r.ensure(3 * size_t(N));
      a.z = b->z.ensure(3 * size_t(N));
      a.p = b->p.ensure(3 * size_t(N));
      a.ap = b->ap.ensure(3 * size_t(N));
      a.dinv = b->dinv.ensure(3 * size_t(N));
      a.part = b->part.ensure(size_t(kDK) * kDMaxBlocks);
      a.gath = b->gath.ensure(size_t(kDK) * world);
      a.st = b->st.ensure(DS_N);
      w.sl.push_back(a);
    }
  }
  std::vector<DSlab>& sl = w.sl;
  for (DSlab& a : sl) {
    WFK_CUDA(cudaMemcpyAsync(a.x, x, size_t(N) * 3 * 8, cudaMemcpyDeviceToDevice, s));  // x0, replicated
    WFK_CUDA(cudaMemsetAsync(a.gath, 0, size_t(kDK) * world * 8, s));
    WFK_CUDA(cudaMemsetAsync(a.st, 0, DS_N * 8, s));
    WFK_CUDA(cudaMemsetAsync(a.part, 0, size_t(kDK) * kDMaxBlocks * 8, s));
  }
  auto reduce = [&](int nv, int phase) {
    for (size_t i = 0; i < sl.size(); ++i)
      k_d_slab_sum<<<1, 32 * kDK, 0, s>>>(sl[i], nv, slab_blocks(sl[i]), ranks[i]);
    tr.allgather(sl);
    for (DSlab& a : sl) k_d_scalars<<<1, 32, 0, s>>>(a, world, phase, tol);
  };
  for (DSlab& a : sl) k_d_init<<<slab_blocks(a), kDBlock, 0, s>>>(a);
  reduce(3, 0);
  for (DSlab& a : sl) k_d_zero<<<slab_blocks(a), kDBlock, 0, s>>>(a);
  count_launch(c, int(4 * sl.size()));
  tr.exchange(sl, &DSlab::p, plan);
  static const bool trace = std::getenv("WFK_DIST_TRACE") != nullptr;
  auto now = [&] {
    if (trace) WFK_CUDA(cudaStreamSynchronize(s));
    return std::chrono::steady_clock::now();
  };
  const auto t0 = now();
  const bool captured = !w.exec;
  if (!w.exec) {
    // graphs of kBatch iterations and of one iteration; batches are replayed
    // one at a time with a convergence check in between (queueing many graph
    // launches back to back was measured to stall for up to a second)
    auto capture = [&](int iters, cudaGraphExec_t* out) {
      cudaGraph_t g = nullptr;
      WFK_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < iters; ++k) {
        for (DSlab& a : sl) k_d_spmv<<<slab_blocks(a), kDBlock, 0, s>>>(a);
        reduce(1, 1);
        for (DSlab& a : sl) k_d_update<<<slab_blocks(a), kDBlock, 0, s>>>(a);
        reduce(2, 2);
        for (DSlab& a : sl) k_d_dir<<<slab_blocks(a), kDBlock, 0, s>>>(a);
        tr.exchange(sl, &DSlab::p, plan);
      }
      WFK_CUDA(cudaStreamEndCapture(s, &g));
      const cudaError_t e = cudaGraphInstantiate(out, g, 0);
      cudaGraphDestroy(g);
      WFK_CUDA(e);
    };
    capture(DistWork::kBatch, &w.exec);
    capture(1, &w.exec1);
    w.kernels_per_iter = int(7 * sl.size());
  }
  for (int it = 0; it < max_iters;) {
    const int k = max_iters - it >= DistWork::kBatch ? DistWork::kBatch : 1;
    WFK_CUDA(cudaGraphLaunch(k == 1 ? w.exec1 : w.exec, s));
    count_launch(c, k * w.kernels_per_iter);
    it += k;
    if (it < max_iters) {  // leave early once converged (identical state on every rank)
      WFK_CUDA(cudaMemcpyAsync(c->h_pinned + 64, sl[0].st + DS_DONE, 8, cudaMemcpyDeviceToHost, s));
      WFK_CUDA(cudaStreamSynchronize(s));
      double done;
      std::memcpy(&done, c->h_pinned + 64, 8);
      if (done != 0) break;
    }
  }
  const auto t2 = now();
  if (trace)
    fprintf(stderr, "[wfk dist] N %d world %d %s loop %.3f ms\n", N, world, captured ? "captured" : "reused",
            std::chrono::duration<double, std::milli>(t2 - t0).count());
  tr.final_x(sl, plan);
  double st_h[DS_N];
  WFK_CUDA(cudaMemcpyAsync(x, sl[0].x, size_t(N) * 3 * 8, cudaMemcpyDeviceToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(st_h, sl[0].st, DS_N * 8, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  WFK_CUDA(cudaGetLastError());
  if (res) {
    res->iterations = int32_t(st_h[DS_ITERS]);
    res->relative_residual = st_h[DS_RELRES];
  }
}

// host-array system: uploaded (every rank holds the caller's full system), solved, x returned
void run_dist_pcg(wfk_ctx* c, int N, int world, const std::vector<int>& ranks, const double* blocks_h,
                  const int32_t* cols_h, const double* rhs_h, double* x_h, double tol, int max_iters,
                  wfk_pcg_result* res, Transport& tr) {
  cudaStream_t s = c->stream;
  DevBuf<double> B, RHS, X;
  DevBuf<int32_t> CL;
  B.ensure(size_t(N) * 27 * 9);
  CL.ensure(size_t(N) * 27);
  RHS.ensure(size_t(N) * 3);
  X.ensure(size_t(N) * 3);
  WFK_CUDA(cudaMemcpyAsync(B.p, blocks_h, size_t(N) * 27 * 9 * 8, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(CL.p, cols_h, size_t(N) * 27 * 4, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(RHS.p, rhs_h, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(X.p, x_h, size_t(N) * 3 * 8, cudaMemcpyHostToDevice, s));
  const DistPlan plan = plan_of(c, N, CL.p, world);
  DistWork w;
  run_dist_pcg_dev(c, N, world, ranks, plan, 0, B.p, CL.p, RHS.p, X.p, tol, max_iters, res, tr, w);
  WFK_CUDA(cudaMemcpyAsync(x_h, X.p, size_t(N) * 3 * 8, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

// partitioned PCG of a device-resident system (the solver's normal equations).
// slabs > 0: that many slab states on this GPU; slabs == 0: this rank of the
// context's communicator.  plan_key identifies the system's row structure: the
// plan (and the captured iteration) is rebuilt when it changes or when `fresh`.
struct PlanCache {
  const wfk_ctx* ctx = nullptr;
  int N = -1, world = 0;
  uint64_t version = 0;
  DistPlan plan;
  DistWork work;
};
static bool same_plan(const DistPlan& a, const DistPlan& b) {
  if (a.world != b.world || a.lo != b.lo || a.hi != b.hi || a.xfers.size() != b.xfers.size()) return false;
  for (size_t i = 0; i < a.xfers.size(); ++i)
    if (a.xfers[i].src != b.xfers[i].src || a.xfers[i].dst != b.xfers[i].dst || a.xfers[i].lo != b.xfers[i].lo ||
        a.xfers[i].hi != b.xfers[i].hi)
      return false;
  return true;
}
// one cache entry per system key (the solver passes its Level), so each level
// keeps its plan, slab buffers and captured iteration from solve to solve
static std::map<const void*, PlanCache>& plan_caches() {
  static std::map<const void*, PlanCache> m;
  return m;
}
static std::mutex& plan_mutex() {  // the map is shared by every context of the process
  static std::mutex m;
  return m;
}

void dist_pcg_device(wfk_ctx* c, int slabs, int N, const double* blocks, const int32_t* cols, const double* rhs,
                     double* x, double tol, int max_iters, const void* plan_key, bool fresh, wfk_pcg_result* res) {
  if (N <= 0) {
    if (res) *res = wfk_pcg_result{0, 0, 0.0};
    return;
  }
  DistComm* d = c->dist;
  if (slabs <= 0 && !d) throw Error(WFK_E_INVALID_ARG, "wfk_dist_init first");
  const int world = slabs > 0 ? slabs : d->world;
  PlanCache* pcp;
  {
    std::lock_guard<std::mutex> lock(plan_mutex());
    pcp = &plan_caches()[plan_key];  // std::map references stay valid across inserts
  }
  PlanCache& pc = *pcp;
  if (fresh || !plan_key || pc.ctx != c || pc.N != N || pc.world != world) {
    DistPlan p = plan_of(c, N, cols, world);
    // an unchanged partition keeps the captured iteration
    if (pc.ctx != c || pc.N != N || pc.world != world || !same_plan(p, pc.plan)) {
      pc.plan = std::move(p);
      ++pc.version;
    }
    pc.ctx = c;
    pc.N = N;
    pc.world = world;
  }
  std::vector<int> ranks;
  if (slabs > 0) {
    for (int q = 0; q < slabs; ++q) ranks.push_back(q);
    SlabsTransport t(c->stream, slabs);
    run_dist_pcg_dev(c, N, world, ranks, pc.plan, pc.version, blocks, cols, rhs, x, tol, max_iters, res, t, pc.work);
  } else {
    ranks.push_back(d->rank);
    NcclTransport tr(c->stream, d);
    SlabsTransport single(c->stream, 1);
    Transport& t = d->comm ? static_cast<Transport&>(tr) : static_cast<Transport&>(single);
    run_dist_pcg_dev(c, N, world, ranks, pc.plan, pc.version, blocks, cols, rhs, x, tol, max_iters, res, t, pc.work);
  }
}

// the context goes away: drop cached work that points into it
void dist_forget(wfk_ctx* c) {
  std::lock_guard<std::mutex> lock(plan_mutex());
  auto& m = plan_caches();
  for (auto it = m.begin(); it != m.end();) {
    if (it->second.ctx == c || it->second.work.ctx == c)
      it = m.erase(it);
    else
      ++it;
  }
}

void dist_plan(int N, const int32_t* cols, int world, int32_t* ranges, int32_t* xfers, int32_t cap,
               int32_t* n_xfers) {
  if (N < 0 || world < 1 || (N > 0 && !cols)) throw Error(WFK_E_INVALID_ARG, "bad plan arguments");
  std::vector<int32_t> mn(static_cast<size_t>(N)), mx(static_cast<size_t>(N));
  for (int r = 0; r < N; ++r) {
    int a = -1, b = -1;
    for (int s = 0; s < 27; ++s) {
      const int c = cols[27 * int64_t(r) + s];
      if (c < 0) continue;
      a = a < 0 ? c : std::min(a, c);
      b = std::max(b, c);
    }
    mn[size_t(r)] = a;
    mx[size_t(r)] = b;
  }
  const DistPlan p = make_plan(N, mn.data(), mx.data(), world);
  if (ranges)
    for (int k = 0; k < world; ++k) {
      ranges[2 * k] = p.lo[size_t(k)];
      ranges[2 * k + 1] = p.hi[size_t(k)];
    }
  *n_xfers = int32_t(p.xfers.size());
  if (!xfers) return;
  if (int32_t(p.xfers.size()) > cap) throw Error(WFK_E_CAPACITY, "transfer buffer too small");
  for (size_t i = 0; i < p.xfers.size(); ++i) {
    xfers[4 * i] = p.xfers[i].src;
    xfers[4 * i + 1] = p.xfers[i].dst;
    xfers[4 * i + 2] = p.xfers[i].lo;
    xfers[4 * i + 3] = p.xfers[i].hi;
  }
}

void dist_unique_id(uint8_t* out) {
  ncclUniqueId id;
  WFK_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out, id.internal, sizeof(id.internal));
}

void dist_init(wfk_ctx* c, int rank, int world, const uint8_t* id_bytes) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(WFK_E_INVALID_ARG, "bad rank / world");
  dist_destroy(c);
  auto* d = new DistComm;
  d->rank = rank;
  d->world = world;
  if (id_bytes) {  // NCCL communicator (also at world 1, which exercises the same transport)
    ncclUniqueId id;
    std::memcpy(id.internal, id_bytes, sizeof(id.internal));
    WFK_CUDA(cudaSetDevice(c->device));
    const ncclResult_t r = nccl().CommInitRank(&d->comm, world, id, rank);
    if (r != ncclSuccess) {
      delete d;
      throw Error(WFK_E_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
  }
  c->dist = d;
}

void dist_pcg(wfk_ctx* c, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x, double tol,
              int max_iters, wfk_pcg_result* res) {
  if (!c->dist) throw Error(WFK_E_INVALID_ARG, "wfk_dist_init first");
  DistComm* d = c->dist;
  if (N <= 0) {
    if (res) *res = wfk_pcg_result{0, 0, 0.0};
    return;
  }
  NcclTransport tr(c->stream, d);
  SlabsTransport single(c->stream, 1);
  Transport& t = d->comm ? static_cast<Transport&>(tr) : static_cast<Transport&>(single);
  run_dist_pcg(c, N, d->world, {d->rank}, blocks, cols, rhs, x, tol, max_iters, res, t);
}

void slabs_pcg(wfk_ctx* c, int slabs, int N, const double* blocks, const int32_t* cols, const double* rhs, double* x,
               double tol, int max_iters, wfk_pcg_result* res) {
  if (slabs < 1) throw Error(WFK_E_INVALID_ARG, "slabs must be >= 1");
  if (N <= 0) {
    if (res) *res = wfk_pcg_result{0, 0, 0.0};
    return;
  }
  std::vector<int> ranks(static_cast<size_t>(slabs));
  for (int q = 0; q < slabs; ++q) ranks[size_t(q)] = q;
  SlabsTransport t(c->stream, slabs);
  run_dist_pcg(c, N, slabs, ranks, blocks, cols, rhs, x, tol, max_iters, res, t);
}

}  // namespace wfk
