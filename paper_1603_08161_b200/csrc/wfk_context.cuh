// Device context of libwfk: one per (process, GPU).  Owns the device-resident
// deformation lattice, the per-level solver workspaces, the frame / map /
// mesh / geometry-buffer buffers and the CUDA stream every call runs on.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/wfk.h"
#include "wfk_common.cuh"

namespace wfk {

struct DistComm;  // dist.cu: rank, world, NCCL communicator

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define WFK_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::wfk::Error(e_ == cudaErrorMemoryAllocation ? WFK_E_OOM : WFK_E_CUDA,       \
                         std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

// WFK_ALLOC_TRACE=1: log every device (re)allocation of a DevBuf to stderr
inline bool alloc_trace() {
  static const bool on = std::getenv("WFK_ALLOC_TRACE") != nullptr;
  return on;
}

// ---- checked mode (WFK_CHECK=1) ---------------------------------------------
// compute-sanitizer is not available on the GPU pool, so the library carries
// its own memcheck / initcheck stand-ins, switched on by the environment when
// the process starts:
//  * every DevBuf allocation is filled with 0xff bytes before use (NaN doubles
//    and floats, -1 integers), so a kernel that reads memory nothing wrote
//    feeds NaNs / -1 indices into results the parity tests compare with the
//    reference -- instead of the zeros a fresh cudaMalloc usually returns;
//  * every DevBuf carries a kGuardBytes canary tail (0xa5) past its capacity,
//    verified after every C-ABI call (guard_verify in api.cu's guard()): a kernel
//    writing past the end of any buffer fails the call with WFK_E_CUDA naming
//    the buffer's size.
// Off (the default), allocations are exactly as before: no fill, no tail.
inline bool check_mode() {
  static const bool on = [] {
    const char* v = std::getenv("WFK_CHECK");
    return v && *v && *v != '0';
  }();
  return on;
}
constexpr size_t kGuardBytes = 256;
constexpr unsigned char kGuardByte = 0xa5;
constexpr unsigned char kPoisonByte = 0xff;
struct GuardEntry {
  size_t bytes;  // usable bytes; the canary starts here
  int device;
};
std::mutex& guard_mutex();
std::map<const void*, GuardEntry>& guard_table();
inline void guard_add(const void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(guard_mutex());
  guard_table()[p] = GuardEntry{bytes, dev};
}
inline void guard_drop(const void* p) {
  std::lock_guard<std::mutex> lock(guard_mutex());
  guard_table().erase(p);
}
// allocation of `bytes` usable bytes (+ the canary in checked mode); poisoned
// and synchronised in checked mode so the fill is ordered before any stream
inline void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  if (!check_mode()) {
    WFK_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  WFK_CUDA(cudaMalloc(&p, bytes + kGuardBytes));
  WFK_CUDA(cudaMemset(p, kPoisonByte, bytes));
  WFK_CUDA(cudaMemset(static_cast<char*>(p) + bytes, kGuardByte, kGuardBytes));
  WFK_CUDA(cudaDeviceSynchronize());
  guard_add(p, bytes);
  return p;
}
inline void dev_free(void* p) {
  if (!p) return;
  if (check_mode()) guard_drop(p);
  cudaFree(p);
}
// verifies every live canary (checked mode); returns the number broken and
// describes the first in *what
int guard_verify(std::string* what);

// Growable device buffer (capacity only grows; contents not preserved).
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { dev_free(p); }
  T* ensure(size_t n) {
    if (n == 0) n = 1;
    if (n > cap) {
      dev_free(p);
      p = nullptr;
      size_t want = n + n / 4;
      p = static_cast<T*>(dev_alloc(want * sizeof(T)));
      if (alloc_trace()) fprintf(stderr, "[wfk alloc] ensure %zu x %zu B\n", want, sizeof(T));
      cap = want;
    }
    return p;
  }
  // exact-size ensure keeping the old contents
  T* grow_keep(size_t n, cudaStream_t s) {
    if (n <= cap) return p;
    size_t want = n + n / 4;
    T* q = static_cast<T*>(dev_alloc(want * sizeof(T)));
    if (alloc_trace()) fprintf(stderr, "[wfk alloc] grow_keep %zu x %zu B\n", want, sizeof(T));
    if (p) {
      WFK_CUDA(cudaMemcpyAsync(q, p, cap * sizeof(T), cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaStreamSynchronize(s));
      dev_free(p);
    }
    p = q;
    cap = want;
    return p;
  }
  operator T*() const { return p; }
};

// Device copy of one wf::Correspondence (input constraints of a solve).
struct ConIn {
  DevBuf<int32_t> kind;     // C
  DevBuf<double> canonical; // 3C
  DevBuf<int32_t> anchor;   // 8C   (node indices, level-0 grid)
  DevBuf<double> weight;    // 8C
  DevBuf<double> target;    // 3C
  DevBuf<double> normal;    // 3C
  DevBuf<double> conf;      // C
  int64_t count = 0;
  int64_t n_sparse = 0;     // SparsePoint records among them (byte model)
};

// Per-level solver workspace (one lattice of the coarse-to-fine hierarchy).
struct Level {
  Grid g{};
  bool owns_field = false;
  // node-indexed deformation field (level 0: aliases the volume)
  DevBuf<double> own_deformed, own_euler;
  DevBuf<uint8_t> own_active;
  double* deformed = nullptr;
  double* euler = nullptr;
  uint8_t* active = nullptr;
  // rows
  int N = 0;
  uint64_t rows_gen = 0;  // level 0: volume active_gen the row structures were built for
  bool rows_valid = false;   // row structures built (coarse levels: for prev_active)
  bool mask_same = false;    // coarse levels: build_hierarchy found the activity mask unchanged
  DevBuf<uint8_t> prev_active;  // coarse levels: mask the rows were last built from
  size_t prev_n = 0;
  int prev_dims[3] = {0, 0, 0};
  DevBuf<int32_t> rows, node_row, nbr, uf;  // nbr: 6 x Ncap SoA
  DevBuf<uint8_t> frozen, comp_flag;
  // per-row state (AoS double3 / row-major 3x3)
  DevBuf<double4> t, x, rhs, r, p, ap, dinv, u, w, crhs, cdiag, z;  // 32 B padded 3-vectors
  DevBuf<double4> mbuf;  // 2 x N: pipelined PCG m = D w, double-buffered
  DevBuf<double4> nbuf;  // N: pipelined PCG n = A m
  DevBuf<double> state_spill;  // pipelined PCG row state when it does not fit shared memory
  DevBuf<int32_t> perm, perm_key, perm_val;  // matrix-free levels: row order by decreasing incidences
  DevBuf<double> rot;
  // assembled B^T B for rows with many incidences (see kAssembleRatio)
  bool assembled = false;
  DevBuf<double> blk;      // N x 27 x 6
  DevBuf<int32_t> cols;    // N x 27
  DevBuf<uint8_t> ent_k;   // corner of the row inside each incident constraint
  DevBuf<int32_t> c_pos;   // 8C: incidence slot of (constraint, corner), -1 if none
  DevBuf<double4> contrib; // E: per-incidence matvec contributions
  DevBuf<int4> xitems;     // extra work items of the balanced matrix-free row pass
  DevBuf<int32_t> xptr;
  DevBuf<int2> xrange;
  DevBuf<double4> wpart;
  int n_xitems = 0;
  bool items_built = false;
  // level constraints
  int64_t C = 0;
  DevBuf<int32_t> c_node;   // 8C anchors at this level
  DevBuf<double> c_w;       // 8C
  DevBuf<int32_t> c_row;    // 8C (row or -1)
  DevBuf<double> c_g;       // 4C: g = R^T n (dense) and coef
  DevBuf<double> c_b;       // 3C: constraint rhs vector before alpha
  DevBuf<double> c_u;       // 3C: matvec scratch
  DevBuf<int32_t> c_kind;   // C
  // concurrent setup (solver_c2f): the level's own stream, completion event,
  // cub scratch and count words while its setup runs beside the other levels'
  cudaStream_t setup_stream = nullptr;
  cudaEvent_t setup_done = nullptr;
  DevBuf<uint8_t> setup_temp;
  DevBuf<int32_t> setup_ivec;
  // CSR transpose: row -> (constraint, alpha)
  int64_t E = 0;
  DevBuf<int32_t> row_ptr, ent_con, key_in, key_out, val_in, val_out;
  DevBuf<double> ent_w;
  DevBuf<int32_t> cnt;
  // WFK_PRECISION_FAST Chronopoulos-Gear PCG: fp32 Krylov vectors (packed xyz)
  DevBuf<float> f_r, f_p, f_s, f_u, f_d, f_dinv, f_contrib, f_wpart;
  // the same packed in fp64 (the default for large CG levels)
  DevBuf<double> d_r, d_p, d_s, d_u, d_d, d_dinv, d_contrib, d_wpart;
  // slab-partitioned CG inside the persistent kernel (WFK_SLABS): rank row
  // ranges, u windows, constraint lists, counters, partials, pointer tables
  DevBuf<int32_t> sl_idx, sl_blk;
  DevBuf<double4> sl_win;
  DevBuf<unsigned> sl_ctr;
  DevBuf<unsigned long long> sl_red, sl_ptr;
  // explicit normal equations of the slab-partitioned solve (solver_c2f_dist)
  DevBuf<double> ne_blocks, ne_rhs, ne_x;
  DevBuf<int32_t> ne_cols;
};

struct VolumeDev {
  Grid g{};
  double mu = 0;
  int64_t n = 0;
  DevBuf<float> tsdf, weight, color;
  DevBuf<double> deformed, euler;
  DevBuf<int32_t> age;
  DevBuf<uint8_t> active;
  uint64_t active_gen = 1;  // bumped whenever the active mask may change
  bool valid = false;
  // device-side checkpoint of the fields a solve / expansion mutates (wfk_volume_checkpoint)
  DevBuf<double> bk_deformed, bk_euler;
  DevBuf<int32_t> bk_age;
  DevBuf<uint8_t> bk_active;
  bool bk_valid = false;
};

struct FrameDev {
  wfk_intrinsics K{};
  bool has_color = false;
  DevBuf<float> depth_buf, color_buf;
  // the frame the kernels read: the upload buffers or a staged slot
  const float* depth = nullptr;
  const float* color = nullptr;
  // PointNormalMap (correspond.hpp:34-42)
  DevBuf<double> point, normal;
  DevBuf<uint8_t> pvalid, nvalid;
  bool maps_valid = false;
};

struct MeshDev {
  int64_t V = 0, T = 0;
  DevBuf<double> can, def, nrm;
  DevBuf<float> col;
  DevBuf<int32_t> tri;
  // marching-cubes scratch
  DevBuf<int32_t> cell_case, cell_tri_off, cell_vert_off, edge_vertex;
  DevBuf<uint8_t> tri_keep;
  DevBuf<int32_t> tri_pos;
  // vertex -> incident triangles (ascending), for compute_normals
  DevBuf<int32_t> adj_ptr, adj_tri, adj_key, adj_val, adj_key2, adj_cnt;
  bool adj_valid = false;
  bool normals_valid = false;
};

struct GBufDev {
  int w = 0, h = 0;
  DevBuf<float> depth;
  DevBuf<double> point, normal, canonical;
  DevBuf<unsigned long long> zkey;
  // triangle setup scratch
  DevBuf<double> setup;
  DevBuf<int32_t> setup_tri;
  DevBuf<int32_t> assoc_pos;
  bool valid = false;
};

constexpr int kMaxLevels = 8;

// feature front-end scratch (features.cu)
constexpr int kFeatOctaves = 8, kFeatLevels = 16;
struct FeatDev {
  DevBuf<float> levels[kFeatOctaves][kFeatLevels];  // per octave: L + 1 gaussian, then L DoG levels
  int L = 0;
  std::vector<int> ws, hs;
  DevBuf<float> gray, base;
  DevBuf<uint8_t> flag, ok, kp, cur_raw;
  DevBuf<int32_t> pos, idx, nori, cnt;
  DevBuf<int4> ext;
  DevBuf<uint32_t> key;
  DevBuf<double> ori;
  int32_t n_cur = 0;
  DevBuf<wfk_feature> cur;            // the last detection's features, compacted
  // FeatureStore (features.hpp:79-95): append-only history, frame ids ascending
  DevBuf<wfk_feature> store;
  int64_t n_store = 0;
  int64_t max_group = 0;  // largest frame group (sizes the matcher's fallback distance area)
  // matching scratch (match_features, features.cpp:354-433)
  DevBuf<double> pred, dist, row_d;
  DevBuf<wfk_feature> xstore;  // wfk_match_features' store upload
  DevBuf<uint32_t> skey;
  DevBuf<int32_t> sidx, mcnt, mpos;
  DevBuf<wfk_feature_match> mslot, matches;
  int32_t n_matches = 0;
  // sparse feature constraints of the frame (sparse_to_constraints, correspond.cpp:152-169)
  DevBuf<wfk_correspondence> sparse;
  DevBuf<uint8_t> sparse_ok;
  int32_t n_sparse = 0;
  // add_features scratch (pipeline.cpp:95-141)
  DevBuf<wfk_feature> lift;
  DevBuf<uint8_t> lift_ok;
};

struct Stats {
  int64_t pcg_iterations = 0;
  int64_t kernel_launches = 0;
};

// Optional device-event profiling (wfk_profile_enable): per-launch duration of
// the flip-flop kernel with its algorithmic bytes, and per-stage durations of
// wfk_process_frame.
constexpr int kStages = 6;  // 0 maps+mesh+raster, 1 associate, 2 solve, 3 redeform, 4 fuse, 5 total
struct Prof {
  bool on = false;
  int64_t ff_launches = 0;
  int64_t pcg_iterations = 0;
  double ff_ms = 0;
  double ff_bytes = 0;       // SURVEY.md 8(d) model (fp32 state, 3-phase PCG)
  double ff_bytes_impl = 0;  // this implementation's fp64 layout
  double stage_ms[kStages] = {0, 0, 0, 0, 0, 0};
  cudaEvent_t ev[2 + 2 * kStages] = {};
  cudaEvent_t timer[16] = {};
};

}  // namespace wfk

struct wfk_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int precision = 0;  // WFK_PRECISION_FP64 | WFK_PRECISION_FAST
  wfk::VolumeDev vol;
  wfk::ConIn cons;
  wfk::Level lv[wfk::kMaxLevels];
  wfk::FrameDev frame;
  wfk::MeshDev mesh;
  wfk::GBufDev gbuf;
  wfk::FeatDev feat;
  wfk::Stats stats;
  wfk::Prof prof;
  // frames staged in device memory (wfk_frame_stage)
  std::vector<wfk_intrinsics> staged_K;
  std::vector<float*> staged_depth, staged_color;
  wfk::DevBuf<uint8_t> l2_flush;
  // scratch
  wfk::DevBuf<double> partials;
  wfk::DevBuf<uint32_t> sync_words;  // grid barrier state of the persistent kernel
  wfk::DevBuf<int32_t> flags;   // device status words
  wfk::DevBuf<uint8_t> temp;    // cub temp storage
  wfk::DevBuf<wfk_trace_entry> trace;
  wfk::DevBuf<int32_t> ivec;    // misc int scratch
  wfk::DevBuf<int64_t> lvec;    // misc int64 scratch
  wfk::DevBuf<double> dvec;     // misc double scratch
  wfk::DevBuf<double> eout;     // energy readback
  wfk::DevBuf<uint8_t> mask;    // misc byte scratch
  int32_t* h_pinned = nullptr;  // small pinned readback area (8 KB)
  // global-pose ICP (assoc.cu)
  wfk::DevBuf<int32_t> icp_pos;
  wfk::DevBuf<double> icp_src, icp_part;
  wfk::DevBuf<uint8_t> icp_state;
  int coop_blocks = 0;          // resident blocks for cooperative kernels
  wfk::DistComm* dist = nullptr;  // slab-partitioned PCG (wfk_dist_init)
  wfk::DevBuf<uint8_t> debug_buf;  // wfk_debug_overrun (checked-mode self-test)
  cudaEvent_t setup_ready = nullptr;  // solver_c2f: hierarchy built, level setups may start
  // wfk_process_frame: feature detection on a side stream beside mesh / raster / ICP
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_ready = nullptr, side_done = nullptr;
  wfk::DevBuf<uint8_t> side_temp;
};

namespace wfk {
// launch-count bookkeeping (bench.py reports gpu_launches from this)
inline void count_launch(wfk_ctx* c, int n = 1) { c->stats.kernel_launches += n; }
inline int grid_for(int64_t n, int block = kBlock) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (1 << 30)) g = 1 << 30;
  return int(g);
}
}  // namespace wfk
