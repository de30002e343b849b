// extern "C" boundary of libwfk (include/wfk.h).  Every entry point validates
// its arguments, runs on the context's stream and returns a status; C++
// exceptions never cross the ABI.
#include <chrono>
#include <cstring>
#include <vector>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"

using namespace wfk;

// checked mode (WFK_CHECK=1, wfk_context.cuh): the canary registry of every
// live DevBuf allocation
namespace wfk {
// never destroyed: a DevBuf freed during static destruction still finds them
std::mutex& guard_mutex() {
  static std::mutex* m = new std::mutex;
  return *m;
}
std::map<const void*, GuardEntry>& guard_table() {
  static auto* t = new std::map<const void*, GuardEntry>;
  return *t;
}
int guard_verify(std::string* what) {
  std::lock_guard<std::mutex> lock(guard_mutex());
  int broken = 0;
  unsigned char tail[kGuardBytes];
  for (const auto& kv : guard_table()) {
    WFK_CUDA(cudaMemcpy(tail, static_cast<const char*>(kv.first) + kv.second.bytes, kGuardBytes,
                        cudaMemcpyDeviceToHost));
    size_t first = kGuardBytes;
    for (size_t i = 0; i < kGuardBytes; ++i)
      if (tail[i] != kGuardByte) {
        first = i;
        break;
      }
    if (first == kGuardBytes) continue;
    if (broken++ == 0 && what)
      *what = "WFK_CHECK: write past the end of a " + std::to_string(kv.second.bytes) +
              "-byte device buffer (canary byte " + std::to_string(first) + " overwritten, device " +
              std::to_string(kv.second.device) + ")";
  }
  return broken;
}
}  // namespace wfk

namespace {

template <class F>
int guard(wfk_ctx* c, F&& f) {
  if (!c) return WFK_E_INVALID_ARG;
  try {
    WFK_CUDA(cudaSetDevice(c->device));
    f();
    if (check_mode()) {
      // every kernel of the call has finished before the canaries are read
      WFK_CUDA(cudaDeviceSynchronize());
      std::string what;
      if (guard_verify(&what) > 0) throw Error(WFK_E_CUDA, what);
    }
    return WFK_OK;
  } catch (const Error& e) {
    c->err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    c->err = e.what();
    return WFK_E_CUDA;
  }
}

void check_params(const wfk_solver_params* p) {
  if (!p) throw Error(WFK_E_INVALID_ARG, "null solver params");
}

int export_trace(wfk_ctx* c, const std::vector<wfk_trace_entry>& t, wfk_trace_entry* out, int32_t cap, int32_t* n_out) {
  if (n_out) *n_out = int32_t(t.size());
  if (int64_t(t.size()) > cap || (!out && !t.empty())) {
    c->err = "trace buffer too small";
    return WFK_E_CAPACITY;
  }
  if (!t.empty()) std::memcpy(out, t.data(), t.size() * sizeof(wfk_trace_entry));
  return WFK_OK;
}

// constraints -> device (SoA), validating the trilinear anchor layout
void upload_constraints(wfk_ctx* c, const wfk_correspondence* h, int64_t n, bool append, bool drop_inactive,
                        int64_t* kept) {
  if (n < 0 || (n > 0 && !h)) throw Error(WFK_E_INVALID_ARG, "bad constraint array");
  const Grid& g = c->vol.g;
  const int64_t npts = c->vol.n;
  std::vector<uint8_t> act;
  if (drop_inactive) {
    act.resize(size_t(npts));
    WFK_CUDA(cudaMemcpyAsync(act.data(), c->vol.active, size_t(npts), cudaMemcpyDeviceToHost, c->stream));
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  }
  std::vector<int32_t> kind, anchor;
  std::vector<double> can, w, tgt, nrm, conf;
  kind.reserve(size_t(n));
  for (int64_t i = 0; i < n; ++i) {
    const wfk_correspondence& r = h[i];
    const int a0 = r.anchor_index[0];
    for (int k = 0; k < 8; ++k)
      if (r.anchor_index[k] < 0 || r.anchor_index[k] >= npts)
        throw Error(WFK_E_OUT_OF_RANGE, "constraint anchor outside the lattice");
    int x, y, z;
    g.idx3(a0, x, y, z);
    if (x > g.nx - 2 || y > g.ny - 2 || z > g.nz - 2)
      throw Error(WFK_E_INVALID_ARG, "anchor 0 is not the min corner of a lattice cell");
    for (int k = 0; k < 8; ++k)
      if (r.anchor_index[k] != g.lin(x + (k & 1), y + ((k >> 1) & 1), z + (k >> 2)))
        throw Error(WFK_E_INVALID_ARG, "anchors are not trilinear cell anchors");
    if (r.kind != WFK_DENSE_PLANE && r.kind != WFK_SPARSE_POINT)
      throw Error(WFK_E_INVALID_ARG, "unknown correspondence kind");
    if (drop_inactive) {
      bool all = true;
      for (int k = 0; k < 8; ++k) all = all && act[size_t(r.anchor_index[k])];
      if (!all) continue;
    }
    kind.push_back(r.kind);
    for (int k = 0; k < 3; ++k) {
      can.push_back(r.canonical[k]);
      tgt.push_back(r.target[k]);
      nrm.push_back(r.target_normal[k]);
    }
    for (int k = 0; k < 8; ++k) {
      anchor.push_back(r.anchor_index[k]);
      w.push_back(r.anchor_weight[k]);
    }
    conf.push_back(r.confidence);
  }
  const int64_t m = int64_t(kind.size());
  if (kept) *kept = m;
  ConIn& ci = c->cons;
  const int64_t base = append ? ci.count : 0;
  const int64_t total = base + m;
  const size_t cap = size_t(total) + 1;
  cudaStream_t s = c->stream;
  ci.kind.grow_keep(cap, s);
  ci.canonical.grow_keep(3 * cap, s);
  ci.anchor.grow_keep(8 * cap, s);
  ci.weight.grow_keep(8 * cap, s);
  ci.target.grow_keep(3 * cap, s);
  ci.normal.grow_keep(3 * cap, s);
  ci.conf.grow_keep(cap, s);
  if (m > 0) {
    WFK_CUDA(cudaMemcpyAsync(ci.kind.p + base, kind.data(), size_t(m) * 4, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.canonical.p + 3 * base, can.data(), size_t(m) * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.anchor.p + 8 * base, anchor.data(), size_t(m) * 32, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.weight.p + 8 * base, w.data(), size_t(m) * 64, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.target.p + 3 * base, tgt.data(), size_t(m) * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.normal.p + 3 * base, nrm.data(), size_t(m) * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(ci.conf.p + base, conf.data(), size_t(m) * 8, cudaMemcpyHostToDevice, s));
  }
  WFK_CUDA(cudaStreamSynchronize(s));  // host staging vectors die on return
  int64_t ns = 0;
  for (int32_t k : kind) ns += k == WFK_SPARSE_POINT ? 1 : 0;
  ci.n_sparse = (append ? ci.n_sparse : 0) + ns;
  ci.count = total;
}

void run_frame(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose* pose, const wfk_pipeline_config* cfg,
               const wfk_correspondence* sparse, int64_t nsparse, int32_t frame_index, wfk_frame_record* rec);

// the context's stream and cub scratch swapped for the side stream's while
// the feature detection is queued there (run_frame)
struct SideScope {
  wfk_ctx* c;
  cudaStream_t saved;
  explicit SideScope(wfk_ctx* c_) : c(c_), saved(c_->stream) {
    c->stream = c->side_stream;
    std::swap(c->temp.p, c->side_temp.p);
    std::swap(c->temp.cap, c->side_temp.cap);
  }
  ~SideScope() {
    std::swap(c->temp.p, c->side_temp.p);
    std::swap(c->temp.cap, c->side_temp.cap);
    c->stream = saved;
  }
};

void stage_mark(wfk_ctx* c, int k) {
  if (c->prof.on) WFK_CUDA(cudaEventRecord(c->prof.ev[2 + k], c->stream));
}

}  // namespace

extern "C" {

int wfk_version(void) { return 1; }

int wfk_create(const wfk_config* cfg, wfk_ctx** out) {
  if (!out) return WFK_E_INVALID_ARG;
  *out = nullptr;
  auto* c = new wfk_ctx;
  c->device = cfg ? cfg->device : 0;
  c->precision = cfg ? cfg->precision : 0;
  try {
    int n = 0;
    WFK_CUDA(cudaGetDeviceCount(&n));
    if (c->device < 0 || c->device >= n) throw Error(WFK_E_INVALID_ARG, "no such CUDA device");
    WFK_CUDA(cudaSetDevice(c->device));
    cudaDeviceProp prop;
    WFK_CUDA(cudaGetDeviceProperties(&prop, c->device));
    if (prop.major < 10) throw Error(WFK_E_CUDA, "libwfk is built for sm_100a (B200)");
    c->num_sms = prop.multiProcessorCount;
    WFK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    WFK_CUDA(cudaMallocHost(&c->h_pinned, 8192));  // 4 KB readback area + 4 KB ICP state staging
    for (cudaEvent_t& e : c->prof.ev) WFK_CUDA(cudaEventCreate(&e));
    for (cudaEvent_t& e : c->prof.timer) WFK_CUDA(cudaEventCreate(&e));
  } catch (const Error& e) {
    delete c;
    return e.code;
  }
  *out = c;
  return WFK_OK;
}

int wfk_set_precision(wfk_ctx* c, int32_t precision) {
  return guard(c, [&] {
    if (precision != WFK_PRECISION_FP64 && precision != WFK_PRECISION_FAST)
      throw Error(WFK_E_INVALID_ARG, "unknown precision");
    c->precision = precision;
  });
}

void wfk_destroy(wfk_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  wfk::dist_forget(c);
  wfk::dist_destroy(c);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  for (cudaEvent_t e : c->prof.ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof.timer)
    if (e) cudaEventDestroy(e);
  for (float* p : c->staged_depth)
    if (p) cudaFree(p);
  for (float* p : c->staged_color)
    if (p) cudaFree(p);
  for (wfk::Level& L : c->lv) {
    if (L.setup_stream) cudaStreamSynchronize(L.setup_stream);
    if (L.setup_done) cudaEventDestroy(L.setup_done);
    if (L.setup_stream) cudaStreamDestroy(L.setup_stream);
  }
  if (c->setup_ready) cudaEventDestroy(c->setup_ready);
  if (c->side_stream) cudaStreamSynchronize(c->side_stream);
  if (c->side_ready) cudaEventDestroy(c->side_ready);
  if (c->side_done) cudaEventDestroy(c->side_done);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* wfk_last_error(const wfk_ctx* c) { return c ? c->err.c_str() : "null context"; }
int64_t wfk_launch_count(const wfk_ctx* c) { return c ? c->stats.kernel_launches : 0; }
int64_t wfk_pcg_iteration_count(const wfk_ctx* c) { return c ? c->stats.pcg_iterations : 0; }

int wfk_volume_upload(wfk_ctx* c, const wfk_volume_view* v, uint32_t fields) {
  return guard(c, [&] {
    if (!v) throw Error(WFK_E_INVALID_ARG, "null volume");
    if (v->dims[0] < 2 || v->dims[1] < 2 || v->dims[2] < 2)
      throw Error(WFK_E_INVALID_ARG, "DeformableVolume: each dim must be >= 2");
    if (!(v->voxel_size > 0)) throw Error(WFK_E_INVALID_ARG, "DeformableVolume: voxel_size must be > 0");
    VolumeDev& d = c->vol;
    const Grid g{v->dims[0], v->dims[1], v->dims[2], v->voxel_size, v->origin[0], v->origin[1], v->origin[2]};
    const int64_t n = g.n();
    if (n >= (int64_t(1) << 31)) throw Error(WFK_E_INVALID_ARG, "lattice too large for 32-bit indices");
    const bool realloc = !d.valid || d.n != n;
    if (realloc) fields = WFK_VOL_ALL;
    d.g = g;
    d.n = n;
    d.mu = v->truncation;
    d.tsdf.ensure(size_t(n));
    d.weight.ensure(size_t(n));
    d.color.ensure(3 * size_t(n));
    d.deformed.ensure(3 * size_t(n));
    d.euler.ensure(3 * size_t(n));
    d.age.ensure(size_t(n));
    d.active.ensure(size_t(n));
    cudaStream_t s = c->stream;
    auto up = [&](uint32_t bit, void* dst, const void* src, size_t bytes) {
      if (!(fields & bit)) return;
      if (!src) throw Error(WFK_E_INVALID_ARG, "volume field pointer is null");
      WFK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    };
    up(WFK_VOL_TSDF, d.tsdf, v->tsdf, size_t(n) * 4);
    up(WFK_VOL_WEIGHT, d.weight, v->weight, size_t(n) * 4);
    up(WFK_VOL_COLOR, d.color, v->color, size_t(n) * 12);
    up(WFK_VOL_DEFORMED, d.deformed, v->deformed, size_t(n) * 24);
    up(WFK_VOL_EULER, d.euler, v->euler, size_t(n) * 24);
    up(WFK_VOL_AGE, d.age, v->age, size_t(n) * 4);
    up(WFK_VOL_ACTIVE, d.active, v->active, size_t(n));
    if (fields & WFK_VOL_ACTIVE) ++d.active_gen;
    WFK_CUDA(cudaStreamSynchronize(s));
    d.valid = true;
  });
}

namespace wfk {
// DeformableVolume's constructor state (volume.cpp:8-25) on the device:
// empty TSDF, t_i = canonical position, identity rotations, age 0, inactive
__global__ void k_volume_init(Grid g, float* tsdf, float* weight, float* color, double* def, double* eul,
                              int32_t* age, uint8_t* active) {
  const int64_t n = g.n();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const V3 c = g.canonical(int(i));
    tsdf[i] = 0.f;
    weight[i] = 0.f;
    color[3 * i] = color[3 * i + 1] = color[3 * i + 2] = 0.f;
    def[3 * i] = c.x;
    def[3 * i + 1] = c.y;
    def[3 * i + 2] = c.z;
    eul[3 * i] = eul[3 * i + 1] = eul[3 * i + 2] = 0.0;
    age[i] = 0;
    active[i] = 0;
  }
}
}  // namespace wfk

int wfk_volume_create(wfk_ctx* c, const int32_t dims[3], double voxel_size, const double origin[3]) {
  return guard(c, [&] {
    if (!dims || !origin) throw Error(WFK_E_INVALID_ARG, "null argument");
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2)
      throw Error(WFK_E_INVALID_ARG, "DeformableVolume: each dim must be >= 2");
    if (!(voxel_size > 0)) throw Error(WFK_E_INVALID_ARG, "DeformableVolume: voxel_size must be > 0");
    VolumeDev& d = c->vol;
    const Grid g{dims[0], dims[1], dims[2], voxel_size, origin[0], origin[1], origin[2]};
    const int64_t n = g.n();
    if (n >= (int64_t(1) << 31)) throw Error(WFK_E_INVALID_ARG, "lattice too large for 32-bit indices");
    d.g = g;
    d.n = n;
    d.mu = 4.0 * voxel_size;  // volume.cpp:14
    d.tsdf.ensure(size_t(n));
    d.weight.ensure(size_t(n));
    d.color.ensure(3 * size_t(n));
    d.deformed.ensure(3 * size_t(n));
    d.euler.ensure(3 * size_t(n));
    d.age.ensure(size_t(n));
    d.active.ensure(size_t(n));
    k_volume_init<<<c->num_sms * 8, kBlock, 0, c->stream>>>(g, d.tsdf, d.weight, d.color, d.deformed, d.euler, d.age,
                                                         d.active);
    count_launch(c);
    WFK_CUDA(cudaGetLastError());
    ++d.active_gen;
    WFK_CUDA(cudaStreamSynchronize(c->stream));
    d.valid = true;
  });
}

int wfk_volume_checkpoint(wfk_ctx* c, int32_t restore) {
  return guard(c, [&] {
    VolumeDev& d = c->vol;
    if (!d.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
    const size_t n = size_t(d.n);
    cudaStream_t s = c->stream;
    if (!restore) {
      d.bk_deformed.ensure(3 * n);
      d.bk_euler.ensure(3 * n);
      d.bk_age.ensure(n);
      d.bk_active.ensure(n);
      WFK_CUDA(cudaMemcpyAsync(d.bk_deformed, d.deformed, 24 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.bk_euler, d.euler, 24 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.bk_age, d.age, 4 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.bk_active, d.active, n, cudaMemcpyDeviceToDevice, s));
      d.bk_valid = true;
    } else {
      if (!d.bk_valid) throw Error(WFK_E_INVALID_ARG, "no checkpoint saved");
      WFK_CUDA(cudaMemcpyAsync(d.deformed, d.bk_deformed, 24 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.euler, d.bk_euler, 24 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.age, d.bk_age, 4 * n, cudaMemcpyDeviceToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.active, d.bk_active, n, cudaMemcpyDeviceToDevice, s));
      ++d.active_gen;
    }
    WFK_CUDA(cudaStreamSynchronize(s));
  });
}

int wfk_volume_download(wfk_ctx* c, wfk_volume_view* v, uint32_t fields) {
  return guard(c, [&] {
    VolumeDev& d = c->vol;
    if (!d.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
    if (!v || int64_t(v->dims[0]) * v->dims[1] * v->dims[2] != d.n)
      throw Error(WFK_E_INVALID_ARG, "volume view does not match the device lattice");
    cudaStream_t s = c->stream;
    auto down = [&](uint32_t bit, void* dst, const void* src, size_t bytes) {
      if (!(fields & bit) || !dst) return;
      WFK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
    };
    const size_t n = size_t(d.n);
    down(WFK_VOL_TSDF, v->tsdf, d.tsdf, n * 4);
    down(WFK_VOL_WEIGHT, v->weight, d.weight, n * 4);
    down(WFK_VOL_COLOR, v->color, d.color, n * 12);
    down(WFK_VOL_DEFORMED, v->deformed, d.deformed, n * 24);
    down(WFK_VOL_EULER, v->euler, d.euler, n * 24);
    down(WFK_VOL_AGE, v->age, d.age, n * 4);
    down(WFK_VOL_ACTIVE, v->active, d.active, n);
    WFK_CUDA(cudaStreamSynchronize(s));
  });
}

int wfk_compute_active_set(wfk_ctx* c, int32_t* out, int64_t cap, int64_t* n_out) {
  return guard(c, [&] { fusion_compute_active_set(c, out, cap, n_out); });
}

int wfk_constraints_upload(wfk_ctx* c, const wfk_correspondence* h, int64_t n) {
  return guard(c, [&] {
    if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "upload the volume before its constraints");
    upload_constraints(c, h, n, false, false, nullptr);
  });
}

int wfk_constraints_append(wfk_ctx* c, const wfk_correspondence* h, int64_t n, int32_t drop_inactive, int64_t* kept) {
  return guard(c, [&] {
    if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "upload the volume before its constraints");
    upload_constraints(c, h, n, true, drop_inactive != 0, kept);
  });
}

int wfk_constraints_download(wfk_ctx* c, wfk_correspondence* out, int64_t cap, int64_t* n_out) {
  return guard(c, [&] {
    ConIn& ci = c->cons;
    const int64_t n = ci.count;
    if (n_out) *n_out = n;
    if (!out) return;
    if (n > cap) throw Error(WFK_E_CAPACITY, "constraint buffer too small");
    if (n == 0) return;
    cudaStream_t s = c->stream;
    const size_t nn = static_cast<size_t>(n);
    std::vector<int32_t> kind(nn), anchor(8 * nn);
    std::vector<double> can(3 * nn), w(8 * nn), tgt(3 * nn), nrm(3 * nn), conf(nn);
    WFK_CUDA(cudaMemcpyAsync(kind.data(), ci.kind, size_t(n) * 4, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(anchor.data(), ci.anchor, size_t(n) * 32, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(can.data(), ci.canonical, size_t(n) * 24, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(w.data(), ci.weight, size_t(n) * 64, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(tgt.data(), ci.target, size_t(n) * 24, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(nrm.data(), ci.normal, size_t(n) * 24, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(conf.data(), ci.conf, size_t(n) * 8, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    for (int64_t i = 0; i < n; ++i) {
      wfk_correspondence& r = out[i];
      std::memset(&r, 0, sizeof(r));
      r.kind = kind[size_t(i)];
      for (int k = 0; k < 3; ++k) {
        r.canonical[k] = can[size_t(3 * i + k)];
        r.target[k] = tgt[size_t(3 * i + k)];
        r.target_normal[k] = nrm[size_t(3 * i + k)];
      }
      for (int k = 0; k < 8; ++k) {
        r.anchor_index[k] = anchor[size_t(8 * i + k)];
        r.anchor_weight[k] = w[size_t(8 * i + k)];
      }
      r.confidence = conf[size_t(i)];
    }
  });
}

int wfk_evaluate_energy(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params* p, wfk_energy* out) {
  return guard(c, [&] {
    check_params(p);
    wfk_energy e{};
    solver_energy(c, pose, *p, &e);
    if (out) *out = e;
  });
}

int wfk_update_rotations(wfk_ctx* c, int32_t) {
  return guard(c, [&] { solver_rotations(c); });
}

int wfk_flip_flop_solve(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params* p, int32_t level,
                        wfk_trace_entry* trace, int32_t cap, int32_t* n_out) {
  std::vector<wfk_trace_entry> t;
  const int rc = guard(c, [&] {
    check_params(p);
    solver_flip_flop(c, pose, *p, level, t);
  });
  if (rc != WFK_OK) return rc;
  return export_trace(c, t, trace, cap, n_out);
}

int wfk_solve_coarse_to_fine(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params* p, wfk_trace_entry* trace,
                             int32_t cap, int32_t* n_out) {
  std::vector<wfk_trace_entry> t;
  const int rc = guard(c, [&] {
    check_params(p);
    solver_c2f(c, pose, *p, t);
  });
  if (rc != WFK_OK) return rc;
  return export_trace(c, t, trace, cap, n_out);
}

int wfk_solve_coarse_to_fine_dist(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params* p,
                                  wfk_trace_entry* trace, int32_t cap, int32_t* n_out) {
  std::vector<wfk_trace_entry> t;
  const int rc = guard(c, [&] {
    check_params(p);
    if (!c->dist) throw Error(WFK_E_INVALID_ARG, "wfk_dist_init first");
    solver_c2f_dist(c, pose, *p, 0, t);
  });
  if (rc != WFK_OK) return rc;
  return export_trace(c, t, trace, cap, n_out);
}

int wfk_solve_coarse_to_fine_slabs(wfk_ctx* c, int32_t slabs, const wfk_pose* pose, const wfk_solver_params* p,
                                   wfk_trace_entry* trace, int32_t cap, int32_t* n_out) {
  std::vector<wfk_trace_entry> t;
  const int rc = guard(c, [&] {
    check_params(p);
    if (slabs < 1) throw Error(WFK_E_INVALID_ARG, "slabs must be >= 1");
    solver_c2f_dist(c, pose, *p, slabs, t);
  });
  if (rc != WFK_OK) return rc;
  return export_trace(c, t, trace, cap, n_out);
}

int wfk_build_normal_equations(wfk_ctx* c, const wfk_pose* pose, const wfk_solver_params* p, wfk_ne_host* out,
                               int32_t* rows_out) {
  return guard(c, [&] {
    check_params(p);
    const int n = solver_build_ne(c, pose, *p, out);
    if (rows_out) *rows_out = n;
  });
}

int wfk_pcg_solve(wfk_ctx* c, int32_t rows, const double* blocks, const int32_t* cols, const double* rhs, double* x,
                  double tol, int32_t max_iters, int32_t, wfk_pcg_result* out) {
  return guard(c, [&] {
    if (rows < 0 || (rows > 0 && (!blocks || !cols || !rhs || !x))) throw Error(WFK_E_INVALID_ARG, "bad system");
    solver_pcg_assembled(c, rows, blocks, cols, rhs, x, tol, max_iters, 0, out, nullptr);
  });
}

int wfk_volume_save(wfk_ctx* c, const char* path) {
  return guard(c, [&] { volume_save(c, path); });
}
int wfk_volume_load(wfk_ctx* c, const char* path) {
  return guard(c, [&] { volume_load(c, path); });
}
int wfk_volume_pack(wfk_ctx* c, uint8_t* out, int64_t cap, int64_t* n_out) {
  return guard(c, [&] { volume_pack(c, out, cap, n_out); });
}
int wfk_volume_unpack(wfk_ctx* c, const uint8_t* in, int64_t n) {
  return guard(c, [&] { volume_unpack(c, in, n); });
}
int wfk_feature_store_save(wfk_ctx* c, const char* path) {
  return guard(c, [&] { feature_store_save(c, path); });
}
int wfk_feature_store_load(wfk_ctx* c, const char* path) {
  return guard(c, [&] { feature_store_load(c, path); });
}
int wfk_frame_load_pnm(wfk_ctx* c, const char* depth_pgm, const char* color_ppm, const wfk_intrinsics* intr) {
  return guard(c, [&] {
    if (!depth_pgm || !intr) throw Error(WFK_E_INVALID_ARG, "null argument");
    frame_load_pnm(c, depth_pgm, color_ppm, *intr);
  });
}
int wfk_frame_save_pnm(wfk_ctx* c, const char* depth_pgm, const char* color_ppm) {
  return guard(c, [&] { frame_save_pnm(c, depth_pgm, color_ppm); });
}
int wfk_frame_download(wfk_ctx* c, float* depth, float* color) {
  return guard(c, [&] { frame_download(c, depth, color); });
}

int wfk_dist_unique_id(uint8_t* out) {
  if (!out) return WFK_E_INVALID_ARG;
  try {
    dist_unique_id(out);
  } catch (const Error& e) {
    return e.code;
  }
  return WFK_OK;
}

int wfk_dist_init(wfk_ctx* c, int32_t rank, int32_t world, const uint8_t* id) {
  return guard(c, [&] {
    if (world > 1 && !id) throw Error(WFK_E_INVALID_ARG, "null NCCL id");
    dist_init(c, rank, world, id);
  });
}

int wfk_dist_plan(int32_t rows, const int32_t* cols, int32_t world, int32_t* ranges, int32_t* xfers, int32_t cap,
                  int32_t* n_xfers) {
  if (!n_xfers) return WFK_E_INVALID_ARG;
  try {
    dist_plan(rows, cols, world, ranges, xfers, cap, n_xfers);
  } catch (const Error& e) {
    return e.code;
  }
  return WFK_OK;
}

int wfk_slab_plan(int32_t rows, const int32_t* row_work, int32_t blocks, int32_t block_threads, int32_t ranks,
                  int32_t* n_tiles, int32_t* tile_rows, int32_t* rank_tiles) {
  if (rows < 0 || blocks < 1 || block_threads < 1 || ranks < 1 || ranks > blocks || !n_tiles || !tile_rows ||
      !rank_tiles || (rows > 0 && !row_work))
    return WFK_E_INVALID_ARG;
  try {
    const int nt = slab_tile_count(rows, blocks, block_threads);
    std::vector<int32_t> incl(size_t(std::max(rows, 1)), 0);
    int64_t acc = 0;
    for (int r = 0; r < rows; ++r) {
      acc += row_work[r];
      if (row_work[r] < 0 || acc > INT32_MAX) return WFK_E_INVALID_ARG;
      incl[size_t(r)] = int32_t(acc);
    }
    for (int t = 0; t <= nt; ++t) tile_rows[t] = slab_tile_bound_host(t, nt, rows, incl.data());
    slab_split(nt, ranks, rank_tiles);
    *n_tiles = nt;
  } catch (const Error& e) {
    return e.code;
  }
  return WFK_OK;
}

int wfk_pcg_solve_dist(wfk_ctx* c, int32_t rows, const double* blocks, const int32_t* cols, const double* rhs,
                       double* x, double tol, int32_t max_iters, wfk_pcg_result* out) {
  return guard(c, [&] {
    if (rows < 0 || (rows > 0 && (!blocks || !cols || !rhs || !x))) throw Error(WFK_E_INVALID_ARG, "bad system");
    dist_pcg(c, rows, blocks, cols, rhs, x, tol, max_iters, out);
  });
}

int wfk_pcg_solve_slabs(wfk_ctx* c, int32_t slabs, int32_t rows, const double* blocks, const int32_t* cols,
                        const double* rhs, double* x, double tol, int32_t max_iters, wfk_pcg_result* out) {
  return guard(c, [&] {
    if (rows < 0 || (rows > 0 && (!blocks || !cols || !rhs || !x))) throw Error(WFK_E_INVALID_ARG, "bad system");
    slabs_pcg(c, slabs, rows, blocks, cols, rhs, x, tol, max_iters, out);
  });
}

int wfk_ne_multiply(wfk_ctx* c, int32_t rows, const double* blocks, const int32_t* cols, const double* x, double* y) {
  return guard(c, [&] {
    if (rows < 0 || (rows > 0 && (!blocks || !cols || !x || !y))) throw Error(WFK_E_INVALID_ARG, "bad system");
    std::vector<double> xc(x, x + 3 * size_t(rows));
    solver_pcg_assembled(c, rows, blocks, cols, nullptr, xc.data(), 0, 0, 1, nullptr, y);
  });
}

int wfk_hierarchy_info(wfk_ctx* c, int32_t levels, int32_t* dims_out, int64_t* active_out) {
  return guard(c, [&] { solver_hierarchy_info(c, levels, dims_out, active_out); });
}

int wfk_frame_upload(wfk_ctx* c, const wfk_frame_view* f) {
  return guard(c, [&] {
    if (!f || !f->depth) throw Error(WFK_E_INVALID_ARG, "null frame");
    const wfk_intrinsics& K = f->intrinsics;
    if (!(K.fx > 0 && K.fy > 0 && K.width > 0 && K.height > 0))
      throw Error(WFK_E_INVALID_ARG, "frame has invalid intrinsics");
    FrameDev& d = c->frame;
    const size_t npx = size_t(K.width) * size_t(K.height);
    d.K = K;
    d.depth = d.depth_buf.ensure(npx);
    WFK_CUDA(cudaMemcpyAsync(d.depth_buf.p, f->depth, npx * 4, cudaMemcpyHostToDevice, c->stream));
    d.has_color = f->color != nullptr;
    if (d.has_color) {
      d.color = d.color_buf.ensure(3 * npx);
      WFK_CUDA(cudaMemcpyAsync(d.color_buf.p, f->color, 3 * npx * 4, cudaMemcpyHostToDevice, c->stream));
    }
    d.maps_valid = false;
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wfk_integrate_frame(wfk_ctx* c, const wfk_pose* pose, const wfk_fusion_params* p, int32_t, wfk_fusion_stats* out) {
  return guard(c, [&] {
    if (!p) throw Error(WFK_E_INVALID_ARG, "null fusion params");
    fusion_integrate(c, pose, *p, out);
  });
}

int wfk_expand_grid(wfk_ctx* c, wfk_expansion_stats* out) {
  return guard(c, [&] { fusion_expand(c, out); });
}

int wfk_advance_ages(wfk_ctx* c, const int32_t* idx, int64_t n) {
  return guard(c, [&] {
    for (int64_t k = 0; k < n; ++k)
      if (idx[k] < 0 || idx[k] >= c->vol.n) throw Error(WFK_E_OUT_OF_RANGE, "advance_ages: index outside the lattice");
    fusion_advance_ages(c, idx, n);
  });
}

int wfk_advance_active_ages(wfk_ctx* c) {
  return guard(c, [&] { fusion_advance_active_ages(c); });
}

int wfk_backproject_depth(wfk_ctx* c, int32_t, wfk_point_normal_map* out) {
  return guard(c, [&] { assoc_backproject(c, out); });
}

int wfk_extract_mesh(wfk_ctx* c, const wfk_pose* pose, int64_t* nv, int64_t* nt) {
  return guard(c, [&] { assoc_extract_mesh(c, pose, nv, nt); });
}

int wfk_mesh_warp(wfk_ctx* c, const wfk_pose* pose) {
  return guard(c, [&] { assoc_mesh_warp(c, pose); });
}

int wfk_compute_normals(wfk_ctx* c) {
  return guard(c, [&] { assoc_compute_normals(c); });
}

int wfk_mesh_upload(wfk_ctx* c, const wfk_mesh_view* m) {
  return guard(c, [&] {
    if (!m || m->num_vertices < 0 || m->num_triangles < 0) throw Error(WFK_E_INVALID_ARG, "bad mesh");
    MeshDev& d = c->mesh;
    const size_t V = size_t(m->num_vertices), T = size_t(m->num_triangles);
    for (size_t t = 0; t < 3 * T; ++t)
      if (m->triangles[t] < 0 || size_t(m->triangles[t]) >= V) throw Error(WFK_E_OUT_OF_RANGE, "triangle index");
    cudaStream_t s = c->stream;
    d.can.ensure(3 * V + 3);
    d.def.ensure(3 * V + 3);
    d.nrm.ensure(3 * V + 3);
    d.col.ensure(3 * V + 3);
    d.tri.ensure(3 * T + 3);
    if (V) {
      WFK_CUDA(cudaMemcpyAsync(d.can, m->vertices_canonical, 24 * V, cudaMemcpyHostToDevice, s));
      WFK_CUDA(cudaMemcpyAsync(d.def, m->vertices_deformed, 24 * V, cudaMemcpyHostToDevice, s));
      if (m->colors) WFK_CUDA(cudaMemcpyAsync(d.col, m->colors, 12 * V, cudaMemcpyHostToDevice, s));
      if (m->normals_deformed) WFK_CUDA(cudaMemcpyAsync(d.nrm, m->normals_deformed, 24 * V, cudaMemcpyHostToDevice, s));
    }
    if (T) WFK_CUDA(cudaMemcpyAsync(d.tri, m->triangles, 12 * T, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    d.V = int64_t(V);
    d.T = int64_t(T);
    d.normals_valid = m->normals_deformed != nullptr;
    d.adj_valid = false;
  });
}

int wfk_mesh_download(wfk_ctx* c, wfk_mesh_view* m) {
  return guard(c, [&] {
    MeshDev& d = c->mesh;
    if (!m) throw Error(WFK_E_INVALID_ARG, "null mesh view");
    const bool sizes_only = !m->vertices_canonical && !m->vertices_deformed && !m->triangles && !m->colors &&
                            !m->normals_deformed;
    if (!sizes_only && (m->num_vertices < d.V || m->num_triangles < d.T))
      throw Error(WFK_E_CAPACITY, "mesh view too small");
    m->num_vertices = d.V;
    m->num_triangles = d.T;
    if (sizes_only) return;
    cudaStream_t s = c->stream;
    const size_t V = size_t(d.V), T = size_t(d.T);
    if (V && m->vertices_canonical) WFK_CUDA(cudaMemcpyAsync(m->vertices_canonical, d.can, 24 * V, cudaMemcpyDeviceToHost, s));
    if (V && m->vertices_deformed) WFK_CUDA(cudaMemcpyAsync(m->vertices_deformed, d.def, 24 * V, cudaMemcpyDeviceToHost, s));
    if (V && m->normals_deformed && d.normals_valid)
      WFK_CUDA(cudaMemcpyAsync(m->normals_deformed, d.nrm, 24 * V, cudaMemcpyDeviceToHost, s));
    if (V && m->colors) WFK_CUDA(cudaMemcpyAsync(m->colors, d.col, 12 * V, cudaMemcpyDeviceToHost, s));
    if (T && m->triangles) WFK_CUDA(cudaMemcpyAsync(m->triangles, d.tri, 12 * T, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  });
}

int wfk_rasterize(wfk_ctx* c, const wfk_intrinsics* intr, int32_t, wfk_geometry_buffer* out) {
  return guard(c, [&] {
    if (!intr) throw Error(WFK_E_INVALID_ARG, "null intrinsics");
    assoc_rasterize(c, *intr, out);
  });
}

int wfk_maps_upload(wfk_ctx* c, const wfk_point_normal_map* m) {
  return guard(c, [&] {
    if (!m || m->width <= 0 || m->height <= 0 || !m->point || !m->normal || !m->point_valid || !m->normal_valid)
      throw Error(WFK_E_INVALID_ARG, "bad point/normal map");
    FrameDev& f = c->frame;
    const size_t npx = size_t(m->width) * size_t(m->height);
    f.point.ensure(3 * npx);
    f.normal.ensure(3 * npx);
    f.pvalid.ensure(npx);
    f.nvalid.ensure(npx);
    cudaStream_t s = c->stream;
    WFK_CUDA(cudaMemcpyAsync(f.point, m->point, npx * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(f.normal, m->normal, npx * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(f.pvalid, m->point_valid, npx, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(f.nvalid, m->normal_valid, npx, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    f.K.width = m->width;
    f.K.height = m->height;
    f.maps_valid = true;
  });
}

int wfk_gbuffer_upload(wfk_ctx* c, const wfk_geometry_buffer* b) {
  return guard(c, [&] {
    if (!b || b->width <= 0 || b->height <= 0) throw Error(WFK_E_INVALID_ARG, "bad geometry buffer");
    GBufDev& d = c->gbuf;
    const size_t npx = size_t(b->width) * size_t(b->height);
    d.w = b->width;
    d.h = b->height;
    d.depth.ensure(npx);
    d.point.ensure(3 * npx);
    d.normal.ensure(3 * npx);
    d.canonical.ensure(3 * npx);
    cudaStream_t s = c->stream;
    WFK_CUDA(cudaMemcpyAsync(d.depth, b->depth, npx * 4, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(d.point, b->point, npx * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(d.normal, b->normal, npx * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaMemcpyAsync(d.canonical, b->canonical, npx * 24, cudaMemcpyHostToDevice, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    d.valid = true;
  });
}

int wfk_find_dense_correspondences(wfk_ctx* c, const wfk_intrinsics* intr, const wfk_correspond_params* p,
                                   int32_t drop_inactive, int64_t* n_out) {
  return guard(c, [&] {
    if (!intr || !p) throw Error(WFK_E_INVALID_ARG, "null argument");
    if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
    assoc_find_dense(c, *intr, *p, drop_inactive != 0, n_out);
  });
}

// Reconstructor::process_frame (pipeline.cpp:143-262): global-pose ICP, feature front-end, association,
// coarse-to-fine solve, fusion and expansion
int wfk_process_frame(wfk_ctx* c, const wfk_frame_view* frame, const wfk_pose* pose, const wfk_pipeline_config* cfg,
                      const wfk_correspondence* sparse, int64_t nsparse, int32_t frame_index, wfk_frame_record* rec) {
  const int rc0 = wfk_frame_upload(c, frame);
  if (rc0 != WFK_OK) return rc0;
  return guard(c, [&] {
    if (!cfg || !rec) throw Error(WFK_E_INVALID_ARG, "null argument");
    if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
    std::memset(rec, 0, sizeof(*rec));
    const wfk_intrinsics& K = frame->intrinsics;
    run_frame(c, K, pose, cfg, sparse, nsparse, frame_index, rec);
  });
}

// frame already on the device (wfk_frame_stage slot)
int wfk_process_staged_frame(wfk_ctx* c, int32_t slot, const wfk_pose* pose, const wfk_pipeline_config* cfg,
                             const wfk_correspondence* sparse, int64_t nsparse, int32_t frame_index,
                             wfk_frame_record* rec) {
  return guard(c, [&] {
    if (!cfg || !rec) throw Error(WFK_E_INVALID_ARG, "null argument");
    if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
    if (slot < 0 || size_t(slot) >= c->staged_depth.size() || !c->staged_depth[size_t(slot)])
      throw Error(WFK_E_INVALID_ARG, "no frame staged in this slot");
    FrameDev& d = c->frame;
    d.K = c->staged_K[size_t(slot)];
    d.depth = c->staged_depth[size_t(slot)];
    d.color = c->staged_color[size_t(slot)];
    d.has_color = d.color != nullptr;
    d.maps_valid = false;
    std::memset(rec, 0, sizeof(*rec));
    run_frame(c, d.K, pose, cfg, sparse, nsparse, frame_index, rec);
  });
}

}  // extern "C"

namespace {
void run_frame(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose* pose_in, const wfk_pipeline_config* cfg,
               const wfk_correspondence* sparse, int64_t nsparse, int32_t frame_index, wfk_frame_record* rec) {
    // the frame's pose (the Reconstructor's pose_), refined by ICP below
    wfk_pose pose_local;
    if (pose_in) {
      pose_local = *pose_in;
    } else {
      std::memset(&pose_local, 0, sizeof(pose_local));
      pose_local.rotation[0] = pose_local.rotation[4] = pose_local.rotation[8] = 1.0;
    }
    const wfk_pose* pose = &pose_local;
    rec->pose = pose_local;
    Prof& pf = c->prof;
    double stage[kStages] = {0, 0, 0, 0, 0, 0};
    auto lap = [&](int k, int a, int b) {
      if (!pf.on) return;
      WFK_CUDA(cudaEventSynchronize(pf.ev[2 + b]));
      float ms = 0;
      WFK_CUDA(cudaEventElapsedTime(&ms, pf.ev[2 + a], pf.ev[2 + b]));
      stage[k] += ms;
    };
    stage_mark(c, 0);
    assoc_backproject(c, nullptr);
    if (frame_index == 0) {  // pipeline.cpp:150-159
      wfk_fusion_params boot = cfg->fusion;
      boot.bootstrap = 1;
      fusion_integrate(c, pose, boot, &rec->fusion);
      fusion_compute_active_set(c, nullptr, 0, nullptr);
      c->feat.n_store = 0;      // a bootstrap starts a reconstruction: its FeatureStore is empty
      c->feat.max_group = 0;
      if (cfg->use_features) {  // pipeline.cpp:155
        int32_t nf = 0;
        features_detect(c, cfg->features, nullptr, 0, &nf, nullptr);
        rec->features_added = features_add(c, *pose, frame_index, true);
      }
      rec->bootstrap = 1;
      return;
    }
    int64_t nv = 0, nt = 0;
    static const bool dbg = getenv("WFK_STAGE_DEBUG") != nullptr;
    auto timed = [&](const char* name, auto&& fn) {
      if (!dbg) return fn();
      WFK_CUDA(cudaStreamSynchronize(c->stream));
      const auto t0 = std::chrono::steady_clock::now();
      fn();
      WFK_CUDA(cudaStreamSynchronize(c->stream));
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      fprintf(stderr, "[wfk stage] frame %d %-10s %8.3f ms  (V %lld T %lld)\n", frame_index, name, ms, (long long)nv,
              (long long)nt);
    };
    // The feature detection (pyramid, DoG, extrema, orientations, descriptors)
    // reads only the frame's colour image: it runs on a side stream beside
    // the mesh / raster / ICP chain, queued after the ICP launches so its own
    // count readbacks do not hold that chain back; the matching and lifting,
    // which need the ICP pose, wait for it on the context stream.
    // WFK_NO_SIDE_FEATURES=1 keeps it in line (A/B).
    static const bool no_side = getenv("WFK_NO_SIDE_FEATURES") != nullptr;
    const bool want_features = cfg->use_features && c->frame.has_color;
    const bool side = want_features && cfg->estimate_pose && !dbg && !no_side;
    if (side) {
      if (!c->side_stream) WFK_CUDA(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
      if (!c->side_ready) WFK_CUDA(cudaEventCreateWithFlags(&c->side_ready, cudaEventDisableTiming));
      if (!c->side_done) WFK_CUDA(cudaEventCreateWithFlags(&c->side_done, cudaEventDisableTiming));
      WFK_CUDA(cudaEventRecord(c->side_ready, c->stream));  // frame image uploaded
    }
    timed("mc", [&] { assoc_extract_mesh(c, pose, &nv, &nt); });
    if (nt == 0) throw Error(WFK_E_LOGIC, "empty isosurface before frame");
    timed("normals", [&] { assoc_compute_normals(c); });
    timed("raster", [&] { assoc_rasterize(c, K, nullptr); });
    if (cfg->estimate_pose) {  // pipeline.cpp:174-183
      wfk_icp_params ip = cfg->icp;
      ip.corr = cfg->correspond;
      wfk_icp_result icp;
      if (side) {
        assoc_estimate_pose_begin(c, K, pose_local, ip);
        {
          SideScope scope(c);
          WFK_CUDA(cudaStreamWaitEvent(c->stream, c->side_ready, 0));
          int32_t nf = 0;
          features_detect(c, cfg->features, nullptr, 0, &nf, nullptr);
          WFK_CUDA(cudaEventRecord(c->side_done, c->stream));
        }
        assoc_estimate_pose_end(c, &icp);
      } else {
        timed("icp", [&] { assoc_estimate_pose(c, K, pose_local, ip, &icp); });
      }
      rec->icp_degraded = icp.degraded;
      rec->icp_rms = icp.rms;
      rec->icp_iterations = icp.iterations;
      pose_local = icp.pose;
      rec->pose = pose_local;
      timed("warp0", [&] { assoc_mesh_warp(c, pose); });  // redeform (pipeline.cpp:167-172)
      timed("normals0", [&] { assoc_compute_normals(c); });
      timed("raster0", [&] { assoc_rasterize(c, K, nullptr); });
    }
    bool features = false;
    if (want_features) {  // sparse term against the history (pipeline.cpp:185-217)
      int32_t nf = 0;
      timed("features", [&] {
        if (side)
          WFK_CUDA(cudaStreamWaitEvent(c->stream, c->side_done, 0));
        else
          features_detect(c, cfg->features, nullptr, 0, &nf, nullptr);
        features_frame_sparse(c, K, pose_local, cfg->features, &rec->match_count);
      });
      features = true;
    }
    stage_mark(c, 1);
    lap(0, 0, 1);
    std::vector<wfk_trace_entry> trace;
    for (int outer = 0; outer < cfg->reassociations; ++outer) {  // pipeline.cpp:226-247
      stage_mark(c, 2);
      int64_t nd = 0;
      assoc_find_dense(c, K, cfg->correspond, true, &nd);
      rec->dense_count = int32_t(nd);
      int64_t kept = 0, kept_caller = 0;
      if (features) kept = features_append_sparse(c);  // pipeline.cpp:229-236
      if (nsparse > 0) upload_constraints(c, sparse, nsparse, true, true, &kept_caller);
      rec->sparse_count = int32_t(kept + kept_caller);
      stage_mark(c, 3);
      lap(1, 2, 3);
      if (c->cons.count == 0) break;
      trace.clear();
      solver_c2f(c, pose, cfg->solver, trace);
      stage_mark(c, 4);
      lap(2, 3, 4);
      for (const wfk_trace_entry& e : trace) {
        rec->anomalies += e.anomaly ? 1 : 0;
        rec->pcg_iterations += e.pcg_iterations;
        ++rec->trace_len;
      }
      if (!trace.empty()) rec->energy = trace.back().energy;
      timed("warp", [&] { assoc_mesh_warp(c, pose); });  // redeform (pipeline.cpp:167-172)
      timed("normals2", [&] { assoc_compute_normals(c); });
      timed("raster2", [&] { assoc_rasterize(c, K, nullptr); });
      stage_mark(c, 5);
      lap(3, 4, 5);
    }
    stage_mark(c, 6);
    fusion_advance_active_ages(c);                      // pipeline.cpp:249-252
    fusion_integrate(c, pose, cfg->fusion, &rec->fusion);  // :254
    fusion_expand(c, &rec->expansion);                  // :255
    if (cfg->use_features && c->frame.has_color) {      // :257
      if (!features) {
        int32_t nf = 0;
        features_detect(c, cfg->features, nullptr, 0, &nf, nullptr);
      }
      timed("feat_add", [&] { rec->features_added = features_add(c, pose_local, frame_index, false); });
    }
    stage_mark(c, 7);
    lap(4, 6, 7);
    lap(5, 0, 7);
    for (int k = 0; k < kStages; ++k) pf.stage_ms[k] += stage[k];
}
}  // namespace

extern "C" {

int wfk_detect_features(wfk_ctx* c, const wfk_feature_params* p, wfk_feature* out, int32_t cap, int32_t* n_out,
                        int32_t* n_keypoints) {
  return guard(c, [&] {
    if (!p || !n_out) throw Error(WFK_E_INVALID_ARG, "null argument");
    features_detect(c, *p, out, cap, n_out, n_keypoints);
  });
}

int wfk_feature_pyramid_level(wfk_ctx* c, int32_t octave, int32_t level, int32_t dog, float* out, int32_t* width,
                              int32_t* height) {
  return guard(c, [&] {
    if (!width || !height) throw Error(WFK_E_INVALID_ARG, "null argument");
    features_level(c, octave, level, dog, out, width, height);
  });
}

int wfk_match_features(wfk_ctx* c, const wfk_feature* cur, int32_t nc, const wfk_feature* store, int32_t ns,
                       const double* predicted, const wfk_intrinsics* intr, const wfk_feature_params* p,
                       wfk_feature_match* out, int32_t cap, int32_t* n_out) {
  return guard(c, [&] {
    if (!intr || !p || !n_out) throw Error(WFK_E_INVALID_ARG, "null argument");
    features_match_host(c, cur, nc, store, ns, predicted, *intr, *p, out, cap, n_out);
  });
}

int wfk_feature_store_upload(wfk_ctx* c, const wfk_feature* in, int64_t n) {
  return guard(c, [&] { features_store_upload(c, in, n); });
}

int wfk_feature_store_download(wfk_ctx* c, wfk_feature* out, int64_t cap, int64_t* n_out) {
  return guard(c, [&] { features_store_download(c, out, cap, n_out); });
}

int wfk_invert_warp(wfk_ctx* c, const wfk_pose* pose, int64_t n, const double* y, const double* seed,
                    int32_t max_iters, double tol, double* x, uint8_t* ok) {
  return guard(c, [&] {
    if (n < 0 || (n > 0 && (!y || !seed || !x || !ok))) throw Error(WFK_E_INVALID_ARG, "null argument");
    volume_invert_warp(c, pose, n, y, seed, max_iters, tol, x, ok);
  });
}

int wfk_estimate_global_pose(wfk_ctx* c, const wfk_intrinsics* intr, const wfk_pose* initial,
                             const wfk_icp_params* params, wfk_icp_result* out) {
  return guard(c, [&] {
    if (!intr || !initial || !params || !out) throw Error(WFK_E_INVALID_ARG, "null argument");
    assoc_estimate_pose(c, *intr, *initial, *params, out);
  });
}

}  // extern "C"

extern "C" {

int wfk_profile_enable(wfk_ctx* c, int32_t on) {
  return guard(c, [&] {
    Prof& p = c->prof;
    p.on = on != 0;
    p.ff_launches = p.pcg_iterations = 0;
    p.ff_ms = p.ff_bytes = p.ff_bytes_impl = 0;
    for (double& s : p.stage_ms) s = 0;
  });
}

int wfk_profile_read(wfk_ctx* c, wfk_profile* out) {
  return guard(c, [&] {
    if (!out) throw Error(WFK_E_INVALID_ARG, "null profile");
    const Prof& p = c->prof;
    out->flip_flop_launches = p.ff_launches;
    out->pcg_iterations = p.pcg_iterations;
    out->flip_flop_ms = p.ff_ms;
    out->flip_flop_bytes = p.ff_bytes;
    out->flip_flop_bytes_impl = p.ff_bytes_impl;
    for (int k = 0; k < 6; ++k) out->stage_ms[k] = p.stage_ms[k];
    out->stage_ms[6] = out->stage_ms[7] = 0;
    out->launches = c->stats.kernel_launches;
  });
}

int wfk_timer_mark(wfk_ctx* c, int32_t slot) {
  return guard(c, [&] {
    if (slot < 0 || slot >= 16) throw Error(WFK_E_INVALID_ARG, "timer slot out of range");
    WFK_CUDA(cudaEventRecord(c->prof.timer[slot], c->stream));
  });
}

int wfk_timer_elapsed_ms(wfk_ctx* c, int32_t a, int32_t b, double* ms) {
  return guard(c, [&] {
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !ms) throw Error(WFK_E_INVALID_ARG, "bad timer slots");
    WFK_CUDA(cudaEventSynchronize(c->prof.timer[b]));
    float f = 0;
    WFK_CUDA(cudaEventElapsedTime(&f, c->prof.timer[a], c->prof.timer[b]));
    *ms = f;
  });
}

int wfk_check_enabled(void) { return check_mode() ? 1 : 0; }

__global__ void k_debug_fill(uint8_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0x5a;
}

int wfk_debug_overrun(wfk_ctx* c, int32_t past_end) {
  if (past_end < 0 || size_t(past_end) > kGuardBytes) {
    if (c) c->err = "past_end must be in [0, 256]";
    return WFK_E_INVALID_ARG;
  }
  return guard(c, [&] {
    dev_free(c->debug_buf.p);  // a fresh buffer (and canary) every call
    c->debug_buf.p = nullptr;
    c->debug_buf.cap = 0;
    uint8_t* p = c->debug_buf.ensure(4000);
    k_debug_fill<<<4, 256, 0, c->stream>>>(p, int64_t(c->debug_buf.cap) + past_end);
    WFK_CUDA(cudaGetLastError());
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wfk_flush_l2(wfk_ctx* c) {
  return guard(c, [&] {
    const size_t bytes = size_t(256) << 20;  // 2x the 126 MB L2
    uint8_t* p = c->l2_flush.ensure(bytes);
    WFK_CUDA(cudaMemsetAsync(p, c->stats.kernel_launches & 0xff, bytes, c->stream));
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int wfk_frame_stage(wfk_ctx* c, int32_t slot, const wfk_frame_view* f) {
  return guard(c, [&] {
    if (slot < 0 || slot > 4096 || !f || !f->depth) throw Error(WFK_E_INVALID_ARG, "bad slot or frame");
    const wfk_intrinsics& K = f->intrinsics;
    if (!(K.fx > 0 && K.fy > 0 && K.width > 0 && K.height > 0))
      throw Error(WFK_E_INVALID_ARG, "frame has invalid intrinsics");
    const size_t need = size_t(slot) + 1;
    if (c->staged_depth.size() < need) {
      c->staged_depth.resize(need, nullptr);
      c->staged_color.resize(need, nullptr);
      c->staged_K.resize(need);
    }
    const size_t npx = size_t(K.width) * size_t(K.height);
    float*& d = c->staged_depth[size_t(slot)];
    float*& col = c->staged_color[size_t(slot)];
    if (d) cudaFree(d);
    if (col) cudaFree(col);
    d = col = nullptr;
    WFK_CUDA(cudaMalloc(&d, npx * 4));
    WFK_CUDA(cudaMemcpyAsync(d, f->depth, npx * 4, cudaMemcpyHostToDevice, c->stream));
    if (f->color) {
      WFK_CUDA(cudaMalloc(&col, npx * 12));
      WFK_CUDA(cudaMemcpyAsync(col, f->color, npx * 12, cudaMemcpyHostToDevice, c->stream));
    }
    c->staged_K[size_t(slot)] = K;
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"

extern "C" {

int wfk_host_alloc(size_t bytes, void** out) {
  if (!out) return WFK_E_INVALID_ARG;
  *out = nullptr;
  const cudaError_t e = cudaMallocHost(out, bytes ? bytes : 1);
  return e == cudaSuccess ? WFK_OK : (e == cudaErrorMemoryAllocation ? WFK_E_OOM : WFK_E_CUDA);
}

void wfk_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
