// Snapshot and frame formats on the device:
//   * DeformableVolume::save / load (volume.cpp:150-217), "WFVOL01\n": a
//     60-byte header and one interleaved 73-byte record per lattice point
//     (tsdf, weight, color[3] float; deformed[3], euler[3] double; age int32;
//     active uint8).  The context's SoA lattice is packed into / unpacked from
//     that byte image by kernels that stage 256 records (18,688 bytes, a
//     multiple of 4) of a block in shared memory, so global memory sees
//     coalesced 32-bit words.
//   * FeatureStore::save / load (features.cpp:306-352), "WFFEAT1\n".
//   * save_depth_pgm / load_depth_pgm and save_color_ppm / load_color_ppm
//     (image.cpp:55-121): 16-bit big-endian millimetre depth and 8-bit RGB,
//     encoded from / decoded into the context's frame buffers on the device.
// The host side only parses / writes the text headers and moves the bytes.
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"

namespace wfk {

constexpr int kVolHeader = 60, kVolRecord = 73, kPackBlock = 256;
static_assert((kVolRecord * kPackBlock) % 4 == 0 && kVolHeader % 4 == 0, "word-aligned block regions");

struct VolArrays {
  int64_t n;
  float *tsdf, *weight, *color;
  double *deformed, *euler;
  int32_t* age;
  uint8_t* active;
};

template <class T>
__device__ __forceinline__ void put_bytes(unsigned char* dst, T v) {
  unsigned char b[sizeof(T)];
  memcpy(b, &v, sizeof(T));
#pragma unroll
  for (int k = 0; k < int(sizeof(T)); ++k) dst[k] = b[k];
}
template <class T>
__device__ __forceinline__ T get_bytes(const unsigned char* src) {
  unsigned char b[sizeof(T)];
#pragma unroll
  for (int k = 0; k < int(sizeof(T)); ++k) b[k] = src[k];
  T v;
  memcpy(&v, b, sizeof(T));
  return v;
}

// SoA lattice -> interleaved records (volume.cpp:163-177)
__global__ void __launch_bounds__(kPackBlock) k_vol_pack(VolArrays a, uint32_t* out_words) {
  __shared__ uint32_t sm[kVolRecord * kPackBlock / 4];
  unsigned char* sb = reinterpret_cast<unsigned char*>(sm);
  const int64_t first = int64_t(blockIdx.x) * kPackBlock;
  const int64_t i = first + threadIdx.x;
  if (i < a.n) {
    unsigned char* r = sb + threadIdx.x * kVolRecord;
    put_bytes(r + 0, a.tsdf[i]);
    put_bytes(r + 4, a.weight[i]);
    for (int k = 0; k < 3; ++k) put_bytes(r + 8 + 4 * k, a.color[3 * i + k]);
    for (int k = 0; k < 3; ++k) put_bytes(r + 20 + 8 * k, a.deformed[3 * i + k]);
    for (int k = 0; k < 3; ++k) put_bytes(r + 44 + 8 * k, a.euler[3 * i + k]);
    put_bytes(r + 68, a.age[i]);
    r[72] = a.active[i];
  }
  __syncthreads();
  const int64_t recs = min(int64_t(kPackBlock), a.n - first);
  const int64_t bytes = recs * kVolRecord;
  uint32_t* dst = out_words + (kVolHeader + first * kVolRecord) / 4;
  for (int64_t w = threadIdx.x; w < bytes / 4; w += kPackBlock) dst[w] = sm[w];
  unsigned char* dstb = reinterpret_cast<unsigned char*>(dst);
  for (int64_t b = (bytes / 4) * 4 + threadIdx.x; b < bytes; b += kPackBlock) dstb[b] = sb[b];
}

// interleaved records -> SoA lattice (volume.cpp:199-213)
__global__ void __launch_bounds__(kPackBlock) k_vol_unpack(VolArrays a, const uint32_t* in_words) {
  __shared__ uint32_t sm[kVolRecord * kPackBlock / 4];
  unsigned char* sb = reinterpret_cast<unsigned char*>(sm);
  const int64_t first = int64_t(blockIdx.x) * kPackBlock;
  const int64_t recs = min(int64_t(kPackBlock), a.n - first);
  const int64_t bytes = recs * kVolRecord;
  const uint32_t* src = in_words + (kVolHeader + first * kVolRecord) / 4;
  for (int64_t w = threadIdx.x; w < bytes / 4; w += kPackBlock) sm[w] = src[w];
  const unsigned char* srcb = reinterpret_cast<const unsigned char*>(src);
  for (int64_t b = (bytes / 4) * 4 + threadIdx.x; b < bytes; b += kPackBlock) sb[b] = srcb[b];
  __syncthreads();
  const int64_t i = first + threadIdx.x;
  if (i >= a.n) return;
  const unsigned char* r = sb + threadIdx.x * kVolRecord;
  a.tsdf[i] = get_bytes<float>(r + 0);
  a.weight[i] = get_bytes<float>(r + 4);
  for (int k = 0; k < 3; ++k) a.color[3 * i + k] = get_bytes<float>(r + 8 + 4 * k);
  for (int k = 0; k < 3; ++k) a.deformed[3 * i + k] = get_bytes<double>(r + 20 + 8 * k);
  for (int k = 0; k < 3; ++k) a.euler[3 * i + k] = get_bytes<double>(r + 44 + 8 * k);
  a.age[i] = get_bytes<int32_t>(r + 68);
  a.active[i] = r[72];
}

static VolArrays vol_arrays(VolumeDev& d) {
  return VolArrays{d.n, d.tsdf.p, d.weight.p, d.color.p, d.deformed.p, d.euler.p, d.age.p, d.active.p};
}

static void vol_header(const VolumeDev& d, unsigned char* h) {
  std::memcpy(h, "WFVOL01\n", 8);
  const int32_t dims[3] = {d.g.nx, d.g.ny, d.g.nz};
  const double rest[5] = {d.g.voxel, d.g.ox, d.g.oy, d.g.oz, d.mu};
  std::memcpy(h + 8, dims, 12);
  std::memcpy(h + 20, rest, 40);
}

int64_t volume_image_bytes(wfk_ctx* c) {
  if (!c->vol.valid) throw Error(WFK_E_INVALID_ARG, "no volume uploaded");
  return kVolHeader + c->vol.n * kVolRecord;
}

// the byte image into a device buffer (header included); returns its size
static int64_t pack_volume(wfk_ctx* c, DevBuf<uint32_t>& img) {
  VolumeDev& d = c->vol;
  const int64_t bytes = volume_image_bytes(c);
  uint32_t* w = img.ensure(size_t((bytes + 3) / 4));
  unsigned char h[kVolHeader];
  vol_header(d, h);
  WFK_CUDA(cudaMemcpyAsync(w, h, kVolHeader, cudaMemcpyHostToDevice, c->stream));
  const int blocks = int((d.n + kPackBlock - 1) / kPackBlock);
  if (blocks > 0) k_vol_pack<<<blocks, kPackBlock, 0, c->stream>>>(vol_arrays(d), w);
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
  return bytes;
}

void volume_pack(wfk_ctx* c, uint8_t* out, int64_t cap, int64_t* n_out) {
  const int64_t bytes = volume_image_bytes(c);
  if (n_out) *n_out = bytes;
  if (!out) return;
  if (cap < bytes) throw Error(WFK_E_CAPACITY, "volume image buffer too small");
  DevBuf<uint32_t> img;
  pack_volume(c, img);
  WFK_CUDA(cudaMemcpyAsync(out, img.p, size_t(bytes), cudaMemcpyDeviceToHost, c->stream));
  WFK_CUDA(cudaStreamSynchronize(c->stream));
}

// DeformableVolume::load semantics: header check, lattice (re)allocated, records unpacked
void volume_unpack(wfk_ctx* c, const uint8_t* in, int64_t n) {
  if (!in || n < kVolHeader || std::memcmp(in, "WFVOL01\n", 8) != 0)
    throw Error(WFK_E_INVALID_ARG, "bad volume snapshot header");
  int32_t dims[3];
  double rest[5];
  std::memcpy(dims, in + 8, 12);
  std::memcpy(rest, in + 20, 40);
  if (dims[0] < 2 || dims[1] < 2 || dims[2] < 2)
    throw Error(WFK_E_INVALID_ARG, "DeformableVolume: each dim must be >= 2");
  if (!(rest[0] > 0)) throw Error(WFK_E_INVALID_ARG, "DeformableVolume: voxel_size must be > 0");
  const int64_t npts = int64_t(dims[0]) * dims[1] * dims[2];
  if (npts >= (int64_t(1) << 31)) throw Error(WFK_E_INVALID_ARG, "lattice too large for 32-bit indices");
  if (n < kVolHeader + npts * kVolRecord) throw Error(WFK_E_INVALID_ARG, "truncated volume snapshot");
  VolumeDev& d = c->vol;
  d.g = Grid{dims[0], dims[1], dims[2], rest[0], rest[1], rest[2], rest[3]};
  d.n = npts;
  d.mu = rest[4];
  d.tsdf.ensure(size_t(npts));
  d.weight.ensure(size_t(npts));
  d.color.ensure(3 * size_t(npts));
  d.deformed.ensure(3 * size_t(npts));
  d.euler.ensure(3 * size_t(npts));
  d.age.ensure(size_t(npts));
  d.active.ensure(size_t(npts));
  DevBuf<uint32_t> img;
  const int64_t bytes = kVolHeader + npts * kVolRecord;
  uint32_t* w = img.ensure(size_t((bytes + 3) / 4));
  WFK_CUDA(cudaMemcpyAsync(w, in, size_t(bytes), cudaMemcpyHostToDevice, c->stream));
  k_vol_unpack<<<int((npts + kPackBlock - 1) / kPackBlock), kPackBlock, 0, c->stream>>>(vol_arrays(d), w);
  count_launch(c);
  WFK_CUDA(cudaStreamSynchronize(c->stream));
  WFK_CUDA(cudaGetLastError());
  ++d.active_gen;
  d.valid = true;
}

namespace {
struct File {
  FILE* f = nullptr;
  File(const char* path, const char* mode) : f(path ? std::fopen(path, mode) : nullptr) {}
  ~File() {
    if (f) std::fclose(f);
  }
};
std::vector<uint8_t> read_all(const char* path) {
  File fl(path, "rb");
  if (!fl.f) throw Error(WFK_E_INVALID_ARG, std::string("cannot open: ") + (path ? path : "(null)"));
  std::vector<uint8_t> b;
  uint8_t buf[1 << 16];
  size_t k;
  while ((k = std::fread(buf, 1, sizeof(buf), fl.f)) > 0) b.insert(b.end(), buf, buf + k);
  return b;
}
void write_all(const char* path, const void* p, size_t n, const std::string& head = std::string()) {
  File fl(path, "wb");
  if (!fl.f) throw Error(WFK_E_INVALID_ARG, std::string("cannot open for writing: ") + (path ? path : "(null)"));
  if (!head.empty() && std::fwrite(head.data(), 1, head.size(), fl.f) != head.size())
    throw Error(WFK_E_INVALID_ARG, "write failed");
  if (n && std::fwrite(p, 1, n, fl.f) != n) throw Error(WFK_E_INVALID_ARG, "write failed");
}
}  // namespace

void volume_save(wfk_ctx* c, const char* path) {
  DevBuf<uint32_t> img;
  const int64_t bytes = pack_volume(c, img);
  uint8_t* host = nullptr;
  WFK_CUDA(cudaMallocHost(&host, size_t(bytes)));
  try {
    WFK_CUDA(cudaMemcpyAsync(host, img.p, size_t(bytes), cudaMemcpyDeviceToHost, c->stream));
    WFK_CUDA(cudaStreamSynchronize(c->stream));
    write_all(path, host, size_t(bytes));
  } catch (...) {
    cudaFreeHost(host);
    throw;
  }
  cudaFreeHost(host);
}

void volume_load(wfk_ctx* c, const char* path) {
  const std::vector<uint8_t> b = read_all(path);
  volume_unpack(c, b.data(), int64_t(b.size()));
}

// ---------------------------------------------------------------------------
// FeatureStore::save / load (features.cpp:306-352): 8-byte magic, int32 count,
// per feature 10 doubles, 128 floats, int32 frame id (596 bytes)
// ---------------------------------------------------------------------------
constexpr int kFeatRecord = 80 + 512 + 4;

void feature_store_save(wfk_ctx* c, const char* path) {
  int64_t n = 0;
  features_store_download(c, nullptr, 0, &n);
  std::vector<wfk_feature> fs(static_cast<size_t>(n));
  if (n > 0) features_store_download(c, fs.data(), n, &n);
  std::vector<uint8_t> out(12 + size_t(n) * kFeatRecord);
  std::memcpy(out.data(), "WFFEAT1\n", 8);
  const int32_t n32 = int32_t(n);
  std::memcpy(out.data() + 8, &n32, 4);
  for (int64_t i = 0; i < n; ++i) {
    uint8_t* r = out.data() + 12 + size_t(i) * kFeatRecord;
    const wfk_feature& f = fs[size_t(i)];
    const double buf[10] = {f.canonical_pos[0], f.canonical_pos[1], f.canonical_pos[2], f.world_pos[0],
                            f.world_pos[1],     f.world_pos[2],     f.pixel[0],         f.pixel[1],
                            f.scale,            f.orientation};
    std::memcpy(r, buf, 80);
    std::memcpy(r + 80, f.descriptor, 512);
    std::memcpy(r + 592, &f.frame_id, 4);
  }
  write_all(path, out.data(), out.size());
}

void feature_store_load(wfk_ctx* c, const char* path) {
  const std::vector<uint8_t> b = read_all(path);
  if (b.size() < 12 || std::memcmp(b.data(), "WFFEAT1\n", 8) != 0)
    throw Error(WFK_E_INVALID_ARG, "bad feature store header");
  int32_t n;
  std::memcpy(&n, b.data() + 8, 4);
  if (n < 0 || b.size() < 12 + size_t(n) * kFeatRecord) throw Error(WFK_E_INVALID_ARG, "truncated feature store");
  std::vector<wfk_feature> fs(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    const uint8_t* r = b.data() + 12 + size_t(i) * kFeatRecord;
    wfk_feature& f = fs[size_t(i)];
    double buf[10];
    std::memcpy(buf, r, 80);
    for (int k = 0; k < 3; ++k) {
      f.canonical_pos[k] = buf[k];
      f.world_pos[k] = buf[3 + k];
    }
    f.pixel[0] = buf[6];
    f.pixel[1] = buf[7];
    f.scale = buf[8];
    f.orientation = buf[9];
    std::memcpy(f.descriptor, r + 80, 512);
    std::memcpy(&f.frame_id, r + 592, 4);
    f.reserved_ = 0;
  }
  features_store_upload(c, fs.data(), n);
}

// ---------------------------------------------------------------------------
// PGM / PPM (image.cpp:21-121)
// ---------------------------------------------------------------------------
__global__ void k_pgm_decode(int64_t n, const uint8_t* raster, float* depth) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint16_t v = uint16_t((raster[2 * i] << 8) | raster[2 * i + 1]);
    depth[i] = v / 1000.0f;
  }
}
__global__ void k_ppm_decode(int64_t n, const uint8_t* raster, float* color) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    color[i] = float(raster[i]);
}
__global__ void k_pgm_encode(int64_t n, const float* depth, uint8_t* raster) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double mm = double(depth[i]) * 1000.0;
    const long q = min(max(lround(mm), 0l), 65535l);
    const uint16_t v = uint16_t(q);
    raster[2 * i] = uint8_t(v >> 8);  // PGM is big-endian
    raster[2 * i + 1] = uint8_t(v & 0xff);
  }
}
__global__ void k_ppm_encode(int64_t n, const float* color, uint8_t* raster) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    raster[i] = uint8_t(min(max(lroundf(color[i]), 0l), 255l));
}

namespace {
// read_pnm_header (image.cpp:40-50): magic, then width / height / maxval each
// after whitespace and '#' comment lines, then one whitespace byte
struct Pnm {
  std::string magic;
  int w = 0, h = 0, maxval = 0;
  size_t raster = 0;  // offset of the raster
};
Pnm parse_pnm(const std::vector<uint8_t>& b) {
  Pnm p;
  size_t i = 0;
  auto skip = [&] {
    for (;;) {
      if (i < b.size() && b[i] == '#') {
        while (i < b.size() && b[i] != '\n') ++i;
        if (i < b.size()) ++i;
      } else if (i < b.size() && std::isspace(b[i])) {
        ++i;
      } else {
        break;
      }
    }
  };
  auto num = [&](int& v) {
    skip();
    size_t j = i;
    while (j < b.size() && std::isdigit(b[j])) ++j;
    if (j == i) throw Error(WFK_E_INVALID_ARG, "bad PNM header");
    v = std::stoi(std::string(b.begin() + long(i), b.begin() + long(j)));
    i = j;
  };
  skip();
  while (i < b.size() && !std::isspace(b[i])) p.magic.push_back(char(b[i++]));
  num(p.w);
  num(p.h);
  num(p.maxval);
  ++i;  // single whitespace before the raster
  p.raster = i;
  return p;
}
}  // namespace

void frame_load_pnm(wfk_ctx* c, const char* depth_path, const char* color_path, const wfk_intrinsics& K) {
  if (!(K.fx > 0 && K.fy > 0 && K.width > 0 && K.height > 0))
    throw Error(WFK_E_INVALID_ARG, "frame has invalid intrinsics");
  const std::vector<uint8_t> db = read_all(depth_path);
  const Pnm dp = parse_pnm(db);
  if (dp.magic != "P5" || dp.maxval != 65535) throw Error(WFK_E_INVALID_ARG, "expected 16-bit binary PGM");
  if (dp.w != K.width || dp.h != K.height) throw Error(WFK_E_INVALID_ARG, "depth image size does not match K");
  const size_t npx = size_t(K.width) * size_t(K.height);
  if (db.size() < dp.raster + 2 * npx) throw Error(WFK_E_INVALID_ARG, "truncated PGM");
  cudaStream_t s = c->stream;
  FrameDev& d = c->frame;
  d.K = K;
  d.depth = d.depth_buf.ensure(npx);
  uint8_t* raw = c->mask.ensure(3 * npx + 1);
  WFK_CUDA(cudaMemcpyAsync(raw, db.data() + dp.raster, 2 * npx, cudaMemcpyHostToDevice, s));
  k_pgm_decode<<<grid_for(int64_t(npx)), kBlock, 0, s>>>(int64_t(npx), raw, d.depth_buf.p);
  count_launch(c);
  d.has_color = color_path != nullptr;
  std::vector<uint8_t> cb;
  if (d.has_color) {
    WFK_CUDA(cudaStreamSynchronize(s));  // raw is reused
    cb = read_all(color_path);
    const Pnm cp = parse_pnm(cb);
    if (cp.magic != "P6" || cp.maxval != 255) throw Error(WFK_E_INVALID_ARG, "expected binary PPM");
    if (cp.w != K.width || cp.h != K.height) throw Error(WFK_E_INVALID_ARG, "color image size does not match K");
    if (cb.size() < cp.raster + 3 * npx) throw Error(WFK_E_INVALID_ARG, "truncated PPM");
    d.color = d.color_buf.ensure(3 * npx);
    WFK_CUDA(cudaMemcpyAsync(raw, cb.data() + cp.raster, 3 * npx, cudaMemcpyHostToDevice, s));
    k_ppm_decode<<<grid_for(int64_t(3 * npx)), kBlock, 0, s>>>(int64_t(3 * npx), raw, d.color_buf.p);
    count_launch(c);
  }
  d.maps_valid = false;
  WFK_CUDA(cudaStreamSynchronize(s));
  WFK_CUDA(cudaGetLastError());
}

void frame_save_pnm(wfk_ctx* c, const char* depth_path, const char* color_path) {
  FrameDev& d = c->frame;
  if (!d.depth) throw Error(WFK_E_INVALID_ARG, "no frame uploaded");
  const int W = d.K.width, H = d.K.height;
  const size_t npx = size_t(W) * size_t(H);
  cudaStream_t s = c->stream;
  uint8_t* raw = c->mask.ensure(3 * npx + 1);
  std::vector<uint8_t> host(3 * npx);
  if (depth_path) {
    k_pgm_encode<<<grid_for(int64_t(npx)), kBlock, 0, s>>>(int64_t(npx), d.depth, raw);
    count_launch(c);
    WFK_CUDA(cudaMemcpyAsync(host.data(), raw, 2 * npx, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    write_all(depth_path, host.data(), 2 * npx, "P5\n" + std::to_string(W) + " " + std::to_string(H) + "\n65535\n");
  }
  if (color_path) {
    if (!d.has_color || !d.color) throw Error(WFK_E_INVALID_ARG, "the frame has no color");
    k_ppm_encode<<<grid_for(int64_t(3 * npx)), kBlock, 0, s>>>(int64_t(3 * npx), d.color, raw);
    count_launch(c);
    WFK_CUDA(cudaMemcpyAsync(host.data(), raw, 3 * npx, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    write_all(color_path, host.data(), 3 * npx, "P6\n" + std::to_string(W) + " " + std::to_string(H) + "\n255\n");
  }
}

void frame_download(wfk_ctx* c, float* depth, float* color) {
  FrameDev& d = c->frame;
  if (!d.depth) throw Error(WFK_E_INVALID_ARG, "no frame uploaded");
  const size_t npx = size_t(d.K.width) * size_t(d.K.height);
  if (depth) WFK_CUDA(cudaMemcpyAsync(depth, d.depth, npx * 4, cudaMemcpyDeviceToHost, c->stream));
  if (color && d.has_color) WFK_CUDA(cudaMemcpyAsync(color, d.color, 3 * npx * 4, cudaMemcpyDeviceToHost, c->stream));
  WFK_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace wfk
