// ORACLE (test infrastructure only): CPU restatement of the reference's snapshot
// and frame formats, used by tests/ to check libwfk's device codecs byte for byte.
//   DeformableVolume::save / load  volume.cpp:150-217   "WFVOL01\n"
//   FeatureStore::save / load      features.cpp:306-352 "WFFEAT1\n"
//   save/load_depth_pgm, save/load_color_ppm  image.cpp:21-121
// Parity pinned by construction against the reference's write order (field by
// field, native little-endian, PGM big-endian) and its round-trip tests
// (test_volume.cpp save/load, test_features.cpp store save/load).
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "wfo.h"

namespace {
template <class T>
void put(std::vector<uint8_t>& b, const T& v) {
  const auto* p = reinterpret_cast<const uint8_t*>(&v);
  b.insert(b.end(), p, p + sizeof(T));
}
template <class T>
T get(const uint8_t*& p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  p += sizeof(T);
  return v;
}
int out_bytes(const std::vector<uint8_t>& b, uint8_t* out, int64_t cap, int64_t* n_out) {
  *n_out = int64_t(b.size());
  if (!out) return WFK_OK;
  if (cap < int64_t(b.size())) return WFK_E_CAPACITY;
  std::memcpy(out, b.data(), b.size());
  return WFK_OK;
}
// read_pnm_header (image.cpp:40-50)
bool pnm_header(const uint8_t* b, int64_t n, std::string& magic, int& w, int& h, int& maxval, int64_t& raster) {
  int64_t i = 0;
  auto skip = [&] {
    for (;;) {
      if (i < n && b[i] == '#') {
        while (i < n && b[i] != '\n') ++i;
        if (i < n) ++i;
      } else if (i < n && std::isspace(b[i])) {
        ++i;
      } else {
        break;
      }
    }
  };
  auto num = [&](int& v) {
    skip();
    int64_t j = i;
    v = 0;
    while (j < n && std::isdigit(b[j])) v = v * 10 + (b[j++] - '0');
    const bool ok = j > i;
    i = j;
    return ok;
  };
  skip();
  magic.clear();
  while (i < n && !std::isspace(b[i])) magic.push_back(char(b[i++]));
  if (!num(w) || !num(h) || !num(maxval)) return false;
  ++i;
  raster = i;
  return true;
}
}  // namespace

extern "C" {

// DeformableVolume::save (volume.cpp:150-178)
int wfo_volume_save_bytes(const wfk_volume_view* v, uint8_t* out, int64_t cap, int64_t* n_out) {
  std::vector<uint8_t> b;
  const char magic[8] = {'W', 'F', 'V', 'O', 'L', '0', '1', '\n'};
  b.insert(b.end(), magic, magic + 8);
  for (int k = 0; k < 3; ++k) put(b, int32_t(v->dims[k]));
  put(b, v->voxel_size);
  for (int k = 0; k < 3; ++k) put(b, v->origin[k]);
  put(b, v->truncation);
  const int64_t n = int64_t(v->dims[0]) * v->dims[1] * v->dims[2];
  b.reserve(b.size() + size_t(n) * 73);
  for (int64_t i = 0; i < n; ++i) {
    put(b, v->tsdf[i]);
    put(b, v->weight[i]);
    for (int k = 0; k < 3; ++k) put(b, v->color[3 * i + k]);
    for (int k = 0; k < 3; ++k) put(b, v->deformed[3 * i + k]);
    for (int k = 0; k < 3; ++k) put(b, v->euler[3 * i + k]);
    put(b, v->age[i]);
    put(b, v->active[i]);
  }
  return out_bytes(b, out, cap, n_out);
}

// DeformableVolume::load (volume.cpp:180-217): header into dims / geometry; with
// arrays in `v` (sized for those dims) the records as well
int wfo_volume_load_bytes(const uint8_t* in, int64_t n, wfk_volume_view* v) {
  if (n < 60 || std::memcmp(in, "WFVOL01\n", 8) != 0) return WFK_E_INVALID_ARG;
  const uint8_t* p = in + 8;
  for (int k = 0; k < 3; ++k) v->dims[k] = get<int32_t>(p);
  v->voxel_size = get<double>(p);
  for (int k = 0; k < 3; ++k) v->origin[k] = get<double>(p);
  v->truncation = get<double>(p);
  const int64_t np = int64_t(v->dims[0]) * v->dims[1] * v->dims[2];
  if (!v->tsdf) return WFK_OK;
  if (n < 60 + np * 73) return WFK_E_INVALID_ARG;
  for (int64_t i = 0; i < np; ++i) {
    v->tsdf[i] = get<float>(p);
    v->weight[i] = get<float>(p);
    for (int k = 0; k < 3; ++k) v->color[3 * i + k] = get<float>(p);
    for (int k = 0; k < 3; ++k) v->deformed[3 * i + k] = get<double>(p);
    for (int k = 0; k < 3; ++k) v->euler[3 * i + k] = get<double>(p);
    v->age[i] = get<int32_t>(p);
    v->active[i] = get<uint8_t>(p);
  }
  return WFK_OK;
}

// FeatureStore::save (features.cpp:306-323)
int wfo_feature_store_bytes(const wfk_feature* f, int32_t nf, uint8_t* out, int64_t cap, int64_t* n_out) {
  std::vector<uint8_t> b;
  const char magic[8] = {'W', 'F', 'F', 'E', 'A', 'T', '1', '\n'};
  b.insert(b.end(), magic, magic + 8);
  put(b, nf);
  for (int32_t i = 0; i < nf; ++i) {
    const double buf[10] = {f[i].canonical_pos[0], f[i].canonical_pos[1], f[i].canonical_pos[2],
                            f[i].world_pos[0],     f[i].world_pos[1],     f[i].world_pos[2],
                            f[i].pixel[0],         f[i].pixel[1],         f[i].scale,
                            f[i].orientation};
    for (double d : buf) put(b, d);
    for (int k = 0; k < 128; ++k) put(b, f[i].descriptor[k]);
    put(b, int32_t(f[i].frame_id));
  }
  return out_bytes(b, out, cap, n_out);
}

// save_depth_pgm (image.cpp:55-69)
int wfo_pgm_encode(const float* depth, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out) {
  const std::string head = "P5\n" + std::to_string(w) + " " + std::to_string(h) + "\n65535\n";
  std::vector<uint8_t> b(head.begin(), head.end());
  for (int64_t i = 0; i < int64_t(w) * h; ++i) {
    const double mm = depth[i] * 1000.0;
    const uint16_t v = static_cast<uint16_t>(std::clamp(std::lround(mm), 0l, 65535l));
    b.push_back(uint8_t(v >> 8));
    b.push_back(uint8_t(v & 0xff));
  }
  return out_bytes(b, out, cap, n_out);
}

// save_color_ppm (image.cpp:90-104)
int wfo_ppm_encode(const float* color, int32_t w, int32_t h, uint8_t* out, int64_t cap, int64_t* n_out) {
  const std::string head = "P6\n" + std::to_string(w) + " " + std::to_string(h) + "\n255\n";
  std::vector<uint8_t> b(head.begin(), head.end());
  for (int64_t i = 0; i < 3 * int64_t(w) * h; ++i)
    b.push_back(static_cast<uint8_t>(std::clamp(std::lround(color[i]), 0l, 255l)));
  return out_bytes(b, out, cap, n_out);
}

// load_depth_pgm / load_color_ppm (image.cpp:71-88, 106-121): channels 1 (PGM) or 3 (PPM)
int wfo_pnm_decode(const uint8_t* in, int64_t n, int32_t channels, int32_t* w, int32_t* h, float* out) {
  std::string magic;
  int W, H, maxval;
  int64_t raster;
  if (!pnm_header(in, n, magic, W, H, maxval, raster)) return WFK_E_INVALID_ARG;
  if (channels == 1 && (magic != "P5" || maxval != 65535)) return WFK_E_INVALID_ARG;
  if (channels == 3 && (magic != "P6" || maxval != 255)) return WFK_E_INVALID_ARG;
  *w = W;
  *h = H;
  if (!out) return WFK_OK;
  const int64_t npx = int64_t(W) * H;
  if (n < raster + (channels == 1 ? 2 : 3) * npx) return WFK_E_INVALID_ARG;
  const uint8_t* r = in + raster;
  if (channels == 1)
    for (int64_t i = 0; i < npx; ++i) out[i] = uint16_t((r[2 * i] << 8) | r[2 * i + 1]) / 1000.0f;
  else
    for (int64_t i = 0; i < 3 * npx; ++i) out[i] = float(r[i]);
  return WFK_OK;
}

}  // extern "C"
