// Feature front-end on sm_100a (features.cpp:12-433, image.cpp:10-17): the
// DoG pyramid, scale-space extrema with the edge test, dominant orientations
// and 4x4x8 descriptors of the context's frame, and mutual-best matching of a
// frame's features against a feature store.
//
// Float work stays float and every multiply/add is rounded separately
// (-fmad=false), so gray levels, pyramid, DoG, extrema, their stable order and
// the edge test are bit-identical to the reference.  Orientation histograms
// and descriptors call device hypot/atan2/exp/cos/sin (glibc's last bits can
// differ): one thread per keypoint keeps the reference's accumulation order,
// so results agree to rounding.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"

namespace wfk {

constexpr int kMaxTaps = 31;  // blur radius <= 15 (sigma <= 5)
struct Taps {
  float k[kMaxTaps];
  int radius;
};
// gaussian_blur's taps (features.cpp:14-21), on the host as the reference computes them
static Taps blur_taps(double sigma) {
  Taps t{};
  t.radius = std::max(1, int(std::ceil(3.0 * sigma)));
  if (2 * t.radius + 1 > kMaxTaps) throw Error(WFK_E_INVALID_ARG, "feature blur sigma too large");
  float sum = 0;
  for (int i = -t.radius; i <= t.radius; ++i) {
    t.k[i + t.radius] = float(std::exp(-0.5 * i * i / (sigma * sigma)));
    sum += t.k[i + t.radius];
  }
  for (int i = 0; i < 2 * t.radius + 1; ++i) t.k[i] /= sum;
  return t;
}

struct FlagToInt {
  __host__ __device__ int32_t operator()(uint8_t v) const { return v; }
};
__global__ void k_iota(int n, int32_t* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = i;
}
__global__ void k_gray(int64_t n, const float* rgb, float* g) {  // to_gray (image.cpp:10-17)
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    g[i] = (0.299f * rgb[3 * i] + 0.587f * rgb[3 * i + 1] + 0.114f * rgb[3 * i + 2]) / 255.0f;
}
template <bool X>
__global__ void k_blur(int w, int h, const float* in, float* out, Taps t) {
  const int64_t n = int64_t(w) * h;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(p % w), y = int(p / w);
    float acc = 0;
    for (int i = -t.radius; i <= t.radius; ++i) {
      const float v = X ? in[int64_t(y) * w + min(max(x + i, 0), w - 1)] : in[int64_t(min(max(y + i, 0), h - 1)) * w + x];
      acc += t.k[i + t.radius] * v;
    }
    out[p] = acc;
  }
}
__global__ void k_sub(int64_t n, const float* a, const float* b, float* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}
__global__ void k_down2(int w, int h, const float* in, int wo, int ho, float* out) {
  const int64_t n = int64_t(wo) * ho;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(p % wo), y = int(p / wo);
    out[p] = in[int64_t(2 * y) * w + 2 * x];
  }
}

// scale-space extrema of one DoG level (features.cpp:150-185); flag[p] = 1
// for a kept extremum at pixel p of octave o
struct ExtArgs {
  const float *dm, *d0, *dp;  // DoG levels l - 1, l, l + 1
  int w, h, scale;
  double contrast, edge_limit;
  const float* depth;
  int dw, dh;
};
__global__ void k_extrema(ExtArgs a, uint8_t* flag) {
  const int64_t n = int64_t(a.w) * a.h;
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    const int x = int(p % a.w), y = int(p / a.w);
    uint8_t keep = 0;
    if (x >= 1 && y >= 1 && x < a.w - 1 && y < a.h - 1) {
      const float v = a.d0[p];
      if (!(fabsf(v) < a.contrast)) {
        bool is_max = true, is_min = true;
        const float* lv[3] = {a.dm, a.d0, a.dp};
        for (int dl = 0; dl < 3 && (is_max || is_min); ++dl)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              if (dl == 1 && dx == 0 && dy == 0) continue;
              const float nv = lv[dl][int64_t(y + dy) * a.w + (x + dx)];
              if (nv >= v) is_max = false;
              if (nv <= v) is_min = false;
            }
        if (is_max || is_min) {
          auto d = [&](int xx, int yy) { return a.d0[int64_t(yy) * a.w + xx]; };
          const double dxx = d(x + 1, y) + d(x - 1, y) - 2 * v;
          const double dyy = d(x, y + 1) + d(x, y - 1) - 2 * v;
          const double dxy = 0.25 * (d(x + 1, y + 1) - d(x - 1, y + 1) - d(x + 1, y - 1) + d(x - 1, y - 1));
          const double tr = dxx + dyy, det = dxx * dyy - dxy * dxy;
          if (!(det <= 0 || tr * tr / det >= a.edge_limit)) {
            const int fx = x * a.scale, fy = y * a.scale;
            if (fx >= 0 && fy >= 0 && fx < a.dw && fy < a.dh && a.depth[int64_t(fy) * a.dw + fx] > 0.f) keep = 1;
          }
        }
      }
    }
    flag[p] = keep;
  }
}
// extremum records in (octave, level, y, x) order
__global__ void k_ext_write(int64_t n, const uint8_t* flag, const int32_t* pos, int octave, int w, const float* d0,
                            int4* ext, uint32_t* key) {
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < n; p += int64_t(gridDim.x) * blockDim.x) {
    if (!flag[p]) continue;
    const int k = pos[p];
    const float v = d0[p];
    ext[k] = make_int4(octave, int(p % w), int(p / w), __float_as_int(v));
    key[k] = __float_as_uint(fabsf(v));  // |response|: positive floats order as their bits
  }
}

struct OctImg {
  const float* g1[8];  // gauss[o][1]
  int w[8], h[8];
};
// dominant_orientations (features.cpp:94-132), one thread per extremum
__global__ void k_orientations(int n, const int4* ext, const int32_t* order, OctImg im, double sigma,
                               wfk_feature_params p, double* ori, int32_t* nori) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int4 e = ext[order[i]];
    const float* img = im.g1[e.x];
    const int W = im.w[e.x], H = im.h[e.x];
    constexpr int kBins = 36;
    double hist[kBins];
    for (int b = 0; b < kBins; ++b) hist[b] = 0;
    const double win_sigma = 1.5 * sigma;
    const int radius = max(1, int(llround(3.0 * win_sigma)));
    const int cx = e.y, cy = e.z;
    for (int dy = -radius; dy <= radius; ++dy)
      for (int dx = -radius; dx <= radius; ++dx) {
        const int px = cx + dx, py = cy + dy;
        if (px < 1 || py < 1 || px >= W - 1 || py >= H - 1) continue;
        const double gx = img[int64_t(py) * W + px + 1] - img[int64_t(py) * W + px - 1];
        const double gy = img[int64_t(py + 1) * W + px] - img[int64_t(py - 1) * W + px];
        const double mag = hypot(gx, gy);
        const double theta = atan2(gy, gx);
        const double w = exp(-0.5 * (dx * dx + dy * dy) / (win_sigma * win_sigma));
        int bin = int(floor((theta + M_PI) / (2 * M_PI) * kBins));
        bin = min(max(bin, 0), kBins - 1);
        hist[bin] += w * mag;
      }
    double peak = hist[0];
    for (int b = 1; b < kBins; ++b) peak = fmax(peak, hist[b]);
    int cnt = 0;
    double val[2] = {0, 0}, ang[2] = {0, 0};
    if (peak > 0) {
      // candidates in bin order, stable by decreasing value: keep the best max_orientations (<= 2)
      for (int b = 0; b < kBins; ++b) {
        const double l = hist[(b + kBins - 1) % kBins], r = hist[(b + 1) % kBins];
        if (hist[b] >= p.orientation_peak_ratio * peak && hist[b] > l && hist[b] > r) {
          const double denom = l - 2 * hist[b] + r;
          const double off = fabs(denom) > 1e-12 ? 0.5 * (l - r) / denom : 0.0;
          const double a = (b + 0.5 + off) / kBins * 2 * M_PI - M_PI;
          // insert keeping (value desc, earlier bin first on ties)
          int at = cnt;
          while (at > 0 && val[at - 1] < hist[b]) --at;
          if (at < 2) {
            for (int q = min(cnt, 1); q > at; --q) {
              val[q] = val[q - 1];
              ang[q] = ang[q - 1];
            }
            val[at] = hist[b];
            ang[at] = a;
            cnt = min(cnt + 1, 2);
          }
        }
      }
    }
    nori[i] = min(cnt, p.max_orientations);
    ori[2 * i] = ang[0];
    ori[2 * i + 1] = ang[1];
  }
}
// keypoints in extremum order until max_keypoints (features.cpp:188-207)
struct KpDev {
  int octave, ox, oy, pad;
  double scale, orientation;
};
__global__ void k_assemble_kp(int n, const int4* ext, const int32_t* order, const double* ori, const int32_t* nori,
                              int max_kp, double sigma_oct, KpDev* kp, int32_t* n_kp) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int m = 0;
  for (int i = 0; i < n && m < max_kp; ++i) {
    const int4 e = ext[order[i]];
    for (int q = 0; q < nori[i] && m < max_kp; ++q) {
      KpDev k;
      k.octave = e.x;
      k.ox = e.y;
      k.oy = e.z;
      k.pad = 0;
      k.scale = sigma_oct * double(1 << e.x);
      k.orientation = ori[2 * i + q];
      kp[m++] = k;
    }
  }
  *n_kp = m;
}
// extract_descriptors (features.cpp:212-286), one thread per keypoint
__global__ void k_descriptors(const int32_t* n_kp, const KpDev* kps, OctImg im, double sigma_oct,
                              wfk_feature* out, uint8_t* ok) {
  const int n = *n_kp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const KpDev kp = kps[i];
    const float* img = im.g1[kp.octave];
    const int W = im.w[kp.octave], H = im.h[kp.octave];
    constexpr int kCells = 4, kOriBins = 8;
    const double cell = 3.0 * sigma_oct;
    const double radius = cell * (kCells + 1) * sqrt(2.0) * 0.5;
    const double cx = kp.ox, cy = kp.oy;
    ok[i] = 0;
    if (cx - radius < 1 || cy - radius < 1 || cx + radius >= W - 1 || cy + radius >= H - 1) continue;
    const double ct = cos(kp.orientation), st = sin(kp.orientation);
    double hist[kCells * kCells * kOriBins];
    for (int q = 0; q < kCells * kCells * kOriBins; ++q) hist[q] = 0;
    const int r = int(ceil(radius));
    for (int dy = -r; dy <= r; ++dy)
      for (int dx = -r; dx <= r; ++dx) {
        const double rx = (ct * dx + st * dy) / cell;
        const double ry = (-st * dx + ct * dy) / cell;
        const double bx = rx + kCells / 2.0 - 0.5;
        const double by = ry + kCells / 2.0 - 0.5;
        if (bx <= -1 || by <= -1 || bx >= kCells || by >= kCells) continue;
        const int px = kp.ox + dx, py = kp.oy + dy;
        const double gx = img[int64_t(py) * W + px + 1] - img[int64_t(py) * W + px - 1];
        const double gy = img[int64_t(py + 1) * W + px] - img[int64_t(py - 1) * W + px];
        const double mag = hypot(gx, gy);
        double theta = atan2(gy, gx) - kp.orientation;
        while (theta < 0) theta += 2 * M_PI;
        while (theta >= 2 * M_PI) theta -= 2 * M_PI;
        const double ob = theta / (2 * M_PI) * kOriBins;
        const double w = mag * exp(-0.5 * (rx * rx + ry * ry) / ((kCells / 2.0) * (kCells / 2.0)));
        const int x0 = int(floor(bx)), y0 = int(floor(by));
        const int o0 = int(floor(ob)) % kOriBins;
        const double fx = bx - floor(bx), fy = by - floor(by), fo = ob - floor(ob);
        for (int ix = 0; ix < 2; ++ix)
          for (int iy = 0; iy < 2; ++iy)
            for (int io = 0; io < 2; ++io) {
              const int xx = x0 + ix, yy = y0 + iy;
              if (xx < 0 || yy < 0 || xx >= kCells || yy >= kCells) continue;
              const int oo = (o0 + io) % kOriBins;
              hist[(yy * kCells + xx) * kOriBins + oo] +=
                  w * (ix ? fx : 1 - fx) * (iy ? fy : 1 - fy) * (io ? fo : 1 - fo);
            }
      }
    wfk_feature& f = out[i];
    const int scale = 1 << kp.octave;
    for (int q = 0; q < 3; ++q) f.canonical_pos[q] = f.world_pos[q] = 0;
    f.pixel[0] = double(kp.ox * scale);
    f.pixel[1] = double(kp.oy * scale);
    f.scale = kp.scale;
    f.orientation = kp.orientation;
    f.frame_id = -1;
    f.reserved_ = 0;
    double norm = 0;
    for (int q = 0; q < 128; ++q) {
      f.descriptor[q] = float(hist[q]);
      norm += f.descriptor[q] * f.descriptor[q];
    }
    norm = sqrt(norm);
    if (norm < 1e-12) continue;  // flat patch
    double norm2 = 0;
    for (int q = 0; q < 128; ++q) {
      const float v = fminf(f.descriptor[q] / float(norm), 0.2f);
      f.descriptor[q] = v;
      norm2 += v * v;
    }
    norm2 = sqrt(norm2);
    for (int q = 0; q < 128; ++q) f.descriptor[q] = float(f.descriptor[q] / norm2);
    ok[i] = 1;
  }
}

// The whole detection of the context's frame; features land in c->feat.cur
// (device) and, when out != null, on the host.
void features_detect(wfk_ctx* c, const wfk_feature_params& p, wfk_feature* out, int32_t cap, int32_t* n_out,
                     int32_t* n_kp_out) {
  FrameDev& f = c->frame;
  *n_out = 0;
  if (n_kp_out) *n_kp_out = 0;
  c->feat.n_cur = 0;
  if (!f.depth) throw Error(WFK_E_INVALID_ARG, "no frame uploaded");
  if (!f.has_color || !f.color) return;  // pipeline.cpp:96
  const int W = f.K.width, H = f.K.height;
  if (W < 64 || H < 64) return;          // pipeline.cpp:98
  if (p.octaves < 1 || p.octaves > 8 || p.dog_levels < 1) throw Error(WFK_E_INVALID_ARG, "bad feature params");
  cudaStream_t s = c->stream;
  FeatDev& fd = c->feat;
  const int L = p.dog_levels;
  // pyramid: per octave L + 1 gaussian levels and L DoG levels (features.cpp:57-88)
  if (2 * L + 2 > kFeatLevels || p.max_orientations > 2)
    throw Error(WFK_E_INVALID_ARG, "feature params beyond the device limits (dog_levels <= 7, max_orientations <= 2)");
  auto G = [&](int o, int l) -> DevBuf<float>& { return fd.levels[o][l]; };
  auto D = [&](int o, int l) -> DevBuf<float>& { return fd.levels[o][L + 1 + l]; };
  fd.L = L;
  fd.ws.assign(size_t(p.octaves), 0);
  fd.hs.assign(size_t(p.octaves), 0);
  std::vector<int>& ws = fd.ws;
  std::vector<int>& hs = fd.hs;
  const double k = std::pow(2.0, 1.0 / L);
  const size_t npx = size_t(W) * H;
  float* gray = fd.gray.ensure(npx);
  float* tmp = fd.tmp.ensure(npx);
  k_gray<<<grid_for(int64_t(npx)), kBlock, 0, s>>>(int64_t(npx), f.color, gray);
  count_launch(c);
  const float* base = gray;
  int w = W, h = H;
  for (int o = 0; o < p.octaves; ++o) {
    ws[size_t(o)] = w;
    hs[size_t(o)] = h;
    const int64_t n = int64_t(w) * h;
    for (int l = 0; l <= L; ++l) {
      const double sigma = l == 0 ? p.sigma0
                                  : std::sqrt(std::pow(p.sigma0 * std::pow(k, l), 2) -
                                              std::pow(p.sigma0 * std::pow(k, l - 1), 2));
      const Taps t = blur_taps(sigma);
      float* dst = G(o, l).ensure(size_t(n));
      const float* src = l == 0 ? base : G(o, l - 1).p;
      k_blur<true><<<grid_for(n), kBlock, 0, s>>>(w, h, src, tmp, t);
      k_blur<false><<<grid_for(n), kBlock, 0, s>>>(w, h, tmp, dst, t);
      count_launch(c, 2);
    }
    for (int l = 0; l < L; ++l) {
      k_sub<<<grid_for(n), kBlock, 0, s>>>(n, G(o, l + 1).p, G(o, l).p, D(o, l).ensure(size_t(n)));
      count_launch(c);
    }
    if (o + 1 < p.octaves) {
      const int wn = w / 2, hn = h / 2;
      float* nb = fd.base.ensure(size_t(wn) * hn + 1);  // consumed by the next octave's first blur
      k_down2<<<grid_for(int64_t(wn) * hn), kBlock, 0, s>>>(w, h, G(o, L).p, wn, hn, nb);
      count_launch(c);
      base = nb;
      w = wn;
      h = hn;
    }
  }
  // extrema in (octave, level, y, x) order (features.cpp:146-185)
  const double edge_limit = (p.edge_ratio + 1) * (p.edge_ratio + 1) / p.edge_ratio;
  int64_t total = 0;
  std::vector<int64_t> off;
  for (int o = 0; o < p.octaves; ++o)
    for (int l = 1; l + 1 < L; ++l) {
      off.push_back(total);
      total += int64_t(ws[size_t(o)]) * hs[size_t(o)];
    }
  int32_t n_ext = 0;
  if (total > 0) {
    uint8_t* flag = fd.flag.ensure(size_t(total) + 1);
    int32_t* pos = fd.pos.ensure(size_t(total) + 1);
    size_t q = 0;
    for (int o = 0; o < p.octaves; ++o)
      for (int l = 1; l + 1 < L; ++l, ++q) {
        ExtArgs a;
        a.dm = D(o, l - 1).p;
        a.d0 = D(o, l).p;
        a.dp = D(o, l + 1).p;
        a.w = ws[size_t(o)];
        a.h = hs[size_t(o)];
        a.scale = 1 << o;
        a.contrast = p.contrast_threshold;
        a.edge_limit = edge_limit;
        a.depth = f.depth;
        a.dw = W;
        a.dh = H;
        k_extrema<<<grid_for(int64_t(a.w) * a.h), kBlock, 0, s>>>(a, flag + off[q]);
        count_launch(c);
      }
    WFK_CUDA(cudaMemsetAsync(flag + total, 0, 1, s));
    thrust::transform_iterator<FlagToInt, const uint8_t*, int32_t> it(flag, FlagToInt());
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, it, pos, int(total + 1), s);
    c->temp.ensure(tb);
    WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tb, it, pos, int(total + 1), s));
    WFK_CUDA(cudaMemcpyAsync(c->h_pinned, pos + total, 4, cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
    n_ext = c->h_pinned[0];
    if (n_ext > 0) {
      int4* ext = fd.ext.ensure(size_t(n_ext));
      uint32_t* key = fd.key.ensure(2 * size_t(n_ext));
      int32_t* idx = fd.idx.ensure(2 * size_t(n_ext));
      q = 0;
      for (int o = 0; o < p.octaves; ++o)
        for (int l = 1; l + 1 < L; ++l, ++q) {
          const int64_t n = int64_t(ws[size_t(o)]) * hs[size_t(o)];
          k_ext_write<<<grid_for(n), kBlock, 0, s>>>(n, flag + off[q], pos + off[q], o, ws[size_t(o)], D(o, l).p,
                                                     ext, key);
          count_launch(c);
        }
      k_iota<<<grid_for(n_ext), kBlock, 0, s>>>(n_ext, idx);
      // stable sort by decreasing |response| (features.cpp:187-189)
      cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, key, key + n_ext, idx, idx + n_ext, n_ext, 0, 32, s);
      c->temp.ensure(tb);
      WFK_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->temp.p, tb, key, key + n_ext, idx, idx + n_ext, n_ext, 0,
                                                         32, s));
    }
  }
  if (n_ext == 0) return;
  OctImg im{};
  for (int o = 0; o < p.octaves && o < 8; ++o) {
    im.g1[o] = G(o, 1).p;
    im.w[o] = ws[size_t(o)];
    im.h[o] = hs[size_t(o)];
  }
  const double sigma_oct = p.sigma0 * std::pow(k, 1.5);
  const int32_t* order = fd.idx.p + n_ext;
  double* ori = fd.ori.ensure(2 * size_t(n_ext));
  int32_t* nori = fd.nori.ensure(size_t(n_ext));
  k_orientations<<<grid_for(n_ext, 64), 64, 0, s>>>(n_ext, fd.ext, order, im, sigma_oct, p, ori, nori);
  KpDev* kp = reinterpret_cast<KpDev*>(fd.kp.ensure(size_t(std::max(p.max_keypoints, 1)) * sizeof(KpDev)));
  int32_t* nkp = fd.cnt.ensure(4);
  k_assemble_kp<<<1, 32, 0, s>>>(n_ext, fd.ext, order, ori, nori, p.max_keypoints, sigma_oct, kp, nkp);
  const int maxk = std::max(p.max_keypoints, 1);
  wfk_feature* cur = reinterpret_cast<wfk_feature*>(fd.cur_raw.ensure(size_t(maxk) * sizeof(wfk_feature)));
  uint8_t* ok = fd.ok.ensure(size_t(maxk));
  k_descriptors<<<grid_for(maxk, 32), 32, 0, s>>>(nkp, kp, im, sigma_oct, cur, ok);
  count_launch(c, 3);
  // compact the valid descriptors in keypoint order (host side: <= max_keypoints records)
  int32_t n_kp = 0;
  WFK_CUDA(cudaMemcpyAsync(&n_kp, nkp, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  std::vector<wfk_feature> hf(static_cast<size_t>(n_kp));
  std::vector<uint8_t> hok(static_cast<size_t>(n_kp));
  if (n_kp > 0) {
    WFK_CUDA(cudaMemcpyAsync(hf.data(), cur, size_t(n_kp) * sizeof(wfk_feature), cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaMemcpyAsync(hok.data(), ok, size_t(n_kp), cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  }
  fd.host_cur.clear();
  for (int i = 0; i < n_kp; ++i)
    if (hok[size_t(i)]) fd.host_cur.push_back(hf[size_t(i)]);
  fd.n_cur = int32_t(fd.host_cur.size());
  *n_out = fd.n_cur;
  if (n_kp_out) *n_kp_out = n_kp;
  if (out) {
    if (fd.n_cur > cap) throw Error(WFK_E_CAPACITY, "feature buffer too small");
    std::copy(fd.host_cur.begin(), fd.host_cur.end(), out);
  }
}

// one pyramid level of the last detection (tests)
void features_level(wfk_ctx* c, int o, int l, int dog, float* out, int32_t* w, int32_t* h) {
  FeatDev& fd = c->feat;
  const int L = fd.L;
  if (o < 0 || o >= int(fd.ws.size()) || l < 0 || l > L || (dog && l >= L))
    throw Error(WFK_E_INVALID_ARG, "no such pyramid level");
  *w = fd.ws[size_t(o)];
  *h = fd.hs[size_t(o)];
  const DevBuf<float>& b = fd.levels[o][dog ? L + 1 + l : l];
  if (out) {
    WFK_CUDA(cudaMemcpyAsync(out, b.p, size_t(*w) * size_t(*h) * 4, cudaMemcpyDeviceToHost, c->stream));
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  }
}

}  // namespace wfk
