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
#include <map>

#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "wfk_context.cuh"
#include "wfk_solver.cuh"
#include "volume_math.cuh"

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

// capacity for size-varying scratch (extrema, store, matches): powers of two
// from 65536, so growth (cudaMalloc / cudaFree synchronise the device: one
// 47 ms frame where the configs[2] store passed 16 K entries at frame 298) is
// rare -- the 300-frame sequence's store ends at 16.4 K entries
static size_t cap_for(size_t n) {
  size_t c = 65536;
  while (c < n) c *= 2;
  return c;
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
// gaussian_blur (features.cpp:23-46): horizontal then vertical pass with
// clamped borders, both in one kernel -- a 32x8 output tile keeps its
// horizontally blurred rows (with the vertical halo) in shared memory; same
// float operations in the same order as two separate passes.  When `prev` is
// given the DoG level out - prev (features.cpp:80-86) is written as well.
constexpr int kBlurTX = 32, kBlurTY = 8, kBlurMaxR = (kMaxTaps - 1) / 2;
__global__ void __launch_bounds__(kBlurTX* kBlurTY) k_blur(int w, int h, const float* in, float* out, Taps t,
                                                          const float* prev, float* dog) {
  __shared__ float tile[kBlurTY + 2 * kBlurMaxR][kBlurTX];
  const int r = t.radius;
  const int tx = threadIdx.x % kBlurTX, ty = threadIdx.x / kBlurTX;
  const int x = blockIdx.x * kBlurTX + tx, y0 = blockIdx.y * kBlurTY;
  for (int row = ty; row < kBlurTY + 2 * r; row += kBlurTY) {
    const int yy = min(max(y0 - r + row, 0), h - 1);
    float acc = 0;
    if (x < w)
      for (int i = -r; i <= r; ++i) acc += t.k[i + r] * in[int64_t(yy) * w + min(max(x + i, 0), w - 1)];
    tile[row][tx] = acc;
  }
  __syncthreads();
  const int y = y0 + ty;
  if (x >= w || y >= h) return;
  float acc = 0;
  for (int i = -r; i <= r; ++i) acc += t.k[i + r] * tile[ty + r + i][tx];
  const int64_t q = int64_t(y) * w + x;
  out[q] = acc;
  if (prev) dog[q] = acc - prev[q];
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
// dominant_orientations (features.cpp:94-132), one warp per extremum: the
// lanes stage (bin, weight) of a chunk of window samples in shared memory,
// then the lane owning a bin adds that bin's samples in window order -- the
// reference's summation order per bin, so the histogram is the serial one.
constexpr int kOriWarps = 4, kOriChunk = 256, kOriBins = 36;
__global__ void __launch_bounds__(32 * kOriWarps) k_orientations(int n, const int4* ext, const int32_t* order,
                                                                 OctImg im, double sigma, wfk_feature_params p,
                                                                 double* ori, int32_t* nori) {
  __shared__ double sw[kOriWarps][kOriChunk];
  __shared__ int8_t sb[kOriWarps][kOriChunk];
  __shared__ double sh[kOriWarps][kOriBins];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int i = blockIdx.x * kOriWarps + warp;
  if (i >= n) return;  // warp-uniform; only __syncwarp below
  const int4 e = ext[order[i]];
  const float* img = im.g1[e.x];
  const int W = im.w[e.x], H = im.h[e.x];
  const double win_sigma = 1.5 * sigma;
  const int radius = max(1, int(llround(3.0 * win_sigma)));
  const int side = 2 * radius + 1, ns = side * side;
  const int cx = e.y, cy = e.z;
  double h0 = 0, h1 = 0;  // bins lane and lane + 32
  for (int c0 = 0; c0 < ns; c0 += kOriChunk) {
    for (int s = lane; s < kOriChunk; s += 32) {
      const int q = c0 + s;
      int bin = -1;
      double v = 0;
      if (q < ns) {
        const int dy = q / side - radius, dx = q % side - radius;
        const int px = cx + dx, py = cy + dy;
        if (!(px < 1 || py < 1 || px >= W - 1 || py >= H - 1)) {
          const double gx = img[int64_t(py) * W + px + 1] - img[int64_t(py) * W + px - 1];
          const double gy = img[int64_t(py + 1) * W + px] - img[int64_t(py - 1) * W + px];
          const double mag = hypot(gx, gy);
          const double theta = atan2(gy, gx);
          const double w = exp(-0.5 * (dx * dx + dy * dy) / (win_sigma * win_sigma));
          bin = int(floor((theta + M_PI) / (2 * M_PI) * kOriBins));
          bin = min(max(bin, 0), kOriBins - 1);
          v = w * mag;
        }
      }
      sb[warp][s] = int8_t(bin);
      sw[warp][s] = v;
    }
    __syncwarp();
    const int m = min(kOriChunk, ns - c0);
    for (int s = 0; s < m; ++s) {
      const int bq = sb[warp][s];
      if (bq == lane) h0 += sw[warp][s];
      else if (bq == lane + 32) h1 += sw[warp][s];
    }
    __syncwarp();
  }
  sh[warp][lane] = h0;
  if (lane + 32 < kOriBins) sh[warp][lane + 32] = h1;
  __syncwarp();
  if (lane != 0) return;
  const double* hist = sh[warp];
  double peak = hist[0];
  for (int b = 1; b < kOriBins; ++b) peak = fmax(peak, hist[b]);
  int cnt = 0;
  double val[2] = {0, 0}, ang[2] = {0, 0};
  if (peak > 0) {
    // candidates in bin order, stable by decreasing value: keep the best max_orientations (<= 2)
    for (int b = 0; b < kOriBins; ++b) {
      const double l = hist[(b + kOriBins - 1) % kOriBins], r = hist[(b + 1) % kOriBins];
      if (hist[b] >= p.orientation_peak_ratio * peak && hist[b] > l && hist[b] > r) {
        const double denom = l - 2 * hist[b] + r;
        const double off = fabs(denom) > 1e-12 ? 0.5 * (l - r) / denom : 0.0;
        const double a = (b + 0.5 + off) / kOriBins * 2 * M_PI - M_PI;
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
// keypoints in extremum order until max_keypoints (features.cpp:188-207)
struct KpDev {
  int octave, ox, oy, pad;
  double scale, orientation;
};
constexpr int kAsmBlock = 256;
__global__ void __launch_bounds__(kAsmBlock) k_assemble_kp(int n, const int4* ext, const int32_t* order,
                                                           const double* ori, const int32_t* nori, int max_kp,
                                                           double sigma_oct, KpDev* kp, int32_t* n_kp) {
  using Scan = cub::BlockScan<int, kAsmBlock>;
  __shared__ typename Scan::TempStorage ts;
  int base = 0;
  for (int c0 = 0; c0 < n && base < max_kp; c0 += kAsmBlock) {  // base is block-uniform
    const int i = c0 + int(threadIdx.x);
    const int cnt = i < n ? nori[i] : 0;
    int pos, agg;
    Scan(ts).ExclusiveSum(cnt, pos, agg);
    if (cnt > 0) {
      const int4 e = ext[order[i]];
      for (int q = 0; q < cnt && base + pos + q < max_kp; ++q) {
        KpDev k;
        k.octave = e.x;
        k.ox = e.y;
        k.oy = e.z;
        k.pad = 0;
        k.scale = sigma_oct * double(1 << e.x);
        k.orientation = ori[2 * i + q];
        kp[base + pos + q] = k;
      }
    }
    base += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_kp = min(base, max_kp);
}
// extract_descriptors (features.cpp:212-286), one 512-thread block per
// keypoint.  Phase 1 (all threads) stages a chunk of window samples (cell /
// orientation bin corner, fractions, weight) in shared memory; phase 2: the
// lane owning one of the 128 histogram bins (warp = cell, lane = orientation)
// adds that bin's trilinear shares in window order, which is the reference's
// summation order per bin.
constexpr int kDescThreads = 512, kDescChunk = 1024;  // 16 warps: one per descriptor cell
__global__ void __launch_bounds__(kDescThreads) k_descriptors(const int32_t* n_kp, const KpDev* kps, OctImg im,
                                                              double sigma_oct, wfk_feature* out, uint8_t* ok) {
  constexpr int kCells = 4, kBins8 = 8;
  __shared__ double s_fx[kDescChunk], s_fy[kDescChunk], s_fo[kDescChunk], s_w[kDescChunk];
  __shared__ int s_c[kDescChunk];  // x0 + 1 | (y0 + 1) << 8 | o0 << 16, or -1 outside the window
  __shared__ float s_desc[128];
  const int n = *n_kp;
  const int tid = threadIdx.x;
  // phase 2: warp w owns descriptor cell w (x = w % 4, y = w / 4); lane l < 8 its orientation bin l
  const int warp = tid / 32, lane = tid % 32;
  const int my_y = warp / kCells, my_x = warp % kCells, my_o = lane % kBins8;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const KpDev kp = kps[i];
    const float* img = im.g1[kp.octave];
    const int W = im.w[kp.octave], H = im.h[kp.octave];
    const double cell = 3.0 * sigma_oct;
    const double radius = cell * (kCells + 1) * sqrt(2.0) * 0.5;
    const double cx = kp.ox, cy = kp.oy;
    if (cx - radius < 1 || cy - radius < 1 || cx + radius >= W - 1 || cy + radius >= H - 1) {
      if (tid == 0) ok[i] = 0;
      continue;  // block-uniform
    }
    const double ct = cos(kp.orientation), st = sin(kp.orientation);
    const int r = int(ceil(radius));
    const int side = 2 * r + 1, ns = side * side;
    double acc = 0;
    for (int c0 = 0; c0 < ns; c0 += kDescChunk) {
      for (int s = tid; s < kDescChunk; s += kDescThreads) {
        const int q = c0 + s;
        int code = -1;
        if (q < ns) {
          const int dy = q / side - r, dx = q % side - r;
          const double rx = (ct * dx + st * dy) / cell;
          const double ry = (-st * dx + ct * dy) / cell;
          const double bx = rx + kCells / 2.0 - 0.5;
          const double by = ry + kCells / 2.0 - 0.5;
          if (!(bx <= -1 || by <= -1 || bx >= kCells || by >= kCells)) {
            const int px = kp.ox + dx, py = kp.oy + dy;
            const double gx = img[int64_t(py) * W + px + 1] - img[int64_t(py) * W + px - 1];
            const double gy = img[int64_t(py + 1) * W + px] - img[int64_t(py - 1) * W + px];
            const double mag = hypot(gx, gy);
            double theta = atan2(gy, gx) - kp.orientation;
            while (theta < 0) theta += 2 * M_PI;
            while (theta >= 2 * M_PI) theta -= 2 * M_PI;
            const double ob = theta / (2 * M_PI) * kBins8;
            s_w[s] = mag * exp(-0.5 * (rx * rx + ry * ry) / ((kCells / 2.0) * (kCells / 2.0)));
            const int x0 = int(floor(bx)), y0 = int(floor(by));
            const int o0 = int(floor(ob)) % kBins8;
            s_fx[s] = bx - floor(bx);
            s_fy[s] = by - floor(by);
            s_fo[s] = ob - floor(ob);
            code = (x0 + 1) | ((y0 + 1) << 8) | (o0 << 16);
          }
        }
        s_c[s] = code;
      }
      __syncthreads();
      // only samples whose corner cell is (x - 1 .. x, y - 1 .. y) touch cell (x, y):
      // a ballot per 32 samples finds them, the warp walks them in window order
      const int m = min(kDescChunk, ns - c0);
      for (int s0 = 0; s0 < m; s0 += 32) {
        const int sl = s0 + lane;
        const int cl = sl < m ? s_c[sl] : -1;
        const int xl = (cl & 0xff) - 1, yl = ((cl >> 8) & 0xff) - 1;
        unsigned mask = __ballot_sync(0xffffffffu, cl >= 0 && unsigned(my_x - xl) <= 1u && unsigned(my_y - yl) <= 1u);
        while (mask) {
          const int j = __ffs(mask) - 1;
          mask &= mask - 1;
          const int code = __shfl_sync(0xffffffffu, cl, j);
          const int s = s0 + j;
          const int ix = my_x - ((code & 0xff) - 1), iy = my_y - (((code >> 8) & 0xff) - 1);
          const int io = (my_o - (code >> 16) + kBins8) % kBins8;
          if (io > 1) continue;
          const double fx = s_fx[s], fy = s_fy[s], fo = s_fo[s];
          acc += s_w[s] * (ix ? fx : 1 - fx) * (iy ? fy : 1 - fy) * (io ? fo : 1 - fo);
        }
      }
      __syncthreads();
    }
    if (lane < kBins8) s_desc[warp * kBins8 + lane] = float(acc);
    __syncthreads();
    if (tid == 0) {
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
      for (int q = 0; q < 128; ++q) norm += s_desc[q] * s_desc[q];
      norm = sqrt(norm);
      if (norm < 1e-12) {  // flat patch
        ok[i] = 0;
      } else {
        double norm2 = 0;
        for (int q = 0; q < 128; ++q) {
          const float v = fminf(s_desc[q] / float(norm), 0.2f);
          s_desc[q] = v;
          norm2 += v * v;
        }
        norm2 = sqrt(norm2);
        for (int q = 0; q < 128; ++q) f.descriptor[q] = float(s_desc[q] / norm2);
        ok[i] = 1;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// ordered compaction in one block (record order kept: keypoint order, store
// order, match order); n from the device (n_dev) or the host
// ---------------------------------------------------------------------------
constexpr int kCompactBlock = 256;
template <class T>
__global__ void __launch_bounds__(kCompactBlock) k_compact_ordered(const int32_t* n_dev, int n_host, const T* in,
                                                                   const uint8_t* ok, T* out, int32_t* n_out) {
  static_assert(sizeof(T) % 8 == 0, "records are copied as 8-byte words");
  constexpr int kWords = int(sizeof(T) / 8);
  using Scan = cub::BlockScan<int, kCompactBlock>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int src[kCompactBlock];
  const int n = n_dev ? *n_dev : n_host;
  int base = 0;
  for (int c0 = 0; c0 < n; c0 += kCompactBlock) {
    const int i = c0 + int(threadIdx.x);
    const int f = (i < n && ok[i]) ? 1 : 0;
    int pos, agg;
    Scan(ts).ExclusiveSum(f, pos, agg);
    if (f) src[pos] = i;
    __syncthreads();
    // the block copies the kept records word by word (coalesced)
    const uint64_t* a = reinterpret_cast<const uint64_t*>(in);
    uint64_t* b = reinterpret_cast<uint64_t*>(out + base);
    for (int q = threadIdx.x; q < agg * kWords; q += kCompactBlock)
      b[q] = a[int64_t(src[q / kWords]) * kWords + q % kWords];
    base += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = base;
}

// current features' world positions from the frame's maps (pipeline.cpp:194-201)
__global__ void k_feat_world(int n, wfk_feature* f, int W, int H, const double* point, const uint8_t* pvalid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int px = int(lround(f[i].pixel[0])), py = int(lround(f[i].pixel[1]));
  V3 w{0, 0, -1};  // invalid, pruned by matching
  if (px >= 0 && py >= 0 && px < W && py < H && pvalid[int64_t(py) * W + px]) w = ld3(point, int64_t(py) * W + px);
  f[i].world_pos[0] = w.x;
  f[i].world_pos[1] = w.y;
  f[i].world_pos[2] = w.z;
}

// the store's predicted world positions (pipeline.cpp:203-207)
__global__ void k_feat_predict(int64_t n, const wfk_feature* st, Grid g, const double* deformed, PoseD pose,
                               double* pred) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const V3 c{st[i].canonical_pos[0], st[i].canonical_pos[1], st[i].canonical_pos[2]};
    st3(pred, i, g.contains(c) ? pose.apply(g.interpolate(deformed, c)) : V3{0, 0, -1});
  }
}

// ---------------------------------------------------------------------------
// match_features (features.cpp:354-433): the store is stably sorted by frame
// id; the block at the head of each run matches that frame's features against
// the current ones (mutual best, cap, sort, prune) into its slot.
// ---------------------------------------------------------------------------
__global__ void k_match_keys(int64_t n, const wfk_feature* st, uint32_t* key, int32_t* idx) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    key[i] = uint32_t(st[i].frame_id) ^ 0x80000000u;  // signed order
    idx[i] = int32_t(i);
  }
}

struct MatchArgs {
  const wfk_feature* cur;
  int nc;
  const wfk_feature* st;
  int ns;
  const uint32_t* key;  // sorted frame keys
  const int32_t* id;    // store index of each sorted position
  const double* pred;   // 3 * ns, by store index
  wfk_intrinsics K;
  int max_cand, keep, slot;
  double tau_desc, tau_px, tau_3d;
  double* dist;         // ns * nc, by sorted position (groups whose tile exceeds tile_cap)
  int tile_cap;         // doubles of shared memory for a group's distance tile
  int32_t* best_row;    // ns
  double* best_row_d;   // ns
  wfk_feature_match* out;  // slot per sorted position
  int32_t* cnt;            // ns + 1
};

// descriptor_distance (features.cpp:288-295) against a current descriptor
// staged transposed in shared memory: sequential fp64 sum, no fused multiply-add
WF_D double desc_dist_t(const float* a, const float* curT, int ldc, int c) {
  const float2* a2 = reinterpret_cast<const float2*>(a);  // wfk_feature is 600 B: 8-byte aligned
  double s = 0;
#pragma unroll 16
  for (int i = 0; i < 64; ++i) {
    const float2 x = a2[i];
    const double d0 = double(x.x) - double(curT[(2 * i) * ldc + c]);
    const double d1 = double(x.y) - double(curT[(2 * i + 1) * ldc + c]);
    s = __dadd_rn(s, __dmul_rn(d0, d0));
    s = __dadd_rn(s, __dmul_rn(d1, d1));
  }
  return sqrt(s);
}

WF_D bool match_less(const wfk_feature_match& x, const wfk_feature_match& y) {
  return x.distance != y.distance ? x.distance < y.distance : x.source_id < y.source_id;
}

// shared-memory plan of k_match_groups (bytes, 16-aligned pieces)
struct MatchSmem {
  size_t curT, best_col, rows, cand, sorted, tile, total;
  int row_cap;
  static size_t al(size_t x) { return (x + 15) / 16 * 16; }
  MatchSmem(int nc, int max_cand, int row_cap_, int tile_cap) : row_cap(row_cap_) {
    curT = 0;
    best_col = curT + al(size_t(128) * nc * 4);
    rows = best_col + al(size_t(nc) * 4);
    cand = rows + al(size_t(row_cap) * 12);
    sorted = cand + al(size_t(max_cand) * 16);
    tile = sorted + al(size_t(max_cand) * 16);
    total = tile + size_t(tile_cap) * 8;
  }
};

constexpr int kMatchBlock = 256;
__global__ void __launch_bounds__(kMatchBlock) k_match_groups(MatchArgs a, MatchSmem L) {
  extern __shared__ __align__(16) unsigned char msm[];
  using Scan = cub::BlockScan<int, kMatchBlock>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int s_nh;
  const int tid = threadIdx.x;
  const int nc = a.nc;
  float* curT = reinterpret_cast<float*>(msm + L.curT);  // [128][nc]
  int32_t* best_col = reinterpret_cast<int32_t*>(msm + L.best_col);
  wfk_feature_match* cand = reinterpret_cast<wfk_feature_match*>(msm + L.cand);
  wfk_feature_match* sorted = reinterpret_cast<wfk_feature_match*>(msm + L.sorted);
  for (int q = tid; q < 128 * nc; q += kMatchBlock) {  // stage the current descriptors once, transposed
    const int c = q / 128, i = q % 128;
    curT[i * nc + c] = a.cur[c].descriptor[i];
  }
  // the blocks stride over the sorted store; the position heading a frame group does its matching
  for (int b = blockIdx.x; b < a.ns; b += gridDim.x) {
  if (b > 0 && a.key[b] == a.key[b - 1]) {  // not the head of a frame group
    if (tid == 0) a.cnt[b] = 0;
    continue;
  }
  if (tid == 0) {
    int e = b + 1;
    while (e < a.ns && a.key[e] == a.key[b]) ++e;
    s_nh = e - b;
  }
  __syncthreads();
  const int nh = s_nh;
  // per history feature: best current feature and its distance (smem when it fits)
  int32_t* brow = nh <= L.row_cap ? reinterpret_cast<int32_t*>(msm + L.rows) : a.best_row + b;
  double* brow_d = nh <= L.row_cap ? reinterpret_cast<double*>(msm + L.rows + 4 * ((L.row_cap + 3) / 4 * 4))
                                   : a.best_row_d + b;
  // distance matrix of the group (rows: history features in store order), in
  // shared memory when it fits
  double* D = int64_t(nh) * nc <= int64_t(a.tile_cap) ? reinterpret_cast<double*>(msm + L.tile)
                                                       : a.dist + int64_t(b) * nc;
  for (int64_t q = tid; q < int64_t(nh) * nc; q += kMatchBlock) {
    const int h = int(q / nc), c = int(q % nc);
    D[q] = desc_dist_t(a.st[a.id[b + h]].descriptor, curT, nc, c);
  }
  __syncthreads();
  for (int h = tid; h < nh; h += kMatchBlock) {  // best current feature of each history feature
    const double* row = D + int64_t(h) * nc;
    double bd = INFINITY;
    int bc = -1;
    for (int c = 0; c < nc; ++c)
      if (row[c] < bd) {
        bd = row[c];
        bc = c;
      }
    brow[h] = bc;
    brow_d[h] = bd;
  }
  for (int c = tid; c < nc; c += kMatchBlock) {  // best history feature of each current feature
    double bd = INFINITY;
    int bh = -1;
    for (int h = 0; h < nh; ++h) {
      const double d = D[int64_t(h) * nc + c];
      if (d < bd) {
        bd = d;
        bh = h;
      }
    }
    best_col[c] = bh;
  }
  __syncthreads();
  // mutual-best candidates in history order, the first max_cand (features.cpp:372-380)
  int base = 0;
  for (int h0 = 0; h0 < nh && base < a.max_cand; h0 += kMatchBlock) {  // base is block-uniform
    const int h = h0 + tid;
    int c = -1, f = 0;
    if (h < nh) {
      c = brow[h];
      f = (c >= 0 && best_col[c] == h) ? 1 : 0;
    }
    int pos, agg;
    Scan(ts).ExclusiveSum(f, pos, agg);
    if (f && base + pos < a.max_cand) cand[base + pos] = wfk_feature_match{a.id[b + h], c, brow_d[h]};
    base += agg;
    __syncthreads();
  }
  const int nk = min(base, a.max_cand);
  // sort by (distance, source id): a total order, so the rank of each candidate is its place
  for (int k = tid; k < nk; k += kMatchBlock) {
    const wfk_feature_match m = cand[k];
    int r = 0;
    for (int j = 0; j < nk; ++j) r += match_less(cand[j], m) ? 1 : 0;
    sorted[r] = m;
  }
  __syncthreads();
  // keep_best, then the descriptor / reprojection / 3-D prune (features.cpp:382-411), in order
  const int nkeep = min(nk, a.keep);
  int done = 0;
  for (int k0 = 0; k0 < nkeep; k0 += kMatchBlock) {
    const int k = k0 + tid;
    int f = 0;
    wfk_feature_match m{};
    if (k < nkeep) {
      m = sorted[k];
      f = 1;
      if (m.distance > a.tau_desc) f = 0;
      const double* pw = a.pred + 3 * int64_t(m.source_id);
      if (f && pw[2] <= 0) f = 0;
      if (f) {
        const double u = a.K.fx * pw[0] / pw[2] + a.K.cx, v = a.K.fy * pw[1] / pw[2] + a.K.cy;
        const wfk_feature& cf = a.cur[m.target_id];
        const double du = u - cf.pixel[0], dv = v - cf.pixel[1];
        if (sqrt(__dadd_rn(__dmul_rn(du, du), __dmul_rn(dv, dv))) > a.tau_px) f = 0;
        const double ex = pw[0] - cf.world_pos[0], ey = pw[1] - cf.world_pos[1], ez = pw[2] - cf.world_pos[2];
        if (f && sqrt(__dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez))) > a.tau_3d)
          f = 0;
      }
    }
    int pos, agg;
    Scan(ts).ExclusiveSum(f, pos, agg);
    if (f) a.out[int64_t(b) * a.slot + done + pos] = m;
    done += agg;
    __syncthreads();
  }
  if (tid == 0) a.cnt[b] = done;
  __syncthreads();  // shared memory is reused by the block's next group
  }
}

__global__ void k_match_scatter(int n, int slot, const wfk_feature_match* in, const int32_t* cnt, const int32_t* pos,
                                wfk_feature_match* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  for (int k = 0; k < cnt[b]; ++k) out[pos[b] + k] = in[int64_t(b) * slot + k];
}

// sparse_to_constraints (correspond.cpp:152-169) of the matches whose current
// feature has a valid world position (pipeline.cpp:210-215)
__global__ void k_sparse_records(int n, const wfk_feature_match* m, const wfk_feature* cur, const wfk_feature* st,
                                 Grid g, wfk_correspondence* rec, uint8_t* ok) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const wfk_feature& cf = cur[m[i].target_id];
  const wfk_feature& sf = st[m[i].source_id];
  const V3 x{sf.canonical_pos[0], sf.canonical_pos[1], sf.canonical_pos[2]};
  const bool good = cf.world_pos[2] > 0 && g.contains(x);
  ok[i] = good ? 1 : 0;
  if (!good) return;
  wfk_correspondence r;
  r.kind = WFK_SPARSE_POINT;
  r.reserved_ = 0;
  r.canonical[0] = x.x;
  r.canonical[1] = x.y;
  r.canonical[2] = x.z;
  g.anchors(x, r.anchor_index, r.anchor_weight);
  for (int k = 0; k < 3; ++k) {
    r.target[k] = cf.world_pos[k];
    r.target_normal[k] = 0;
  }
  r.confidence = 1.0;
  rec[i] = r;
}

// append the records whose eight anchors are active to the constraint arrays
// (pipeline.cpp:221-235)
__global__ void __launch_bounds__(kCompactBlock) k_append_active(int n, const wfk_correspondence* rec,
                                                                 const uint8_t* ok, const uint8_t* active, int64_t base,
                                                                 int32_t* kind, double* can, int32_t* anchor,
                                                                 double* weight, double* tgt, double* nrm,
                                                                 double* conf, int32_t* n_out) {
  using Scan = cub::BlockScan<int, kCompactBlock>;
  __shared__ typename Scan::TempStorage ts;
  int done = 0;
  for (int c0 = 0; c0 < n; c0 += kCompactBlock) {
    const int i = c0 + int(threadIdx.x);
    int f = 0;
    if (i < n && ok[i]) {
      f = 1;
      for (int k = 0; k < 8; ++k) f &= active[rec[i].anchor_index[k]] ? 1 : 0;
    }
    int pos, agg;
    Scan(ts).ExclusiveSum(f, pos, agg);
    if (f) {
      const wfk_correspondence& r = rec[i];
      const int64_t j = base + done + pos;
      kind[j] = r.kind;
      for (int k = 0; k < 3; ++k) {
        can[3 * j + k] = r.canonical[k];
        tgt[3 * j + k] = r.target[k];
        nrm[3 * j + k] = r.target_normal[k];
      }
      for (int k = 0; k < 8; ++k) {
        anchor[8 * j + k] = r.anchor_index[k];
        weight[8 * j + k] = r.anchor_weight[k];
      }
      conf[j] = r.confidence;
    }
    done += agg;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = done;
}

// add_features (pipeline.cpp:95-141): world position from the maps, canonical
// position by inverting the warp from a rasterized seed within 4 pixels
struct LiftArgs {
  int n;
  const wfk_feature* cur;
  int W, H;
  const double* point;
  const uint8_t* pvalid;
  int bootstrap;
  const float* bdepth;
  const double* bcanon;
  int bw, bh;
  Grid g;
  const double* deformed;
  PoseD pose;
  int frame_id;
  wfk_feature* out;
  uint8_t* ok;
};
__global__ void k_feat_lift(LiftArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  a.ok[i] = 0;
  wfk_feature f = a.cur[i];
  const int px = int(lround(f.pixel[0])), py = int(lround(f.pixel[1]));
  if (px < 0 || py < 0 || px >= a.W || py >= a.H) return;
  const int64_t idx = int64_t(py) * a.W + px;
  if (!a.pvalid[idx]) return;
  const V3 w = ld3(a.point, idx);
  V3 can = w;  // bootstrap frame: the warp is the identity
  if (!a.bootstrap) {
    V3 seed{0, 0, 0};
    bool have = false;
    for (int r = 0; r <= 4 && !have; ++r)
      for (int dy = -r; dy <= r && !have; ++dy)
        for (int dx = -r; dx <= r && !have; ++dx) {
          const int sx = px + dx, sy = py + dy;
          if (sx < 0 || sy < 0 || sx >= a.bw || sy >= a.bh) continue;
          const int64_t q = int64_t(sy) * a.bw + sx;
          if (!isfinite(a.bdepth[q])) continue;  // GeometryBuffer::valid (isosurface.hpp:42)
          seed = ld3(a.bcanon, q);
          have = true;
        }
    if (!have) return;
    if (!invert_warp_point(a.g, a.deformed, a.pose, w, seed, 20, 1e-6, can) || !a.g.contains(can)) return;
  }
  if (!a.g.contains(can)) return;
  f.world_pos[0] = w.x;
  f.world_pos[1] = w.y;
  f.world_pos[2] = w.z;
  f.canonical_pos[0] = can.x;
  f.canonical_pos[1] = can.y;
  f.canonical_pos[2] = can.z;
  f.frame_id = a.frame_id;
  a.out[i] = f;
  a.ok[i] = 1;
}

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
      const dim3 grid((w + kBlurTX - 1) / kBlurTX, (h + kBlurTY - 1) / kBlurTY);
      k_blur<<<grid, kBlurTX * kBlurTY, 0, s>>>(w, h, src, dst, t, l == 0 ? nullptr : G(o, l - 1).p,
                                                l == 0 ? nullptr : D(o, l - 1).ensure(size_t(n)));
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
      int4* ext = fd.ext.ensure(cap_for(size_t(n_ext)));
      uint32_t* key = fd.key.ensure(2 * cap_for(size_t(n_ext)));
      int32_t* idx = fd.idx.ensure(2 * cap_for(size_t(n_ext)));
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
  double* ori = fd.ori.ensure(2 * cap_for(size_t(n_ext)));
  int32_t* nori = fd.nori.ensure(cap_for(size_t(n_ext)));
  k_orientations<<<(n_ext + kOriWarps - 1) / kOriWarps, 32 * kOriWarps, 0, s>>>(n_ext, fd.ext, order, im, sigma_oct,
                                                                               p, ori, nori);
  KpDev* kp = reinterpret_cast<KpDev*>(fd.kp.ensure(size_t(std::max(p.max_keypoints, 1)) * sizeof(KpDev)));
  int32_t* nkp = fd.cnt.ensure(4);  // [0] keypoints, [1] features, [2] sparse kept, [3] store added
  k_assemble_kp<<<1, kAsmBlock, 0, s>>>(n_ext, fd.ext, order, ori, nori, p.max_keypoints, sigma_oct, kp, nkp);
  const int maxk = std::max(p.max_keypoints, 1);
  wfk_feature* cur = reinterpret_cast<wfk_feature*>(fd.cur_raw.ensure(size_t(maxk) * sizeof(wfk_feature)));
  uint8_t* ok = fd.ok.ensure(size_t(maxk));
  k_descriptors<<<std::min(maxk, 4 * c->num_sms), kDescThreads, 0, s>>>(nkp, kp, im, sigma_oct, cur, ok);
  count_launch(c, 3);
  // compact the valid descriptors in keypoint order (features.cpp:279-283)
  wfk_feature* dst = fd.cur.ensure(size_t(maxk));
  int32_t* dn = fd.cnt.p + 1;
  k_compact_ordered<wfk_feature><<<1, kCompactBlock, 0, s>>>(nkp, 0, cur, ok, dst, dn);
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, nkp, 8, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  const int32_t n_kp = c->h_pinned[0];
  fd.n_cur = c->h_pinned[1];
  *n_out = fd.n_cur;
  if (n_kp_out) *n_kp_out = n_kp;
  if (out) {
    if (fd.n_cur > cap) throw Error(WFK_E_CAPACITY, "feature buffer too small");
    if (fd.n_cur > 0) {
      WFK_CUDA(cudaMemcpyAsync(out, dst, size_t(fd.n_cur) * sizeof(wfk_feature), cudaMemcpyDeviceToHost, s));
      WFK_CUDA(cudaStreamSynchronize(s));
    }
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

// ---------------------------------------------------------------------------
// host side of matching, sparse constraints and the store
// ---------------------------------------------------------------------------
namespace {
PoseD pose_dev(const wfk_pose& p) {
  PoseD d;
  for (int i = 0; i < 9; ++i) d.r.a[i / 3][i % 3] = p.rotation[i];
  d.t = V3{p.translation[0], p.translation[1], p.translation[2]};
  return d;
}
void check_match_params(const wfk_feature_params& p) {
  if (p.keep_best < 0 || p.max_candidates > 4096)
    throw Error(WFK_E_INVALID_ARG, "feature params beyond the device limits (keep_best >= 0, max_candidates <= 4096)");
}
}  // namespace

// match_features (features.cpp:416-433) of device arrays; result in fd.matches / fd.n_matches
void features_match_dev(wfk_ctx* c, const wfk_feature* cur, int nc, const wfk_feature* st, int64_t ns,
                        const double* pred, const wfk_intrinsics& K, const wfk_feature_params& p, int64_t max_group) {
  FeatDev& fd = c->feat;
  fd.n_matches = 0;
  check_match_params(p);
  if (nc <= 0 || ns <= 0) return;
  if (ns >= (int64_t(1) << 31) || int64_t(ns) * nc >= (int64_t(1) << 40))
    throw Error(WFK_E_INVALID_ARG, "feature store too large");
  cudaStream_t s = c->stream;
  const int n = int(ns);
  uint32_t* key = fd.skey.ensure(2 * cap_for(size_t(n)));
  int32_t* idx = fd.sidx.ensure(2 * cap_for(size_t(n)));
  k_match_keys<<<grid_for(n), kBlock, 0, s>>>(n, st, key, idx);
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key + n, idx, idx + n, n, 0, 32, s);
  c->temp.ensure(tb);
  WFK_CUDA(cub::DeviceRadixSort::SortPairs(c->temp.p, tb, key, key + n, idx, idx + n, n, 0, 32, s));
  count_launch(c, 2);
  MatchArgs a;
  a.cur = cur;
  a.nc = nc;
  a.st = st;
  a.ns = n;
  a.key = key + n;
  a.id = idx + n;
  a.pred = pred;
  a.K = K;
  a.max_cand = std::max(p.max_candidates, 1);  // the cap is tested after each push
  a.keep = p.keep_best;
  a.slot = std::max(std::min(a.max_cand, a.keep), 1);
  a.tau_desc = p.tau_descriptor;
  a.tau_px = p.tau_pixels;
  a.tau_3d = p.tau_3d;
  a.dist = nullptr;  // set below when a group's distance tile can exceed shared memory
  int32_t* rows = fd.mpos.ensure(2 * cap_for(size_t(n) + 1));
  a.best_row = rows + n + 1;
  a.best_row_d = fd.row_d.ensure(cap_for(size_t(n)));
  a.out = fd.mslot.ensure(cap_for(size_t(n)) * size_t(a.slot));
  a.cnt = fd.mcnt.ensure(cap_for(size_t(n) + 1));
  // shared memory: transposed current descriptors, best rows of groups up to
  // 1024 features, candidates, and the group's distance tile when it fits
  const int row_cap = 1024;
  const MatchSmem L0(nc, a.max_cand, row_cap, 0);
  if (L0.total > 160 * 1024) throw Error(WFK_E_INVALID_ARG, "too many current features for the matcher");
  a.tile_cap = int(std::min<size_t>((200 * 1024 - L0.total) / 8, 16384));
  const MatchSmem L(nc, a.max_cand, row_cap, a.tile_cap);
  if (max_group * nc > a.tile_cap) a.dist = fd.dist.ensure(cap_for(size_t(n) * size_t(nc)));
  WFK_CUDA(cudaFuncSetAttribute(k_match_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total)));
  WFK_CUDA(cudaMemsetAsync(a.cnt + n, 0, 4, s));
  k_match_groups<<<std::min(n, c->num_sms), kMatchBlock, L.total, s>>>(a, L);
  int32_t* pos = rows;  // n + 1 exclusive offsets
  cub::DeviceScan::ExclusiveSum(nullptr, tb, a.cnt, pos, n + 1, s);
  c->temp.ensure(tb);
  WFK_CUDA(cub::DeviceScan::ExclusiveSum(c->temp.p, tb, a.cnt, pos, n + 1, s));
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, pos + n, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  fd.n_matches = c->h_pinned[0];
  if (fd.n_matches > 0) {
    wfk_feature_match* m = fd.matches.ensure(cap_for(size_t(fd.n_matches)));
    k_match_scatter<<<grid_for(n), kBlock, 0, s>>>(n, a.slot, a.out, a.cnt, pos, m);
    count_launch(c);
  }
  count_launch(c, 2);
  WFK_CUDA(cudaGetLastError());
}

void features_match_host(wfk_ctx* c, const wfk_feature* cur, int32_t nc, const wfk_feature* st, int32_t ns,
                         const double* pred, const wfk_intrinsics& K, const wfk_feature_params& p,
                         wfk_feature_match* out, int32_t cap, int32_t* n_out) {
  FeatDev& fd = c->feat;
  cudaStream_t s = c->stream;
  *n_out = 0;
  if (nc < 0 || ns < 0 || (nc > 0 && !cur) || (ns > 0 && (!st || !pred))) throw Error(WFK_E_INVALID_ARG, "bad arrays");
  if (nc == 0 || ns == 0) return;
  wfk_feature* dcur = fd.lift.ensure(cap_for(size_t(nc)));
  wfk_feature* dst = fd.xstore.ensure(size_t(ns));
  double* dp = fd.pred.ensure(3 * cap_for(size_t(ns)));
  WFK_CUDA(cudaMemcpyAsync(dcur, cur, size_t(nc) * sizeof(wfk_feature), cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(dst, st, size_t(ns) * sizeof(wfk_feature), cudaMemcpyHostToDevice, s));
  WFK_CUDA(cudaMemcpyAsync(dp, pred, 3 * size_t(ns) * 8, cudaMemcpyHostToDevice, s));
  std::map<int32_t, int64_t> groups;  // frame id -> entries (sizes the fallback distance area)
  int64_t max_group = 0;
  for (int32_t i = 0; i < ns; ++i) max_group = std::max(max_group, ++groups[st[i].frame_id]);
  features_match_dev(c, dcur, nc, dst, ns, dp, K, p, max_group);
  *n_out = fd.n_matches;
  if (fd.n_matches > cap) throw Error(WFK_E_CAPACITY, "match buffer too small");
  if (fd.n_matches > 0 && out) {
    WFK_CUDA(cudaMemcpyAsync(out, fd.matches.p, size_t(fd.n_matches) * sizeof(wfk_feature_match),
                             cudaMemcpyDeviceToHost, s));
    WFK_CUDA(cudaStreamSynchronize(s));
  }
}

// the sparse term of a frame (pipeline.cpp:185-217): the detected features'
// world positions, the store's predicted positions, matches, constraint records
void features_frame_sparse(wfk_ctx* c, const wfk_intrinsics& K, const wfk_pose& pose, const wfk_feature_params& p,
                           int32_t* match_count) {
  FeatDev& fd = c->feat;
  FrameDev& f = c->frame;
  cudaStream_t s = c->stream;
  fd.n_sparse = 0;
  *match_count = 0;
  if (fd.n_cur == 0) return;
  k_feat_world<<<grid_for(fd.n_cur, 64), 64, 0, s>>>(fd.n_cur, fd.cur, f.K.width, f.K.height, f.point, f.pvalid);
  count_launch(c);
  if (fd.n_store == 0) return;
  double* pred = fd.pred.ensure(3 * cap_for(size_t(fd.n_store)));
  k_feat_predict<<<grid_for(fd.n_store), kBlock, 0, s>>>(fd.n_store, fd.store, c->vol.g, c->vol.deformed,
                                                        pose_dev(pose), pred);
  count_launch(c);
  features_match_dev(c, fd.cur, fd.n_cur, fd.store, fd.n_store, pred, K, p, fd.max_group);
  *match_count = fd.n_matches;
  if (fd.n_matches == 0) return;
  fd.n_sparse = fd.n_matches;
  k_sparse_records<<<grid_for(fd.n_sparse, 64), 64, 0, s>>>(fd.n_sparse, fd.matches, fd.cur, fd.store, c->vol.g,
                                                           fd.sparse.ensure(cap_for(size_t(fd.n_sparse))),
                                                           fd.sparse_ok.ensure(cap_for(size_t(fd.n_sparse))));
  count_launch(c);
  WFK_CUDA(cudaGetLastError());
}

// append the frame's sparse records with all anchors active (pipeline.cpp:229-236)
int64_t features_append_sparse(wfk_ctx* c) {
  FeatDev& fd = c->feat;
  if (fd.n_sparse == 0) return 0;
  ConIn& ci = c->cons;
  cudaStream_t s = c->stream;
  const int64_t base = ci.count;
  const size_t cap = size_t(base + fd.n_sparse) + 1;
  ci.kind.grow_keep(cap, s);
  ci.canonical.grow_keep(3 * cap, s);
  ci.anchor.grow_keep(8 * cap, s);
  ci.weight.grow_keep(8 * cap, s);
  ci.target.grow_keep(3 * cap, s);
  ci.normal.grow_keep(3 * cap, s);
  ci.conf.grow_keep(cap, s);
  int32_t* kept = fd.cnt.ensure(4) + 2;
  k_append_active<<<1, kCompactBlock, 0, s>>>(fd.n_sparse, fd.sparse, fd.sparse_ok, c->vol.active, base, ci.kind,
                                              ci.canonical, ci.anchor, ci.weight, ci.target, ci.normal, ci.conf, kept);
  count_launch(c);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, kept, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  const int64_t m = c->h_pinned[0];
  ci.n_sparse += m;
  ci.count = base + m;
  return m;
}

// add_features (pipeline.cpp:95-141) of the last detection; returns the count added
int32_t features_add(wfk_ctx* c, const wfk_pose& pose, int32_t frame_id, bool bootstrap) {
  FeatDev& fd = c->feat;
  if (fd.n_cur == 0) return 0;
  FrameDev& f = c->frame;
  GBufDev& b = c->gbuf;
  if (!f.maps_valid) throw Error(WFK_E_INVALID_ARG, "add_features: no point/normal maps");
  if (!bootstrap && !b.valid) throw Error(WFK_E_INVALID_ARG, "add_features: no geometry buffer");
  cudaStream_t s = c->stream;
  LiftArgs a;
  a.n = fd.n_cur;
  a.cur = fd.cur;
  a.W = f.K.width;
  a.H = f.K.height;
  a.point = f.point;
  a.pvalid = f.pvalid;
  a.bootstrap = bootstrap ? 1 : 0;
  a.bdepth = bootstrap ? nullptr : b.depth.p;
  a.bcanon = bootstrap ? nullptr : b.canonical.p;
  a.bw = b.w;
  a.bh = b.h;
  a.g = c->vol.g;
  a.deformed = c->vol.deformed;
  a.pose = pose_dev(pose);
  a.frame_id = frame_id;
  a.out = fd.lift.ensure(cap_for(size_t(fd.n_cur)));
  a.ok = fd.lift_ok.ensure(cap_for(size_t(fd.n_cur)));
  k_feat_lift<<<grid_for(a.n, 64), 64, 0, s>>>(a);
  fd.store.grow_keep(cap_for(size_t(fd.n_store + fd.n_cur)), s);
  int32_t* added = fd.cnt.ensure(4) + 3;
  k_compact_ordered<wfk_feature><<<1, kCompactBlock, 0, s>>>(nullptr, a.n, a.out, a.ok, fd.store.p + fd.n_store,
                                                              added);
  count_launch(c, 2);
  WFK_CUDA(cudaMemcpyAsync(c->h_pinned, added, 4, cudaMemcpyDeviceToHost, s));
  WFK_CUDA(cudaStreamSynchronize(s));
  fd.n_store += c->h_pinned[0];
  fd.max_group = std::max<int64_t>(fd.max_group, c->h_pinned[0]);
  return c->h_pinned[0];
}

void features_store_upload(wfk_ctx* c, const wfk_feature* in, int64_t n) {
  if (n < 0 || (n > 0 && !in)) throw Error(WFK_E_INVALID_ARG, "bad feature array");
  FeatDev& fd = c->feat;
  fd.store.ensure(size_t(n));
  if (n > 0)
    WFK_CUDA(cudaMemcpyAsync(fd.store.p, in, size_t(n) * sizeof(wfk_feature), cudaMemcpyHostToDevice, c->stream));
  WFK_CUDA(cudaStreamSynchronize(c->stream));
  fd.n_store = n;
  std::map<int32_t, int64_t> groups;
  fd.max_group = 0;
  for (int64_t i = 0; i < n; ++i) fd.max_group = std::max(fd.max_group, ++groups[in[i].frame_id]);
}

void features_store_download(wfk_ctx* c, wfk_feature* out, int64_t cap, int64_t* n_out) {
  FeatDev& fd = c->feat;
  if (n_out) *n_out = fd.n_store;
  if (!out) return;
  if (fd.n_store > cap) throw Error(WFK_E_CAPACITY, "feature buffer too small");
  if (fd.n_store > 0) {
    WFK_CUDA(cudaMemcpyAsync(out, fd.store.p, size_t(fd.n_store) * sizeof(wfk_feature), cudaMemcpyDeviceToHost,
                             c->stream));
    WFK_CUDA(cudaStreamSynchronize(c->stream));
  }
}

}  // namespace wfk
