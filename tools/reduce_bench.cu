// Microbenchmark: grid-wide deterministic reduction variants for the
// persistent PCG kernel (148 blocks x 512 threads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// (a) block partial -> cg grid.sync -> every block's warp 0 reads all partials
__global__ void k_a(int iters, double* partials, double* out, double4* vec, int n, int stores) {
  cg::grid_group g = cg::this_grid();
  __shared__ double sm[32];
  __shared__ double bc;
  double acc = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    double v = threadIdx.x * 1e-3 + it;
    for (int s = 0; s < stores; ++s) {
      const int i = (blockIdx.x * blockDim.x + threadIdx.x) * stores + s;
      if (i < n) vec[i] = make_double4(v, v, v, 0);
    }
    v = warp_sum(v);
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    double* base = partials + (it & 1) * gridDim.x;
    if (warp == 0) {
      double s = warp_sum(lane < (blockDim.x >> 5) ? sm[lane] : 0.0);
      if (lane == 0) base[blockIdx.x] = s;
    }
    g.sync();
    if (warp == 0) {
      double vv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) vv[j] = (lane + 32 * j) < gridDim.x ? __ldcg(base + lane + 32 * j) : 0.0;
      double s = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) s += vv[j];
      s = warp_sum(s);
      if (lane == 0) bc = s;
    }
    __syncthreads();
    acc += bc;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

// (b) last-arriving block reduces: partial + atomic counter; the last block
// sums partials in fixed order, publishes the total and bumps the generation;
// everyone waits on the generation word.
__global__ void k_b(int iters, double* partials, unsigned* count, unsigned* gen, double* total, double* out,
                    double4* vec, int n, int stores) {
  __shared__ double sm[32];
  __shared__ double bc;
  double acc = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned my_gen = 0;
  for (int it = 0; it < iters; ++it) {
    double v = threadIdx.x * 1e-3 + it;
    for (int s = 0; s < stores; ++s) {
      const int i = (blockIdx.x * blockDim.x + threadIdx.x) * stores + s;
      if (i < n) vec[i] = make_double4(v, v, v, 0);
    }
    v = warp_sum(v);
    if (lane == 0) sm[warp] = v;
    __syncthreads();
    if (warp == 0) {
      double s = warp_sum(lane < (blockDim.x >> 5) ? sm[lane] : 0.0);
      if (lane == 0) {
        partials[blockIdx.x] = s;
        __threadfence();
        const unsigned old = atom_add_acqrel(count, 1);
        bc = (old == gridDim.x - 1) ? 1.0 : 0.0;
      }
      __syncwarp();
      const bool last = __shfl_sync(0xffffffffu, bc, 0) != 0.0;
      if (last) {
        double vv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) vv[j] = (lane + 32 * j) < gridDim.x ? __ldcg(partials + lane + 32 * j) : 0.0;
        double t = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) t += vv[j];
        t = warp_sum(t);
        if (lane == 0) {
          total[0] = t;
          *count = 0;
          __threadfence();
          st_release(gen, my_gen + 1);
        }
      }
      if (lane == 0) {
        while (ld_acquire(gen) == my_gen) {
        }
        bc = __ldcg(total);
      }
    }
    my_gen += 1;
    __syncthreads();
    acc += bc;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *partials, *out, *total;
  unsigned *count, *gen;
  double4* vec;
  const int n = 1 << 22;
  cudaMalloc(&partials, 4096 * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&total, 8);
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaMalloc(&vec, size_t(n) * 32);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 5000;
  for (int stores : {0, 1, 4}) {
    for (int variant = 0; variant < 2; ++variant) {
      int threads = 512, blocks = sms;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(count, 0, 4);
        cudaMemset(gen, 0, 4);
        cudaEventRecord(e0);
        if (variant == 0) {
          void* args[] = {&iters, &partials, &out, &vec, (void*)&n, &stores};
          cudaLaunchCooperativeKernel((void*)k_a, blocks, threads, args, 0, 0);
        } else {
          void* args[] = {&iters, &partials, &count, &gen, &total, &out, &vec, (void*)&n, &stores};
          cudaLaunchCooperativeKernel((void*)k_b, blocks, threads, args, 0, 0);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("variant %c stores/thread=%d : %.3f us per reduction (%s)\n", 'a' + variant, stores,
             best * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
