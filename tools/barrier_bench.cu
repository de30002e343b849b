// Microbenchmark: cost of a grid-wide barrier on B200 for persistent kernels.
// (a) cooperative_groups::this_grid().sync()
// (b) hand-rolled sense-reversing barrier: one red.release per block, leader
//     spins with ld.acquire on a flag word.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// counter-based barrier: generation g, each block adds 1; the last arriver
// bumps the generation word; others wait for it
__device__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks, unsigned& my_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = my_gen;
    const unsigned old = atom_add_acqrel(count, 1);
    if (old == nblocks - 1) {
      *count = 0;
      red_release_add(gen, 1);
    } else {
      while (ld_acquire(gen) == g0) {
      }
    }
  }
  my_gen += 1;
  __syncthreads();
}

__global__ void k_custom(int iters, unsigned* count, unsigned* gen, double* out) {
  unsigned my_gen = 0;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    grid_barrier(count, gen, gridDim.x, my_gen);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  unsigned *count, *gen;
  cudaMalloc(&out, 8);
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int threads : {256, 512, 1024}) {
    for (int per : {1, 2}) {
      if (threads * per > 1024 && threads == 1024) continue;
      int blocks = sms * per;
      int iters = 20000;
      void* args[] = {&iters, &out};
      cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_cg, blocks, threads, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      cudaError_t e = cudaGetLastError();
      printf("cg::grid.sync   blocks=%4d threads=%4d : %.3f us/sync %s\n", blocks, threads, ms * 1e3 / iters,
             cudaGetErrorString(e));
      cudaMemset(count, 0, 4);
      cudaMemset(gen, 0, 4);
      void* args2[] = {&iters, &count, &gen, &out};
      cudaLaunchCooperativeKernel((void*)k_custom, blocks, threads, args2, 0, 0);
      cudaMemset(count, 0, 4);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_custom, blocks, threads, args2, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      e = cudaGetLastError();
      printf("custom barrier  blocks=%4d threads=%4d : %.3f us/sync %s\n", blocks, threads, ms * 1e3 / iters,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
