// Microbenchmark: grid barrier of the persistent kernel (1 CTA of 512 threads
// per SM) -- flat (every CTA arrives on one counter) vs hierarchical through
// thread-block clusters (cluster barrier, one arrival per cluster, cluster
// barrier).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_barrier_bench cluster_barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
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
template <int CS>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned* count, unsigned* gen, double* out) {
  extern __shared__ double pad[];
  double acc = 0;
  unsigned g = 0;
  const unsigned parts = gridDim.x / CS;
  for (int i = 0; i < iters; ++i) {
    acc += threadIdx.x;
    if (CS > 1) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
    const bool leader = CS == 1 || cg::this_cluster().block_rank() == 0;
    if (leader && threadIdx.x == 0) {
      const unsigned old = atom_add_acqrel(count, 1);
      if (old == parts * (g + 1) - 1) {
        st_release(gen, g + 1);
      } else {
        while (ld_acquire(gen) == g) {
        }
      }
    }
    g += 1;
    if (CS > 1) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc + pad[0] * 0;
}
template <int CS>
void run(int sms, unsigned* count, unsigned* gen, double* out) {
  const int iters = 20000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms / CS * CS);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 150 * 1024;  // one CTA per SM
  cudaFuncSetAttribute(k<CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(count, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k<CS>, iters, count, gen, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("cluster %d: %d CTAs, %.3f us per grid barrier (%s)\n", CS, sms / CS * CS, best * 1e3 / iters,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *count, *gen;
  double* out;
  cudaMalloc(&count, 4);
  cudaMalloc(&gen, 4);
  cudaMalloc(&out, 8);
  run<1>(sms, count, gen, out);
  run<2>(sms, count, gen, out);
  run<4>(132, count, gen, out);
  return 0;
}
