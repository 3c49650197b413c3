// Microbenchmark: cost of the software grid barrier variants (no work between).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1604_07994_b200/csrc/kernels_fused.cuh"
using namespace stk;

__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// monotonic-counter barrier: one atomic per CTA, spin until the count reaches the next multiple of M
__device__ __forceinline__ void mono_barrier(unsigned long long* cnt, int M) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(cnt) : "memory");
    const unsigned long long target = (old / M + 1) * M;
    while (ld_acq64(cnt) < target) {
    }
  }
  __syncthreads();
}

__global__ void k_bar_gen(unsigned* bar, int iters, int M) {
  for (int i = 0; i < iters; ++i)
    if ((int)blockIdx.x < M) grid_barrier(bar, M);
}
__global__ void k_bar_mono(unsigned long long* cnt, int iters, int M) {
  for (int i = 0; i < iters; ++i)
    if ((int)blockIdx.x < M) mono_barrier(cnt, M);
}
__global__ void k_empty() {}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  unsigned* bar;
  unsigned long long* cnt;
  cudaMalloc(&bar, 8 * 4096);
  cudaMalloc(&cnt, 8);
  cudaMemset(bar, 0, 8 * 4096);
  cudaMemset(cnt, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int G : {148, 296}) {
    for (int M : {1, 3, 20, 148, 296}) {
      if (M > G) continue;
      for (int v = 0; v < 2; ++v) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(G);
        lc.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(cnt, 0, 8);  // the monotonic counter must start at a multiple of M
          cudaEventRecord(e0);
          cudaError_t e = v == 0 ? cudaLaunchKernelEx(&lc, k_bar_gen, bar, iters, M)
                                 : cudaLaunchKernelEx(&lc, k_bar_mono, cnt, iters, M);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep == 1) printf("G=%d M=%d %s: %.3f us per barrier (%s)\n", G, M, v ? "mono" : "gen ", ms * 1e3 / iters,
                               cudaGetErrorString(e));
        }
      }
    }
  }
  // launch latency of empty kernels back to back, plain and in a graph
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int i = 0; i < 10; ++i) k_empty<<<148, 256, 0, s>>>();
  cudaEventRecord(e0, s);
  for (int i = 0; i < 1000; ++i) k_empty<<<148, 256, 0, s>>>();
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty kernel stream launch: %.3f us each\n", ms);
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
  for (int i = 0; i < 1000; ++i) k_empty<<<148, 256, 0, s>>>();
  cudaStreamEndCapture(s, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty kernel in graph: %.3f us each\n", ms);
  return 0;
}
