// Micro-probe: fp64 FMA throughput and fp64 stream-copy bandwidth on the box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-9, b = 1.0000001, c = 0.9999999;
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
      x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d smem/SM %zu L2 %d MB mem %.1f GB\n", p.name, p.multiProcessorCount, p.sharedMemPerMultiprocessor, p.l2CacheSize >> 20, p.totalGlobalMem / 1e9);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  fma_loop<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0); fma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf("fp64 FMA: %.2f TFLOP/s\n", flops / ms / 1e9);
  size_t n = (size_t)1 << 28; // 2^28 double2 = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMemset(a, 0, n * 16);
  copy_k<<<p.multiProcessorCount * 16, 512>>>(a, b, n);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); copy_k<<<p.multiProcessorCount * 16, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("fp64 copy: %.1f GB/s\n", 2.0 * n * 16 / best / 1e6);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
