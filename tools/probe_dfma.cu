// fp64 DFMA dependent-chain latency and throughput, LDS.64 latency (one warp / full SM)
#include <cstdio>
__global__ void k_chain(double* out, int iters, double a, double b) {
  double x = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / (iters * 16.0);
  out[1 + threadIdx.x] = x;
}
__global__ void k_tput(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
  out[1 + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_lds(double* out, int iters) {
  __shared__ int nxt[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i + 33) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = nxt[p];
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
  out[1 + threadIdx.x] = p;
}
int main() {
  double* d;
  cudaMalloc(&d, 8 * 4096);
  double h;
  k_chain<<<1, 32>>>(d, 1000, 1.0000001, 1e-9);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h);
  for (int w : {1, 4, 8, 16, 32}) {
    k_tput<<<1, 32 * w>>>(d, 1000, 1.0000001, 1e-9);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 independent chains, %2d warps on one SM: %.2f cycles per iteration (8 DFMA per thread)\n", w, h);
  }
  k_lds<<<1, 32>>>(d, 1000);
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", h);
  return 0;
}
