// Microbenchmark: latency of one dependent "phase" (load a few values per row,
// store them back) in a single CTA, with __syncthreads between phases.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_phase(double* a, double* b, int rows, int iters) {
  for (int it = 0; it < iters; ++it) {
    const double* src = (it & 1) ? b : a;
    double* dst = (it & 1) ? a : b;
    for (int t = threadIdx.x; t < rows; t += blockDim.x) {
      double v0, v1, v2;
      if (MODE == 0) { v0 = __ldcg(src + t); v1 = __ldcg(src + rows + t); v2 = __ldcg(src + 2 * rows + t); }
      else if (MODE == 1) { v0 = src[t]; v1 = src[rows + t]; v2 = src[2 * rows + t]; }
      else { v0 = __ldcv(src + t); v1 = __ldcv(src + rows + t); v2 = __ldcv(src + 2 * rows + t); }
      dst[t] = v0 + 1.0;
      dst[rows + t] = v1;
      dst[2 * rows + t] = v2;
    }
    __syncthreads();
  }
}
__global__ void k_chase(const int* nxt, int iters, int* out) {  // pointer chase: pure L2 latency
  int p = threadIdx.x;
  for (int i = 0; i < iters; ++i) p = __ldcg(nxt + p);
  out[threadIdx.x] = p;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double *a, *b;
  cudaMalloc(&a, 8 << 20);
  cudaMalloc(&b, 8 << 20);
  cudaMemset(a, 0, 8 << 20);
  cudaMemset(b, 0, 8 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1000;
  for (int rows : {256, 768, 4096}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k_phase<0><<<1, 256>>>(a, b, rows, iters);
        if (mode == 1) k_phase<1><<<1, 256>>>(a, b, rows, iters);
        if (mode == 2) k_phase<2><<<1, 256>>>(a, b, rows, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("rows=%d mode=%s: %.3f us per phase\n", rows, mode == 0 ? "ldcg" : mode == 1 ? "ld  " : "ldcv", ms * 1e3 / iters);
      }
    }
  }
  // pointer chase latency
  int* nxt;
  int* out;
  const int N = 1 << 20;
  cudaMalloc(&nxt, N * sizeof(int));
  cudaMalloc(&out, 1024 * sizeof(int));
  int* h = new int[N];
  for (int i = 0; i < N; ++i) h[i] = (int)((i * 2654435761u + 12345u) % N) & ~31;  // stride over lines
  cudaMemcpy(nxt, h, N * sizeof(int), cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k_chase<<<1, 1>>>(nxt, 10000, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) printf("pointer chase (4 MB, L2): %.1f ns per load\n", ms * 1e6 / 10000);
  }
  return 0;
}
