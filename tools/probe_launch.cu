// Per-kernel cost of tiny dependent kernels replayed in a CUDA graph (the coarse
// V-cycle levels are ~400 such kernels per cycle).
#include <cstdio>
#include <cuda_runtime.h>
struct Big { double* p[16]; long long v[16]; };
__global__ void k_empty(int n) {}
__global__ void k_copy(const double* __restrict__ a, double* __restrict__ b, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) b[t] = a[t] + 1.0;
}
__global__ void k_copy_big(const __grid_constant__ Big B, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) B.p[1][t] = B.p[0][t] + 1.0;
}
__global__ void k_chain3(const double* __restrict__ a, double* __restrict__ b, const int* idx, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) { int i1 = __ldg(idx + t); int i2 = __ldg(idx + i1); b[t] = a[i2] + 1.0; }
}
// the same with programmatic dependent launch: index math before the wait
__global__ void k_chain3_pdl(const double* a, double* b, const int* idx, int n) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (t < n) { int i1 = idx[t]; int i2 = idx[i1]; b[t] = a[i2] + 1.0; }
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  double *a, *b; int* idx;
  cudaMalloc(&a, 1 << 24); cudaMalloc(&b, 1 << 24); cudaMalloc(&idx, 1 << 22);
  cudaMemset(a, 0, 1 << 24); cudaMemset(b, 0, 1 << 24); cudaMemset(idx, 0, 1 << 22);
  Big B{}; B.p[0] = a; B.p[1] = b;
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int R = 400;
  for (int n : {729, 4913, 35937, 274625}) {
    const int nb = (n + 127) / 128;
    for (int kind = 0; kind < 5; ++kind) {
      cudaGraph_t gr; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
      for (int r = 0; r < R; ++r) {
        if (kind == 0) k_empty<<<nb, 128, 0, s>>>(n);
        if (kind == 1) k_copy<<<nb, 128, 0, s>>>((r & 1) ? b : a, (r & 1) ? a : b, n);
        if (kind == 2) k_copy_big<<<nb, 128, 0, s>>>(B, n);
        if (kind == 3) k_chain3<<<nb, 128, 0, s>>>(a, b, idx, n);
        if (kind == 4) {
          cudaLaunchConfig_t lc{};
          lc.gridDim = dim3(nb); lc.blockDim = dim3(128); lc.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          lc.attrs = at; lc.numAttrs = 1;
          cudaLaunchKernelEx(&lc, k_chain3_pdl, (const double*)a, b, (const int*)idx, n);
        }
      }
      cudaStreamEndCapture(s, &gr);
      cudaGraphInstantiate(&ge, gr, 0);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e0, s);
      cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      static const char* nm[] = {"empty", "copy", "copy_bigparam", "chain3", "chain3_pdl"};
      printf("n=%7d %-14s %.3f us per kernel in graph\n", n, nm[kind], ms * 1e3 / R);
      cudaGraphExecDestroy(ge); cudaGraphDestroy(gr);
    }
  }
  return 0;
}
