// Probe: TMA tiled box with negative start coordinates (OOB zero fill) for fp64, 4-D map.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int c0, int c1, int c2) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* bar = (uint64_t*)(sm + 34 * 10 * 8 + 64);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 340; e += blockDim.x) buf[e] = -7.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(340 * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_u32(buf)), "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(smem_u32(bar)) : "memory");
  }
  uint32_t ok = 0;
  long spins = 0;
  while (!ok && spins < 100000000) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
    ++spins;
  }
  if (!ok && threadIdx.x == 0) out[340] = 12345.0;
  __syncthreads();
  for (int e = threadIdx.x; e < 340; e += blockDim.x) out[e] = buf[e];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int NX = 48, NY = 20, NZ = 4;  // pitch 48 doubles
  double* h = new double[NX * NY * NZ];
  for (int i = 0; i < NX * NY * NZ; ++i) h[i] = 1000.0 + i;
  double *d, *o;
  cudaMalloc(&d, sizeof(double) * NX * NY * NZ);
  cudaMalloc(&o, sizeof(double) * 341);
  cudaMemset(o, 0, sizeof(double) * 341);
  cudaMemcpy(d, h, sizeof(double) * NX * NY * NZ, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  // map origin at element (2, 2, 1): logical extent 40 x 16 x 3
  CUtensorMap map;
  cuuint64_t dims[4] = {40, 16, 3, 1};
  cuuint64_t strides[3] = {NX * 8, NX * NY * 8, NX * NY * NZ * 8};
  cuuint32_t box[4] = {34, 10, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d + 1 * NX * NY + 2 * NX + 2, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  int cases[4][3] = {{-2, -1, 0}, {20, 10, 2}, {-2, -1, -1}, {0, 0, 3}};
  int bad = 0;
  for (auto& c : cases) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    k<<<1, 128, 8192>>>(map, o, c[0], c[1], c[2]);
    cudaError_t e = cudaDeviceSynchronize();
    double out[341];
    cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
    int wrong = 0;
    for (int y = 0; y < 10; ++y)
      for (int x = 0; x < 34; ++x) {
        int gx = c[0] + x, gy = c[1] + y, gz = c[2];
        double ex = (gx < 0 || gy < 0 || gz < 0 || gx >= 40 || gy >= 16 || gz >= 3) ? 0.0
                    : h[(gz + 1) * NX * NY + (gy + 2) * NX + gx + 2];
        if (out[y * 34 + x] != ex) ++wrong;
      }
    printf("coords (%d,%d,%d): err=%s wrong=%d timeout=%d\n", c[0], c[1], c[2], cudaGetErrorString(e), wrong, out[340] == 12345.0);
    bad += wrong;
  }
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return 0;
}
