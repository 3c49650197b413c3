// Probe: the exact tensor map / box / coordinate set of k_fsweep at n = 64 (one rank),
// one CTA per (tile, chunk, plane, field) case; reports the first failing coordinates.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap map, int c0, int c1, int c2, int c3, int bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* raw = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  uint64_t* bar = (uint64_t*)(raw + 16384);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_u32(raw)), "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)) : "memory");
  }
  uint32_t ok = 0;
  long spins = 0;
  while (!ok && spins < 50000000) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
    ++spins;
  }
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int n = 64, nzl = 65, px = 80, py = px * (n + 2);
  const long fs = ((long)(nzl + 3) * py + 31) / 32 * 32;
  const int BX = argc > 1 ? atoi(argv[1]) : 36, BY = argc > 2 ? atoi(argv[2]) : 12;
  double* d;
  cudaMalloc(&d, sizeof(double) * 4 * fs);
  cudaMemset(d, 0, sizeof(double) * 4 * fs);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)n + 2, (cuuint64_t)n + 2, (cuuint64_t)nzl + 2, 4};
  cuuint64_t strides[3] = {(cuuint64_t)px * 8, (cuuint64_t)py * 8, (cuuint64_t)fs * 8};
  cuuint32_t box[4] = {(cuuint32_t)BX, (cuuint32_t)BY, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("box %dx%d encode %d\n", BX, BY, (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  int xs[2] = {0, 31}, ys[3] = {0, 23, 55}, zs[6] = {0, 1, 30, 64, 66, 67};
  for (int x : xs) for (int y : ys) for (int z : zs) for (int f = 0; f < 4; f += 3) {
    k<<<1, 32, 20000>>>(map, x, y, z, f, BX * BY * 8);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("FAIL x=%d y=%d z=%d f=%d: %s\n", x, y, z, f, cudaGetErrorString(e)); return 1; }
  }
  printf("all ok\n");
  return 0;
}
