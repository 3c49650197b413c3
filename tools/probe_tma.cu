// Standalone TMA probe: 4-D box load of one plane of a padded field array.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* bar = (uint64_t*)(sm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(34 * 10 * 8) : "memory");
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(smem_u32(buf)), "l"(&map), "r"(-1), "r"(-1), "r"(1), "r"(mode), "r"(smem_u32(bar)) : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
  }
  for (int e = threadIdx.x; e < 340; e += blockDim.x) out[e] = buf[e];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  int n = 64, px = 80, nz = 67;
  size_t fs = (size_t)px * (n + 1) * nz;
  double* d; cudaMalloc(&d, fs * 4 * 8);
  double* h = (double*)malloc(fs * 4 * 8);
  for (size_t q = 0; q < fs * 4; ++q) h[q] = (double)q;
  cudaMemcpy(d, h, fs * 4 * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  printf("entry %p status %d\n", fn, (int)qr);
  CUtensorMap map;
  cuuint64_t dims[4] = {(cuuint64_t)n + 1, (cuuint64_t)n + 1, (cuuint64_t)nz, 4};
  cuuint64_t str[3] = {(cuuint64_t)px * 8, (cuuint64_t)px * (n + 1) * 8, fs * 8};
  cuuint32_t box[4] = {34, 10, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = ((PFN)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  double* out; cudaMalloc(&out, 340 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<<<1, 128, 8192>>>(map, out, 2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double ho[340]; cudaMemcpy(ho, out, 340 * 8, cudaMemcpyDeviceToHost);
  // expected: field 2, plane 1, rows -1..8, cols -1..32 (OOB = 0)
  int bad = 0;
  for (int lj = 0; lj < 10; ++lj) for (int li = 0; li < 34; ++li) {
    int gi = li - 1, gj = lj - 1;
    double ex = (gi < 0 || gj < 0) ? 0.0 : (double)(2 * fs + (size_t)1 * px * (n + 1) + (size_t)gj * px + gi);
    if (ho[lj * 34 + li] != ex) ++bad;
  }
  printf("mismatches %d\n", bad);
  return 0;
}
