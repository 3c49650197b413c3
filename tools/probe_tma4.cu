// TMA probe 3: encode via libcuda dlsym vs runtime entry point; warp-converged issue; fp32 2-D map.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int DIM>
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int converged, int bytes, int c0, int c1) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* buf = (float*)sm;
  uint64_t* bar = (uint64_t*)(sm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  bool leader;
  if (converged) {
    uint32_t pred = 0;
    if (threadIdx.x < 32)
      asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}" : "=r"(pred));
    leader = pred != 0;
  } else {
    leader = threadIdx.x == 0;
  }
  if (leader) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    if (DIM == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(buf)), "l"(&map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
  }
  for (int e = threadIdx.x; e < 256; e += blockDim.x) out[e] = buf[e];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int use_dl = 0, converged = 0;
  int es8 = atoi(argv[1]), bx = atoi(argv[2]), by = atoi(argv[3]), c0 = atoi(argv[4]), c1 = atoi(argv[5]);
  int l2 = argc > 6 ? atoi(argv[6]) : 0;
  cudaFree(0);
  float* d; cudaMalloc(&d, 64 * 64 * 4);
  float h[4096]; for (int q = 0; q < 4096; ++q) h[q] = q;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  if (use_dl) {
    void* lib = dlopen("libcuda.so.1", RTLD_NOW);
    fn = lib ? dlsym(lib, "cuTensorMapEncodeTiled") : nullptr;
  } else {
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  }
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  cuuint64_t dims[2] = {64, 64};
  cuuint64_t str[1] = {(cuuint64_t)(es8 ? 32 * 8 : 64 * 4)};
  if (es8) dims[0] = 32;  // 32 doubles per row of the same buffer
  cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}, es[2] = {1, 1};
  CUresult r = ((PFN)fn)(&map, es8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         l2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("es8 %d box %dx%d at (%d,%d) l2 %d encode %d ", es8, bx, by, c0, c1, l2, (int)r);
  float* out; cudaMalloc(&out, 256 * 4);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<2><<<1, 128, 8192>>>(map, out, converged, bx * by * (es8 ? 8 : 4), c0, c1);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[256]; cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("kernel: %s\n", cudaGetErrorString(e));
  return 0;
}
