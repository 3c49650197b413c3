// TMA probe 3: encode via libcuda dlsym vs runtime entry point; warp-converged issue; fp32 2-D map.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <dlfcn.h>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int DIM>
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int converged) {
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
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(32 * 8 * 4) : "memory");
    if (DIM == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(buf)), "l"(&map), "r"(0), "r"(0), "r"(smem_u32(bar)) : "memory");
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
  int use_dl = atoi(argv[1]), converged = atoi(argv[2]);
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
  cuuint64_t str[1] = {64 * 4};
  cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult r = ((PFN)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("dl %d conv %d fn %p encode %d desc:", use_dl, converged, fn, (int)r);
  for (int q = 0; q < 16; ++q) printf(" %016llx", (unsigned long long)((uint64_t*)&map)[q]);
  printf("\n");
  float* out; cudaMalloc(&out, 256 * 4);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  k<2><<<1, 128, 8192>>>(map, out, converged);
  cudaError_t e = cudaDeviceSynchronize();
  float ho[256]; cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < 8; ++y) for (int x = 0; x < 32; ++x) if (ho[y * 32 + x] != (float)(y * 64 + x)) ++bad;
  printf("kernel: %s mismatches %d\n", cudaGetErrorString(e), bad);
  return 0;
}
