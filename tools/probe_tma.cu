// Standalone TMA probe: 4-D box load of one plane of a padded field array.
// variant 0: descriptor = __grid_constant__ param, 1: descriptor in global memory,
// 2: descriptor in __constant__ memory, 3: param + no ".tile" qualifier, 4: 2-D map
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__constant__ CUtensorMap c_map;
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, double* out, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* bar = (uint64_t*)(sm + 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const void* mp = V == 1 ? (const void*)gmap : (V == 2 ? (const void*)&c_map : (const void*)&map);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(34 * 10 * 8) : "memory");
    if (V == 6)
      asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(smem_u32(buf)), "l"(mp), "r"(-1), "r"(-1), "r"(1), "r"(mode), "r"(smem_u32(bar)) : "memory");
    else if (V == 7)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(0) : "memory");
    else if (V == 8)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(buf)), "l"(out), "r"(2720), "r"(smem_u32(bar)) : "memory");
    else if (V == 3)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(smem_u32(buf)), "l"(mp), "r"(-1), "r"(-1), "r"(1), "r"(mode), "r"(smem_u32(bar)) : "memory");
    else if (V == 4)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(buf)), "l"(mp), "r"(-1), "r"(-1), "r"(smem_u32(bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(smem_u32(buf)), "l"(mp), "r"(-1), "r"(-1), "r"(1), "r"(mode), "r"(smem_u32(bar)) : "memory");
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
int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int dtype64 = argc > 2 ? atoi(argv[2]) : 1;
  int n = 64, px = 80, nz = 67;
  size_t fs = (size_t)px * (n + 1) * nz;
  double* d; cudaMalloc(&d, fs * 4 * 8);
  double* h = (double*)malloc(fs * 4 * 8);
  for (size_t q = 0; q < fs * 4; ++q) h[q] = (double)q;
  cudaMemcpy(d, h, fs * 4 * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  CUtensorMap map;
  CUresult r;
  cuuint32_t es[4] = {1, 1, 1, 1};
  if (variant == 4) {
    cuuint64_t dims[2] = {(cuuint64_t)n + 1, (cuuint64_t)(n + 1) * nz * 4};
    cuuint64_t str[1] = {(cuuint64_t)px * 8};
    cuuint32_t box[2] = {34, 10};
    r = ((PFN)fn)(&map, dtype64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT64, 2, d, dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)n + 1, (cuuint64_t)n + 1, (cuuint64_t)nz, 4};
    cuuint64_t str[3] = {(cuuint64_t)px * 8, (cuuint64_t)px * (n + 1) * 8, fs * 8};
    cuuint32_t box[4] = {34, 10, 1, 1};
    r = ((PFN)fn)(&map, dtype64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_INT64, 4, d, dims, str, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("variant %d dtype64 %d encode %d\n", variant, dtype64, (int)r);
  CUtensorMap* gm; cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_map, &map, sizeof(map));
  double* out; cudaMalloc(&out, 340 * 8);
  void (*kk)(CUtensorMap, const CUtensorMap*, double*, int) =
      variant == 0 ? k<0> : variant == 1 ? k<1> : variant == 2 ? k<2> : variant == 3 ? k<3> : variant == 4 ? k<4>
      : variant == 6 ? k<6> : variant == 7 ? k<7> : variant == 8 ? k<8> : k<0>;
  cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  if (variant == 5) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 8192;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, k<0>, map, (const CUtensorMap*)gm, out, 2);
    printf("launchEx: %s\n", cudaGetErrorString(le));
  } else {
    kk<<<1, 128, 8192>>>(map, gm, out, 2);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  double ho[340]; cudaMemcpy(ho, out, 340 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int lj = 0; lj < 10; ++lj) for (int li = 0; li < 34; ++li) {
    int gi = li - 1, gj = lj - 1;
    double ex;
    if (variant == 4) ex = (gi < 0 || gj < 0) ? 0.0 : (double)((size_t)gj * px + gi);
    else ex = (gi < 0 || gj < 0) ? 0.0 : (double)(2 * fs + (size_t)1 * px * (n + 1) + (size_t)gj * px + gi);
    if (ho[lj * 34 + li] != ex) ++bad;
  }
  printf("mismatches %d first %g %g %g\n", bad, ho[0], ho[35], ho[36]);
  return 0;
}
