// Probe: TMA 4-D fp64 boxes of 36 x 12 (ring-2 tiles) with negative start coordinates,
// 6 slots x 4 boxes issued back to back, 84 KB dynamic smem (the k_fsweep pattern).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
constexpr int PLMAX = 40 * 12, SLOT = 4 * PLMAX, RING = 6;
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int c0, int c1, int c2, int nslots, int PL, int nf) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* raw = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  double* ring = (double*)raw;
  uint64_t* bar = (uint64_t*)(raw + RING * SLOT * 8);
  if (threadIdx.x == 0) {
    for (int s = 0; s < RING; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < nslots; ++s) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(4 * PL * 8) : "memory");
      for (int f = 0; f < 4; ++f)
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(smem_u32(ring + s * SLOT + f * ((PL + 15) / 16 * 16))), "l"(&map), "r"(c0), "r"(c1), "r"(c2 + s), "r"(f % nf), "r"(smem_u32(&bar[s])) : "memory");
    }
  }
  for (int s = 0; s < nslots; ++s) {
    uint32_t ok = 0;
    long spins = 0;
    while (!ok && spins < 50000000) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(0) : "memory");
      ++spins;
    }
    if (!ok && threadIdx.x == 0) out[PL] = 12345.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < PL; e += blockDim.x) out[e] = ring[e];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int NX = 80, NY = 80, NZ = 70;
  double* h = new double[(size_t)NX * NY * NZ];
  for (size_t i = 0; i < (size_t)NX * NY * NZ; ++i) h[i] = 1000.0 + i;
  double *d, *o;
  cudaMalloc(&d, sizeof(double) * NX * NY * NZ);
  cudaMalloc(&o, sizeof(double) * (PLMAX + 1));
  cudaMemcpy(d, h, sizeof(double) * NX * NY * NZ, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  const int smem = 1024 + RING * SLOT * 8 + RING * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int cases[1][6];
  if (argc < 7) return 2;
  for (int q = 0; q < 6; ++q) cases[0][q] = atoi(argv[1 + q]);
  for (auto& c : cases) {
    CUtensorMap map;
    const int NF = getenv("NF") ? atoi(getenv("NF")) : 1;
    cuuint64_t dims[4] = {63, 63, 20, (cuuint64_t)NF};
    cuuint64_t strides[3] = {NX * 8, (cuuint64_t)NX * NY * 8, (cuuint64_t)NX * NY * 21 * 8};
    cuuint32_t box[4] = {(cuuint32_t)c[0], (cuuint32_t)c[1], 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d + 2, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 256, smem>>>(map, o, c[2], c[3], c[4], c[5], c[0] * c[1], NF);
    cudaError_t e = cudaDeviceSynchronize();
    printf("box %dx%d coords (%d,%d,%d): encode %d -> %s\n", c[0], c[1], c[2], c[3], c[4], (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, sizeof(double) * NX * NY * NZ); cudaMalloc(&o, sizeof(double) * (PLMAX + 1)); cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); }
  }
  return 0;
}
