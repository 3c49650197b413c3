// Probe: 4-D fp64 tile map (box 32x8x1x1) as used for the staged auxiliary
// fields, 4 fields landing on one mbarrier next to a 34x10 halo box.
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int c0, int c1, int c2, int nf, int bsz) {
  extern __shared__ __align__(1024) unsigned char sm[];
  double* buf = (double*)sm;
  uint64_t* bar = (uint64_t*)(sm + 4 * 4096);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(nf * bsz * 8) : "memory");
    for (int f = 0; f < nf; ++f)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(smem_u32(buf + f * 512)), "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(f), "r"(smem_u32(bar)) : "memory");
  }
  uint32_t ok = 0;
  long spins = 0;
  while (!ok && spins < 100000000) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(0) : "memory");
    ++spins;
  }
  if (!ok && threadIdx.x == 0) out[4000] = 12345.0;
  __syncthreads();
  for (int e = threadIdx.x; e < nf * 512; e += blockDim.x) out[e] = buf[e];
}
typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int BX = argc > 1 ? atoi(argv[1]) : 32, BY = argc > 2 ? atoi(argv[2]) : 8, NF = argc > 3 ? atoi(argv[3]) : 4;
  const int L2P = argc > 4 ? atoi(argv[4]) : 1;
  const int ORG = argc > 5 ? atoi(argv[5]) : 1;   // origin row offset (0: base, 1: +px)
  const int NZX = argc > 6 ? atoi(argv[6]) : 0;   // 1: dims z = 3 (small)
  const int n = 64, nzl = 65;
  const long px = ((n + 3 + 15) / 16) * 16, py = px * (n + 2), fs = (((long)(nzl + 2) * py + 31) / 32) * 32;
  const long tot = 4 * fs;
  double* h = new double[tot];
  for (long i = 0; i < tot; ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, sizeof(double) * tot);
  cudaMalloc(&o, sizeof(double) * 4096);
  cudaMemcpy(d, h, sizeof(double) * tot, cudaMemcpyHostToDevice);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  PFN enc = (PFN)p;
  CUtensorMap map;
  const double* origin = d + ORG * px;
  cuuint64_t dims[4] = {(cuuint64_t)(n + 2), (cuuint64_t)(n + 2 - ORG), (cuuint64_t)(NZX ? 3 : nzl + 2), 4};
  cuuint64_t strides[3] = {(cuuint64_t)px * 8, (cuuint64_t)py * 8, (cuuint64_t)fs * 8};
  cuuint32_t box[4] = {(cuuint32_t)BX, (cuuint32_t)BY, 1, 1}, es[4] = {1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)origin, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, L2P ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("box %dx%d nf %d l2p %d org %d nzx %d encode %d\n", BX, BY, NF, L2P, ORG, NZX, (int)r);
  int bad = 0;
  int cases[3][3] = {{1, 0, 1}, {33, 56, 66}, {1, 8, 0}};
  for (auto& c : cases) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64);
    k<<<1, 128, 16384 + 64>>>(map, o, c[0], c[1], c[2], NF, BX * BY);
    cudaError_t e = cudaDeviceSynchronize();
    static double out[4096];
    cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
    int wrong = 0;
    for (int f = 0; f < NF; ++f)
      for (int y = 0; y < BY; ++y)
        for (int x = 0; x < BX; ++x) {
          const long gx = c[0] + x, gy = c[1] + y, gz = c[2];
          double ex = (gx >= n + 2 || gy >= n + 2 - ORG || gz >= (NZX ? 3 : nzl + 2)) ? 0.0 : h[ORG * px + f * fs + gz * py + gy * px + gx];
          if (out[f * 512 + y * BX + x] != ex) ++wrong;
        }
    printf("coords (%d,%d,%d): err=%s wrong=%d timeout=%d\n", c[0], c[1], c[2], cudaGetErrorString(e), wrong, out[4000] == 12345.0);
    bad += wrong + (e != cudaSuccess);
    if (e != cudaSuccess) break;
  }
  printf(bad ? "PROBE FAIL\n" : "PROBE OK\n");
  return 0;
}
