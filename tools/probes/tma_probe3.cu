// Bisect 2: odd box start coordinates, L2 promotion, large dims, dynamic smem alignment.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_2304_14021_b200/csrc/tma.cuh"
using namespace pd;

__global__ void k_tma(const __grid_constant__ CUtensorMap tm, int c0, int c1, double* dst, int rows) {
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* buf = reinterpret_cast<unsigned char*>(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 128 * rows);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(bar, 128 * rows); tma_load_2d(buf, &tm, c0, c1, bar); }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < 16 * rows; i += blockDim.x) dst[i] = reinterpret_cast<double*>(buf)[i];
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t n = (size_t)65025 * 64;
  double* a; cudaMalloc(&a, n * 8); double* d; cudaMalloc(&d, 1 << 20);
  std::vector<double> h(n); for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  struct C { long d0, d1; int rows, c0, c1, promo, sw; } cs[] = {
    {64, 64, 8, 0, 0, 0, 1}, {64, 64, 8, 1, 0, 0, 1}, {64, 64, 8, 2, 0, 0, 1}, {64, 64, 8, 1, 0, 0, 0},
    {130050, 32, 32, 0, 0, 0, 1}, {130050, 32, 32, 0, 0, 2, 1}, {130050, 32, 32, 65025, 0, 0, 1}, {130050, 32, 32, 16, 0, 2, 1}};
  for (auto& c : cs) {
    CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)c.d0, (cuuint64_t)c.d1}; cuuint64_t st[1] = {(cuuint64_t)c.d0 * 8};
    cuuint32_t box[2] = {16, (cuuint32_t)c.rows}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     c.sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     c.promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k_tma<<<1, 128, 1024 + 128 * c.rows + 16>>>(m, c.c0, c.c1, d, c.rows);
    cudaError_t e = cudaDeviceSynchronize();
    printf("d0=%ld rows=%d c0=%d promo=%d sw=%d encode=%d -> %s\n", c.d0, c.rows, c.c0, c.promo, c.sw, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
