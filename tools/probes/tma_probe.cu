// Minimal check of the pair-view TMA staging of tma.cuh (load, swizzled read, TMA store).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../../paper_2304_14021_b200/csrc/tma.cuh"
using namespace pd;

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int ns, int nt) {
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* tile = reinterpret_cast<unsigned char*>(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int BOXB = 16 * (nt / 2) * 8;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tile + 2 * BOXB);
  if (threadIdx.x == 0) {
    if (MODE & 4) tma_prefetch_desc(&tm);
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int s0 = blockIdx.x * 16;
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, 2 * BOXB);
    for (int b = 0; b < 2; ++b) tma_load_2d(tile + b * BOXB, &tm, b * ns + s0, 0, bar);
  }
  mbar_wait(bar, 0);
  if (MODE & 1) {   // plain readback through the swizzle
    for (int i = threadIdx.x; i < nt * 16; i += blockDim.x) {
      const int t = i / 16, c = i % 16;
      if (s0 + c < ns) out[(size_t)t * ns + s0 + c] = *reinterpret_cast<double*>(tile + (t & 1) * BOXB + sw128(t >> 1, c)) + 1.0;
    }
  } else {          // modify in smem, TMA store back in place
    for (int i = threadIdx.x; i < nt * 16; i += blockDim.x) {
      const int t = i / 16, c = i % 16;
      *reinterpret_cast<double*>(tile + (t & 1) * BOXB + sw128(t >> 1, c)) += 1.0;
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && s0 + 16 <= ns) {
      for (int b = 0; b < 2; ++b) tma_store_2d(&tm, b * ns + s0, 0, tile + b * BOXB);
      tma_commit();
      tma_wait_all();
    }
  }
}

int main() {
  const int ns = 65025, nt = 64;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  printf("entry %d\n", (int)cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  std::vector<double> h((size_t)ns * nt);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *a, *o;
  cudaMalloc(&a, h.size() * 8);
  cudaMalloc(&o, h.size() * 8);
  for (int mode : {1, 5, 0}) {
    cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(o, 0, h.size() * 8);
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)(2 * ns), (cuuint64_t)(nt / 2)};
    cuuint64_t st[1] = {(cuuint64_t)(2 * ns * 8)};
    cuuint32_t box[2] = {16, (cuuint32_t)(nt / 2)}, es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 1024 + 2 * 16 * (nt / 2) * 8 + 16;
    const int grid = (ns + 15) / 16;
    if (mode == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<1><<<grid, 128, smem>>>(m, o, ns, nt); }
    if (mode == 5) { cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<5><<<grid, 128, smem>>>(m, o, ns, nt); }
    if (mode == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); k<0><<<grid, 128, smem>>>(m, o, ns, nt); }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> g(h.size());
    cudaMemcpy(g.data(), mode ? o : a, g.size() * 8, cudaMemcpyDeviceToHost);
    size_t bad = 0;
    for (size_t i = 0; i < g.size(); ++i) {
      const bool ragged = (i % ns) >= (size_t)(ns / 16) * 16;
      const double want = h[i] + ((mode || !ragged) ? 1.0 : 0.0);
      if (g[i] != want) ++bad;
    }
    printf("mode %d encode %d err %s bad %zu\n", mode, (int)r, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
