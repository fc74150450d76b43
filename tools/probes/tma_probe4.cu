// Probe: layout of a 3D TMA box {8 fp64 (64 B), R rows, 1 slice} written with SWIZZLE_128B into
// shared memory, loads and stores.  Hypothesis checked: element (row r, column c) of the box lands
// at byte a ^ (((a >> 7) & 7) << 4) with a = 64 r + 8 c (the 128-byte swizzle applied to the
// dense 64-byte-row box, base 1024-byte aligned); rows beyond the tensor's extent read as zero.
// Also checks the store direction (smem -> global through the same map).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe4 tma_probe4.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2304_14021_b200/csrc/tma.cuh"
using namespace pd;

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int x0, int y0, int n, int nbox, int rows,
                        double* dump, int do_store) {
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* buf = reinterpret_cast<unsigned char*>(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf + 64 * rows * nbox);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, 64 * rows * nbox);
    for (int b = 0; b < nbox; ++b)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
          ::"r"(smem_u32(buf + 64 * rows * b)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0 + rows * b), "r"(n),
            "r"(smem_u32(bar)) : "memory");
  }
  mbar_wait(bar, 0);
  const double* d = reinterpret_cast<const double*>(buf);
  for (int i = threadIdx.x; i < 8 * rows * nbox; i += blockDim.x) dump[i] = d[i];
  __syncthreads();
  // store the same boxes 8 columns to the right through the same map
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0 && do_store) {
    for (int b = 0; b < nbox; ++b)
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                   ::"l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0 + 8), "r"(y0 + rows * b), "r"(n),
                     "r"(smem_u32(buf + 64 * rows * b)) : "memory");
    tma_commit();
    tma_wait_all();
  }
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1, do_store = argc > 2 ? atoi(argv[2]) : 1;
  const int swz = argc > 3 ? atoi(argv[3]) : 2;
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int nx = 2049, pitch = 2056, ny = 2049, nt = 3;
  const size_t n = (size_t)nt * ny * pitch;
  double *a, *dump;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&dump, 1 << 20);
  std::vector<double> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  int fails = 0;
  struct C { int rows, nbox, x0, y0, n; } cs[] = {{32, 4, 8, 0, 1}, {32, 2, 2040, 2016, 2}, {32, 3, 0, 2000, 0}, {8, 4, 16, 2040, 1}};
  for (int ci = 0; ci < 4; ++ci) {
    if (only >= 0 && ci != only) continue;
    auto& c = cs[ci];
    CUtensorMap m;
    cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nt};
    cuuint64_t st[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * ny * 8};
    cuuint32_t box[3] = {8, (cuuint32_t)c.rows, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz == 2 ? CU_TENSOR_MAP_SWIZZLE_128B : swz == 1 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
    k_probe<<<1, 128, 1024 + 64 * c.rows * c.nbox + 64>>>(m, c.x0, c.y0, c.n, c.nbox, c.rows, dump, do_store);
    cudaError_t e = cudaDeviceSynchronize();
    printf("rows=%d nbox=%d x0=%d y0=%d n=%d encode=%d -> %s\n", c.rows, c.nbox, c.x0, c.y0, c.n, (int)r,
           cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<double> d(8 * c.rows * c.nbox);
    cudaMemcpy(d.data(), dump, d.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0, badplain = 0;
    for (int rr = 0; rr < c.rows * c.nbox; ++rr)
      for (int cc = 0; cc < 8; ++cc) {
        const int y = c.y0 + rr, x = c.x0 + cc;
        const double want = (y < ny && x < nx) ? h[((size_t)c.n * ny + y) * pitch + x] : 0.0;
        const unsigned a0 = 64 * rr + 8 * cc, asw = a0 ^ (((a0 >> 7) & 7) << 4);
        if (d[asw / 8] != want) ++bad;
        if (d[a0 / 8] != want) ++badplain;
      }
    printf("  swizzle hypothesis mismatches %d, unswizzled mismatches %d\n", bad, badplain);
    if (bad && badplain) for (int i = 0; i < 48; ++i) printf("    smem[%d] = %.0f\n", i, d[i]);
    fails += bad != 0 && swz == 2;
    if (!do_store) continue;
    // store check: the boxes went to x0 + 8 in gout (= a, overwritten in place)
    std::vector<double> g(n);
    cudaMemcpy(g.data(), a, n * 8, cudaMemcpyDeviceToHost);
    int sbad = 0;
    for (int rr = 0; rr < c.rows * c.nbox; ++rr)
      for (int cc = 0; cc < 8; ++cc) {
        const int y = c.y0 + rr, x = c.x0 + 8 + cc;
        if (y >= ny || x >= nx) continue;
        const int xs = c.x0 + cc;
        const double want = (xs < nx) ? h[((size_t)c.n * ny + y) * pitch + xs] : 0.0;
        if (g[((size_t)c.n * ny + y) * pitch + x] != want) ++sbad;
      }
    // nothing outside the box (in particular row 2049.. of the slice, column nx..pitch) was written
    int spill = 0;
    for (size_t i = 0; i < n; ++i) {
      const int x = (int)(i % pitch), y = (int)((i / pitch) % ny), nn = (int)(i / ((size_t)pitch * ny));
      const bool inbox = nn == c.n && y >= c.y0 && y < c.y0 + c.rows * c.nbox && x >= c.x0 + 8 && x < c.x0 + 16;
      if (!inbox && g[i] != h[i]) ++spill;
    }
    printf("  store mismatches %d, writes outside the box %d\n", sbad, spill);
    fails += sbad != 0 || spill != 0;
  }
  printf(fails ? "PROBE FAILED\n" : "PROBE OK\n");
  return fails;
}
