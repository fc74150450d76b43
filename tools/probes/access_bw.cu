// Micro-probe: HBM bandwidth of the access patterns the 2D ParaDiag passes use (no arithmetic).
//   rowsT<R,X>: read R full-width row segments (contiguous, length X) of the [n][y][x] layout, write
//               them transposed into [n][x][y] (pitch P): R contiguous doubles per x.
//   colsT<R,X>: the reverse (read R-wide segments of [n][x][y], write rows).
//   tile<S>:    read / write S consecutive points of all NT time slices (stride ns) — time pencils.
// Built here, run on the box:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a access_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NX = 2049, PITCH = 2056;

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// A[n][y][x] (pitch NX) -> B[n][x][y] (pitch PITCH); CTA tile = R rows x X columns
template <int R, int X>
__global__ void __launch_bounds__(256) rowsT(const double* __restrict__ A, double* __restrict__ B, int nslices) {
  __shared__ double t[R][X + 1];
  const int tx = (NX + X - 1) / X, ty = (NX + R - 1) / R;
  const long ntiles = (long)nslices * tx * ty;
  for (long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const int n = g / (tx * ty), rem = g % (tx * ty), iy = rem / tx, ix = rem % tx;
    const int y0 = iy * R, x0 = ix * X;
    const double* a = A + (size_t)n * NX * NX;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int r = i / X, c = i % X;
      const int y = y0 + r, x = x0 + c;
      t[r][c] = (y < NX && x < NX) ? a[(size_t)y * NX + x] : 0.0;
    }
    __syncthreads();
    double* b = B + (size_t)n * NX * PITCH;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int c = i / R, r = i % R;
      const int y = y0 + r, x = x0 + c;
      if (y < NX && x < NX) b[(size_t)x * PITCH + y] = t[r][c];
    }
    __syncthreads();
  }
}

// B[n][x][y] -> A[n][y][x]
template <int R, int X>
__global__ void __launch_bounds__(256) colsT(const double* __restrict__ B, double* __restrict__ A, int nslices) {
  __shared__ double t[R][X + 1];
  const int tx = (NX + X - 1) / X, ty = (NX + R - 1) / R;
  const long ntiles = (long)nslices * tx * ty;
  for (long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const int n = g / (tx * ty), rem = g % (tx * ty), iy = rem / tx, ix = rem % tx;
    const int y0 = iy * R, x0 = ix * X;
    const double* b = B + (size_t)n * NX * PITCH;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int c = i / R, r = i % R;
      const int y = y0 + r, x = x0 + c;
      t[r][c] = (y < NX && x < NX) ? b[(size_t)x * PITCH + y] : 0.0;
    }
    __syncthreads();
    double* a = A + (size_t)n * NX * NX;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int r = i / X, c = i % X;
      const int y = y0 + r, x = x0 + c;
      if (y < NX && x < NX) a[(size_t)y * NX + x] = t[r][c];
    }
    __syncthreads();
  }
}

// time tiles: S points x NT slices, in place-ish copy in -> out (same layout)
template <int S>
__global__ void __launch_bounds__(256) tile_k(const double* __restrict__ in, double* __restrict__ out, size_t ns, int NT) {
  extern __shared__ double t[];
  const long ntiles = (ns + S - 1) / S;
  for (long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const size_t s0 = g * S;
    for (int i = threadIdx.x; i < S * NT; i += 256) {
      const int j = i / S, c = i % S;
      t[j * (S + 1) + c] = s0 + c < ns ? in[(size_t)j * ns + s0 + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < S * NT; i += 256) {
      const int j = i / S, c = i % S;
      if (s0 + c < ns) out[(size_t)j * ns + s0 + c] = t[j * (S + 1) + c] * 1.0000001;
    }
    __syncthreads();
  }
}


__device__ __forceinline__ void pf_l2(const void* p, unsigned bytes) {
  const size_t a = (size_t)p & ~(size_t)15, e = ((size_t)p + bytes + 15) & ~(size_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}
// time tiles with an L2 bulk prefetch of the CTA's next tile issued before the current tile's loads
template <int S>
__global__ void __launch_bounds__(256) tile_pf(const double* __restrict__ in, double* __restrict__ out, size_t ns, int NT) {
  extern __shared__ double t[];
  const long ntiles = (ns + S - 1) / S;
  for (long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const size_t s0 = g * S;
    const long gn = g + gridDim.x;
    if (gn < ntiles)
      for (int j = threadIdx.x; j < NT; j += 256) pf_l2(in + (size_t)j * ns + gn * S, S * 8);
    for (int i = threadIdx.x; i < S * NT; i += 256) {
      const int j = i / S, c = i % S;
      t[j * (S + 1) + c] = s0 + c < ns ? in[(size_t)j * ns + s0 + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < S * NT; i += 256) {
      const int j = i / S, c = i % S;
      if (s0 + c < ns) out[(size_t)j * ns + s0 + c] = t[j * (S + 1) + c] * 1.0000001;
    }
    __syncthreads();
  }
}
// B[n][x][y] -> A[n][y][x] with prefetch of the next tile
template <int R, int X>
__global__ void __launch_bounds__(256) colsT_pf(const double* __restrict__ B, double* __restrict__ A, int nslices) {
  __shared__ double t[R][X + 1];
  const int tx = (NX + X - 1) / X, ty = (NX + R - 1) / R;
  const long ntiles = (long)nslices * tx * ty;
  for (long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const int n = g / (tx * ty), rem = g % (tx * ty), iy = rem / tx, ix = rem % tx;
    const int y0 = iy * R, x0 = ix * X;
    const long gn = g + gridDim.x;
    if (gn < ntiles) {
      const int nn = gn / (tx * ty), rr = gn % (tx * ty), yy = (rr / tx) * R, xx = (rr % tx) * X;
      const double* bn = B + (size_t)nn * NX * PITCH;
      for (int c = threadIdx.x; c < X; c += 256)
        if (xx + c < NX) pf_l2(bn + (size_t)(xx + c) * PITCH + yy, R * 8);
    }
    const double* b = B + (size_t)n * NX * PITCH;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int c = i / R, r = i % R;
      const int y = y0 + r, x = x0 + c;
      t[r][c] = (y < NX && x < NX) ? b[(size_t)x * PITCH + y] : 0.0;
    }
    __syncthreads();
    double* a = A + (size_t)n * NX * NX;
    for (int i = threadIdx.x; i < R * X; i += 256) {
      const int r = i / X, c = i % X;
      const int y = y0 + r, x = x0 + c;
      if (y < NX && x < NX) a[(size_t)y * NX + x] = t[r][c];
    }
    __syncthreads();
  }
}
template <class F>
float timeit(F f);

template <class F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const int ns_slices = 128;
  const size_t nA = (size_t)ns_slices * NX * NX, nB = (size_t)ns_slices * NX * PITCH;
  double *A, *B;
  cudaMalloc(&A, nB * 8);
  cudaMalloc(&B, nB * 8);
  cudaMemset(A, 0, nB * 8);
  cudaMemset(B, 0, nB * 8);
  const double gb = 2.0 * nA * 8 / 1e9;
  int nsm = 148;
  {
    float ms = timeit([&] { copy_k<<<nsm * 16, 512>>>((double2*)A, (double2*)B, nA / 2); });
    printf("copy contiguous           %8.1f GB/s\n", gb / ms * 1e3);
  }
#define RT(R, X)                                                                                   \
  {                                                                                                \
    float ms = timeit([&] { rowsT<R, X><<<nsm * 4, 256>>>(A, B, ns_slices); });                    \
    float ms2 = timeit([&] { colsT<R, X><<<nsm * 4, 256>>>(B, A, ns_slices); });                   \
    printf("rowsT R=%2d X=%4d %8.1f GB/s   colsT %8.1f GB/s\n", R, X, gb / ms * 1e3, gb / ms2 * 1e3); \
  }
  RT(4, 1024) RT(8, 512) RT(16, 256) RT(32, 128) RT(4, 512) RT(8, 256) RT(16, 128)
#define TT(S, NT)                                                                                   \
  {                                                                                                 \
    const size_t ns = nA / NT;                                                                      \
    const size_t sm = (size_t)NT * (S + 1) * 8;                                                     \
    cudaFuncSetAttribute(tile_k<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);          \
    int per = (int)(200000 / sm); per = per < 1 ? 1 : per > 8 ? 8 : per;                             \
    float ms = timeit([&] { tile_k<S><<<nsm * per, 256, sm>>>(A, B, ns, NT); });                    \
    printf("time tile S=%2d NT=%4d     %8.1f GB/s (%d CTA/SM)\n", S, NT, gb / ms * 1e3, per);        \
  }
  TT(4, 512) TT(8, 512) TT(16, 512) TT(32, 256) TT(16, 128) TT(32, 128)

#define TP(S, NT, PER)                                                                              \
  {                                                                                                 \
    const size_t ns = nA / NT;                                                                      \
    const size_t sm = (size_t)NT * (S + 1) * 8;                                                     \
    cudaFuncSetAttribute(tile_pf<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);         \
    float ms = timeit([&] { tile_pf<S><<<nsm * PER, 256, sm>>>(A, B, ns, NT); });                   \
    printf("time tile+pf S=%2d NT=%4d  %8.1f GB/s (%d CTA/SM)\n", S, NT, gb / ms * 1e3, PER);       \
  }
  TP(8, 512, 2) TP(8, 512, 4) TP(16, 512, 1) TP(16, 512, 2) TP(32, 256, 2) TP(16, 128, 4)
#define CP(R, X)                                                                                    \
  {                                                                                                 \
    float ms2 = timeit([&] { colsT_pf<R, X><<<nsm * 4, 256>>>(B, A, ns_slices); });                 \
    printf("colsT+pf R=%2d X=%4d %8.1f GB/s\n", R, X, gb / ms2 * 1e3);                               \
  }
  CP(8, 512) CP(16, 256) CP(32, 128)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
